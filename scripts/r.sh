ISDC_SR_TY=48 python -m pytest tests/test_gpu_fullsize.py -x -q -k "cfg3" 2>&1 | tail -2 > gpurun_out/par.log
for t in 40 48 40 48; do ISDC_SR_TY=$t python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b3_$t.json 2>/dev/null; python scripts/show.py gpurun_out/b3_$t.json | grep "==\|fine_def" >> gpurun_out/cmp.log; done
