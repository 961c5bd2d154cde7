ISDC_SM_TY=40 python -m pytest tests/test_gpu_fullsize.py -x -q -k "cfg3" 2>&1 | tail -2 > gpurun_out/par.log
rm -f gpurun_out/cmp.log
for t in 24 32 40 24 32 40; do ISDC_SM_TY=$t python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b3_$t.json 2>/dev/null; echo "TY $t" >> gpurun_out/cmp.log; python scripts/show.py gpurun_out/b3_$t.json | grep "==\|fine_pro" >> gpurun_out/cmp.log; done
