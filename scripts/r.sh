rm -f gpurun_out/cmp.log
for m in 2047 1023 2047 1023; do ISDC_SR_TY32_MIN=$m python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b3_$m.json 2>/dev/null; echo "MIN $m" >> gpurun_out/cmp.log; python scripts/show.py gpurun_out/b3_$m.json | grep "==\|coarse" >> gpurun_out/cmp.log; done
