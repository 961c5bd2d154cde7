rm -f gpurun_out/cmp.log
for y in 0 32 128 256; do ISDC_STREAM_YC=$y python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b3_$y.json 2>/dev/null; echo "YC $y" >> gpurun_out/cmp.log; python scripts/show.py gpurun_out/b3_$y.json | grep "==\|rhs\|resid" >> gpurun_out/cmp.log; done
