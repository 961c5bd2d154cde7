python bench.py --config 3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/pf_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_smooth2" -s 60 -c 2 -o gpurun_out/pf2d python bench.py --config 3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/pf2d_ncu.log 2>&1
