bash scripts/ncu_one.sh p3d_smooth5 5 "k_smooth2" 10 1
ncu --set full --clock-control none --import-source on -k regex:"k_bl" -s 4 -c 1 -o gpurun_out/p3d_bl5 python bench.py --config 5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/p3d_bl5_ncu.log 2>&1
