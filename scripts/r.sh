bash scripts/gpu_quick.sh r01f "-m gpu -k 'vcycle or sweep or fullsize'" 4 5
ISDC_SMOOTH3D_ROWS=4 python bench.py --config 5 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r01f/bench_cfg5_r4.json 2>&1
