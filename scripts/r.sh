for r in 2 3 4; do ISDC_SMOOTH3D_ROWS=$r python bench.py --config 5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b5_r$r.json 2>/dev/null; done
