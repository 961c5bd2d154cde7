python -m pytest tests/test_gpu_fullsize.py -x -q -k "cfg3 or cfg2" 2>&1 | tail -2 > gpurun_out/par.log
python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b3.json 2>/dev/null
