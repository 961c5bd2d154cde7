python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_table1.py -x -q -k "not cfg5" 2>&1 | tail -2 > gpurun_out/par.log
python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b3.json 2>/dev/null
python bench.py --config 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b2.json 2>/dev/null
