python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "not cfg5" 2>&1 | tail -3 > gpurun_out/par.log
ISDC_RES_NMW=1 python -m pytest tests/test_gpu_fullsize.py -x -q -k "cfg3" 2>&1 | tail -2 >> gpurun_out/par.log
python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b3.json 2>gpurun_out/b3.err
ISDC_RES_NMW=1 python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b3_n1.json 2>gpurun_out/b3.err
