ISDC_SM_TY32_MIN=2047 ISDC_SM_TY=24 python -m pytest tests/test_gpu_fullsize.py -x -q -k "cfg3" 2>&1 | tail -2 > gpurun_out/par.log
ISDC_SM_TY32_MIN=2047 ISDC_SM_TY=24 python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b3_24.json 2>/dev/null
python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b3_16.json 2>/dev/null
