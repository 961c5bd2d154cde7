ISDC_BL_NM4=1 python -m pytest tests/test_gpu_fullsize.py -x -q -k "cfg5" 2>&1 | tail -2 > gpurun_out/par.log
ISDC_BL_NM4=1 python bench.py --config 5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b5_nm4.json 2>gpurun_out/b5.err
python bench.py --config 5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b5.json 2>>gpurun_out/b5.err
