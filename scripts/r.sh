timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/par.log 2>&1
for sg in 0 1; do for c in 2 3 4; do ISDC_STEP_GRAPH=$sg python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b${c}_sg$sg.json 2>gpurun_out/b${c}_sg$sg.err; done; done
