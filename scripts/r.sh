timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/par.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for sg in 0 1; do ISDC_STEP_GRAPH=$sg python bench.py --config 1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/b1_sg$sg.json 2>/dev/null; done
