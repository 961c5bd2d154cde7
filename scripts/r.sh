python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ISDC_RHS16=1 timeout 900 python -m pytest tests -m gpu -q -x -k "rhs or sweep or steps or fullsize" > gpurun_out/pt16.log 2>&1
for c in 5 4; do
ISDC_RHS16=1 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b${c}_rhs16.json 2>&1
python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b${c}_rhs8.json 2>&1
done
