python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in 2 3 5; do
  python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b${c}_pdl1.json 2>&1
  ISDC_PDL=0 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b${c}_pdl0.json 2>&1
done
