python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python scripts/dbg_fuse.py > gpurun_out/dbg_fuse.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pt_sr.log 2>&1
for c in 3 2; do
  python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b${c}_sr1.json 2>&1
  ISDC_SR_STREAM=0 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b${c}_sr0.json 2>&1
done
