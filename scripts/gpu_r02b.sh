O=gpurun_out/r02b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
{ time timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > $O/ref.json 2> $O/ref.err; } 2> $O/ref.time
nproc > $O/nproc.txt; lscpu > $O/lscpu.txt 2>&1
timeout 900 bash scripts/ncu_classes.sh r02b 3 3000 400
