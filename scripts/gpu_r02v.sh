#!/bin/bash
O=gpurun_out/r02v; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in 3 4 5; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --extra "" --pfasst 0 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
B="python bench.py --config 3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --extra= --pfasst 0"
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:k_smooth2r -c 14 --csv --log-file $O/sr.csv $B > $O/ncu.log 2>&1
