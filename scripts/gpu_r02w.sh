#!/bin/bash
# HEAD verification: whole GPU suite, the driver's default bench line, both arms, and the launch list
O=gpurun_out/r02w; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
( time python bench.py ) > $O/bench_default.json 2> $O/bench_default.err
( time python bench.py --impl reference ) > $O/bench_reference.json 2> $O/bench_reference.err
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --extra= --pfasst 0"
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 600 --csv --log-file $O/cfg5_launches.csv $B > $O/ncu.log 2>&1
