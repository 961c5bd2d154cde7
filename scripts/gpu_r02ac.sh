#!/bin/bash
# final verification of round 2: whole GPU suite, both bench arms, cfg4 bench, cfg5 launch list and
# per-kernel ncu metrics (restriction with the de-interleaved defect plane, CD4 f^E with the z ring)
O=gpurun_out/r02ac; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
( time python bench.py ) > $O/bench_default.json 2> $O/bench_default.err
( time python bench.py --impl reference ) > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --extra "" --pfasst 0 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --extra= --pfasst 0"
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -s 3000 -c 600 --csv --log-file $O/cfg5_launches.csv $B > $O/ncu.log 2>&1
bash scripts/ncu_classes.sh r02ac 5 3000 300 --extra= --pfasst 0
