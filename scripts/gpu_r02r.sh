#!/bin/bash
O=gpurun_out/r02r; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "steps_bitwise or cfg5 or residual or rhs" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --extra "" --pfasst 0 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
B="python bench.py --config 5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --extra= --pfasst 0"
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:k_resid4 -c 3 --csv --log-file $O/r4.csv $B > $O/ncu.log 2>&1
