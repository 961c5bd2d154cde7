#!/bin/bash
# bench lines of every config (round-2 DESIGN §10 table) + the execution-path tests after the knob cleanup
O=gpurun_out/r02j; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_burgers.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in 1 2 3 4 5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --extra "" --pfasst 0 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
for c in 1 3; do
  timeout 600 python bench.py --config $c --mode sdc --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --extra "" --pfasst 0 > $O/bench_cfg${c}_sdc.json 2> $O/bench_cfg${c}_sdc.err
done
