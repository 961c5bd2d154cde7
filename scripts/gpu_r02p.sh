#!/bin/bash
O=gpurun_out/r02p; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "execution_paths or steps_bitwise or vcycle" > $O/pytest_parity.log 2>&1; echo "rc=$?" >> $O/pytest_parity.log
for c in 1 3 4 5; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --extra "" --pfasst 0 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
for c in 4 5; do
  ISDC_CTAIL=0 timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --extra "" --pfasst 0 > $O/bench_cfg${c}_noct.json 2> $O/bench_cfg${c}_noct.err
done
