#!/bin/bash
O=gpurun_out/r02q; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "execution_paths or steps_bitwise or vcycle or cfg5 or cfg4" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in 4 5; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --extra "" --pfasst 0 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
