#!/bin/bash
# TMA stages of the shifted ws smoother: 8 (default) vs 10 vs 6; then the whole GPU suite and the default bench
O=gpurun_out/r02ae; mkdir -p $O
for v in 8 10 6 10 8; do
  ISDC_WS_NS=$v timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --extra "" --pfasst 0 >> $O/bench_ns_$v.json 2>> $O/bench.err
done
( time timeout 1200 python -m pytest tests -m gpu -x -q ) > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
( time python bench.py ) > $O/bench_default.json 2> $O/bench_default.err
