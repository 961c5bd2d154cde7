#!/bin/bash
# experiment: 8 TMA stages in the shifted ws smoother (ISDC_WS_NS8=1) vs 6
O=gpurun_out/r02ad; mkdir -p $O
for v in 0 1 0 1; do
  ISDC_WS_NS8=$v timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --extra "" --pfasst 0 >> $O/bench_ns8_$v.json 2>> $O/bench.err
done
ISDC_WS_NS8=1 timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "cfg5 or cfg4_seed0" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
