#!/bin/bash
# shifted 3D tiling: parity (reduced + full size) and cfg4 / cfg5 bench with and without it
O=gpurun_out/r02x; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_mlsdc.py -x -q -k "3d or cfg4 or cfg5 or execution or 3D or mlsdc" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in 5 4; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --extra "" --pfasst 0 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
  ISDC_SHIFT3D=0 timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --extra "" --pfasst 0 > $O/bench_cfg${c}_old.json 2> $O/bench_cfg${c}_old.err
done
