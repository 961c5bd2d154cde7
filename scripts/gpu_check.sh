#!/bin/bash
# One gpurun call: gpu tests, bench lines, launch list. Usage: bash scripts/gpu_check.sh TAG [configs...]
TAG=${1:-run}; shift
CFGS=${@:-3}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for c in $CFGS; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
