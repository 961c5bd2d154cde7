#!/bin/bash
# Usage: bash scripts/gpu_quick.sh TAG "pytest-args" configs...   (build, gpu tests, bench lines)
TAG=${1:-run}; PT=${2:-"-m gpu"}; shift; shift
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
if [ "$PT" != "none" ]; then eval timeout 1500 python -m pytest tests $PT -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; fi
for c in "$@"; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
