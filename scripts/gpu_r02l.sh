#!/bin/bash
O=gpurun_out/r02l; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python scripts/residual_kinds.py > $O/residual_kinds.log 2>&1; echo "rc=$?" >> $O/residual_kinds.log
cp profiles/residual_kinds_r02.md $O/ 2>/dev/null
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
