#!/bin/bash
# ws smoother TMA depth experiment (cfg5) + the default bench with the PFASST extra
O=gpurun_out/r02g; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
i=0
for E in "ISDC_WS_NS=6" "ISDC_WS_NS=8" "ISDC_WS_NS=10"; do
  env $E timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --extra "" --pfasst 0 > $O/bench_$i.json 2> $O/bench_$i.err
  echo "$i: $E rc=$?" >> $O/index.txt; i=$((i+1))
done
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_default.json 2> $O/bench_default.err; echo "rc=$?" >> $O/bench_default.err
