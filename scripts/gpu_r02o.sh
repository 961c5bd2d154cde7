#!/bin/bash
O=gpurun_out/r02o; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for C in 3 5; do
  B="python bench.py --config $C --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --extra= --pfasst 0"
  ncu --set full --clock-control none --import-source on -k "regex:k_ctail" -s 5 -c 1 -o $O/full_c${C}_ctail $B > $O/ncu_c${C}.log 2>&1
  ncu -i $O/full_c${C}_ctail.ncu-rep --page raw --csv > $O/full_c${C}_ctail.raw.csv 2>/dev/null
  ncu -i $O/full_c${C}_ctail.ncu-rep --page source --csv > $O/full_c${C}_ctail.source.csv 2>/dev/null
  ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -s 3000 -c 200 --csv --log-file $O/launches_c$C.csv $B > $O/ncu_l$C.log 2>&1
done
find gpurun_out -name "*.ncu-rep" -size +8M -delete
