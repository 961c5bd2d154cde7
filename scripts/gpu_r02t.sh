#!/bin/bash
O=gpurun_out/r02t; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
B="python bench.py --config 3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --extra= --pfasst 0"
for D in 1 2 4 8; do
ISDC_RHS128_DIV=$D ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_rhs_f2 -c 4 --csv --log-file $O/rhs_d$D.csv $B > $O/ncu_d$D.log 2>&1
done
