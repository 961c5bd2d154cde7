#!/bin/bash
# final profile refresh at HEAD (8-stage shifted smoother): cfg5 launch list + per-kernel ncu metrics
O=gpurun_out/r02af; mkdir -p $O
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --extra= --pfasst 0"
$B > $O/plain.log 2>&1
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -s 3000 -c 600 --csv --log-file $O/cfg5_launches.csv $B > $O/ncu.log 2>&1
bash scripts/ncu_classes.sh r02af 5 3000 300 --extra= --pfasst 0
