#!/bin/bash
# per-kernel ncu metrics of the current kernels (cfg5, cfg3) + full captures of the 3D smoother and residual
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash scripts/ncu_classes.sh r02e 5 2500 400 --extra=
bash scripts/ncu_classes.sh r02e 3 3000 400 --extra=
O=gpurun_out/r02e
B="python bench.py --config 5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --extra="
ncu --set full --clock-control none --import-source on -k "regex:k_smooth2ws" -s 0 -c 9 -o $O/prof_ws $B > $O/ncu_ws.log 2>&1; echo "rc=$?" >> $O/ncu_ws.log
ncu --set full --clock-control none --import-source on -k "regex:k_resid4" -s 0 -c 1 -o $O/prof_r4 $B > $O/ncu_r4.log 2>&1; echo "rc=$?" >> $O/ncu_r4.log
