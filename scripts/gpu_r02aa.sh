#!/bin/bash
# end-of-round evidence: full ncu captures (cfg5: ws smoother, RHS, residual, restriction) exported
# to CSV on the box, per-kernel metrics and the launch list of cfg3 at HEAD
O=gpurun_out/r02aa; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
B="python bench.py --config 5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --extra= --pfasst 0"
$B > $O/plain5.log 2>&1
for K in k_smooth2ws k_resid4 k_restrict k_bl k_prolong; do
  ncu --set full --clock-control none --import-source on -k "regex:$K" -s 0 -c 1 -o $O/full_$K $B > $O/ncu_$K.log 2>&1
  ncu -i $O/full_$K.ncu-rep --page details --csv > $O/full_$K.details.csv 2>/dev/null
  ncu -i $O/full_$K.ncu-rep --page raw --csv > $O/full_$K.raw.csv 2>/dev/null
  ncu -i $O/full_$K.ncu-rep --page source --csv > $O/full_$K.source.csv 2>/dev/null
done
bash scripts/ncu_classes.sh r02aa 3 3000 400 --extra= --pfasst 0
B3="python bench.py --config 3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --extra= --pfasst 0"
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -s 3000 -c 600 --csv --log-file $O/cfg3_launches.csv $B3 > $O/ncu3.log 2>&1
find gpurun_out -name "*.ncu-rep" -size +8M -delete
du -sh gpurun_out/* > $O/du.txt
[ $(du -sm gpurun_out | cut -f1) -gt 55 ] && rm -f $O/*.source.csv; du -sh gpurun_out >> $O/du.txt
