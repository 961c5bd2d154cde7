#!/bin/bash
# full ncu captures of the 2D kernels (cfg3) and the tails, exported to CSV on the box
O=gpurun_out/r02m; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for C in 3 5; do
  B="python bench.py --config $C --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --extra= --pfasst 0"
  if [ $C = 3 ]; then KS="k_smooth2r k_resid_t k_tail k_rhs_s"; else KS="k_tail"; fi
  for K in $KS; do
    ncu --set full --clock-control none --import-source on -k "regex:$K" -s 2 -c 1 -o $O/full_c${C}_$K $B > $O/ncu_c${C}_$K.log 2>&1
    ncu -i $O/full_c${C}_$K.ncu-rep --page raw --csv > $O/full_c${C}_$K.raw.csv 2>/dev/null
    ncu -i $O/full_c${C}_$K.ncu-rep --page source --csv > $O/full_c${C}_$K.source.csv 2>/dev/null
  done
done
find gpurun_out -name "*.ncu-rep" -size +8M -delete
[ $(du -sm gpurun_out | cut -f1) -gt 55 ] && rm -f $O/*.source.csv
du -sh gpurun_out > $O/du.txt
