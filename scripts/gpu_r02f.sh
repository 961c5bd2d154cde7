#!/bin/bash
# PFASST GPU parity + per-kernel ncu metrics (cfg5, cfg3) + one full capture each of the fine 3D
# smoother and the 3D residual, exported to CSV on the box (the .ncu-rep files stay small)
O=gpurun_out/r02f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_pfasst.py tests/test_gpu_mlsdc.py -x -q > $O/pytest_pfasst.log 2>&1; echo "rc=$?" >> $O/pytest_pfasst.log
bash scripts/ncu_classes.sh r02f 5 2500 400 --extra=
bash scripts/ncu_classes.sh r02f 3 3000 400 --extra=
B="python bench.py --config 5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --extra="
for K in k_smooth2ws k_resid4 k_restrict k_bl; do
  ncu --set full --clock-control none --import-source on -k "regex:$K" -s 0 -c 1 -o $O/full_$K $B > $O/ncu_$K.log 2>&1
  ncu -i $O/full_$K.ncu-rep --page details --csv > $O/full_$K.details.csv 2>/dev/null
  ncu -i $O/full_$K.ncu-rep --page raw --csv > $O/full_$K.raw.csv 2>/dev/null
  ncu -i $O/full_$K.ncu-rep --page source --csv > $O/full_$K.source.csv 2>/dev/null
done
find gpurun_out -name "*.ncu-rep" -size +8M -delete
du -sh gpurun_out/* > $O/du.txt
[ $(du -sm gpurun_out | cut -f1) -gt 55 ] && rm -f $O/*.source.csv $O/*.raw.csv; du -sh gpurun_out >> $O/du.txt
