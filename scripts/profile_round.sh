#!/bin/bash
# Round evidence: launch lists + one ncu --set full capture of the dominant fine-level kernel for
# config 3 (2D; PART=3) and config 5 (3D; PART=5).  Each ncu run follows the same command exiting
# 0 without ncu.  Outputs in gpurun_out/prof_<tag>*.  Run the parts in separate gpurun calls
# (each .ncu-rep is ~30 MB; gpurun copies back at most 64 MiB).
TAG=${1:-r01}
PART=${2:-3}
if [ "$PART" = 3 ]; then
B3="python bench.py --config 3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$B3 > gpurun_out/prof_${TAG}_cfg3_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 400 --csv --log-file gpurun_out/prof_${TAG}_cfg3_launches.csv $B3 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_smooth2r<.int.0," -s 2 -c 1 -o gpurun_out/prof_${TAG}_cfg3 $B3 > gpurun_out/prof_${TAG}_cfg3_ncu.log 2>&1
echo "cfg3 rc=$?" >> gpurun_out/prof_${TAG}_rc.log
else
B5="python bench.py --config 5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$B5 > gpurun_out/prof_${TAG}_cfg5_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv --log-file gpurun_out/prof_${TAG}_cfg5_launches.csv $B5 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_smooth2 -s 10 -c 1 -o gpurun_out/prof_${TAG}_cfg5 $B5 > gpurun_out/prof_${TAG}_cfg5_ncu.log 2>&1
echo "cfg5 rc=$?" >> gpurun_out/prof_${TAG}_rc.log
fi
