#!/bin/bash
# Usage: bash scripts/ncu_one.sh TAG CONFIG KERNEL_REGEX SKIP [COUNT]  -> gpurun_out/TAG.ncu-rep (full set)
TAG=$1; CFG=$2; KR=$3; SKIP=${4:-3}; CNT=${5:-1}
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$KR" -s $SKIP -c $CNT -o gpurun_out/$TAG $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_ncu.log
