#!/bin/bash
# Usage: bash scripts/launches.sh TAG CONFIG SKIP COUNT  -> gpurun_out/TAG_launches.csv (duration + grid per launch)
TAG=$1; CFG=$2; SKIP=${3:-1000}; CNT=${4:-400}
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none -s $SKIP -c $CNT --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_ncu.log
