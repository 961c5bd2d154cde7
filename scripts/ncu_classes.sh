#!/bin/bash
# Per-kernel ncu metrics (DRAM bytes, warps active, issue active, LSU / L1, L2 hit rate, fp64 pipe,
# registers) for every kernel of a window of launches of one bench config, as CSV.  The plain run
# of the same command exits 0 first (B200_PROFILING.md).
#   bash scripts/ncu_classes.sh TAG CONFIG SKIP COUNT [extra bench args]
TAG=${1:-r02}; CFG=${2:-5}; SKIP=${3:-3000}; COUNT=${4:-300}; shift 4
O=gpurun_out/$TAG; mkdir -p $O
B="python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu-baseline $@"
MET=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,lts__t_sector_hit_rate.pct,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__block_size
$B > $O/plain_cfg$CFG.log 2>&1 && \
ncu --metrics $MET --clock-control none -s $SKIP -c $COUNT --csv --log-file $O/ncu_cfg${CFG}.csv $B > $O/ncu_cfg${CFG}.log 2>&1
echo "cfg$CFG ncu rc=$?" >> $O/rc.log
