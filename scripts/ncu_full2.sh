# ncu --set full on selected kernels of one bench config.  Usage: bash scripts/ncu_full2.sh TAG CONFIG REGEX [SKIP] [COUNT]
TAG=$1; CFG=$2; RX=$3; SKIP=${4:-2}; CNT=${5:-1}
O=gpurun_out/$TAG; mkdir -p $O
B="python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --extra="
$B > $O/plain_$CFG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:$RX" -s $SKIP -c $CNT -o $O/prof_cfg$CFG $B > $O/ncu_$CFG.log 2>&1
echo "ncu rc=$?" >> $O/ncu_$CFG.log
