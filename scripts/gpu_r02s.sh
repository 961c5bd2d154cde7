#!/bin/bash
O=gpurun_out/r02s; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_table1.py tests/test_gpu_mlsdc.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for E in "ISDC_RHS128=1" "ISDC_RHS128=0"; do
  env $E timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --extra "" --pfasst 0 > $O/bench_cfg3_$E.json 2> $O/bench_cfg3_$E.err
done
B="python bench.py --config 3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --extra= --pfasst 0"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_rhs -c 6 --csv --log-file $O/rhs.csv $B > $O/ncu.log 2>&1
ISDC_RHS128=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_rhs -c 6 --csv --log-file $O/rhs0.csv $B > $O/ncu0.log 2>&1
