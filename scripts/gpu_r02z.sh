#!/bin/bash
# Full-size oracle golden of config 5 (511^3, 5 steps) on the GPU box's host cores: the committed
# writer scripts/oracle_golden.py, which calls only oracle/ and synth/ (no CUDA path).  The golden
# JSON is rewritten after every finished step and copied to gpurun_out/ as it appears.
O=gpurun_out/r02z; mkdir -p $O
nproc > $O/nproc.txt
python -c "import oracle; print(oracle.num_threads())" > $O/threads.txt 2>&1
( while true; do cp -f tests/golden/full_cfg5_seed0_isdc.json $O/ 2>/dev/null; sleep 20; done ) &
CP=$!
( time python scripts/oracle_golden.py 5:0:isdc:5 ) > $O/golden.log 2>&1; echo "rc=$?" >> $O/golden.log
kill $CP
cp -f tests/golden/full_cfg5_seed0_isdc.json $O/
# the CUDA path against the new golden (all five steps)
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k cfg5 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
