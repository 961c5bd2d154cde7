#!/bin/bash
# config-5 golden, part 1 of 2: steps 1-3 (the writer checkpoints after every step under
# /tmp/isdc_golden_ckpt; part 2 resumes there if the next call lands on the same box)
O=gpurun_out/r02g1; mkdir -p $O
rm -rf /tmp/isdc_golden_ckpt
( time python scripts/oracle_golden.py 5:0:isdc:3 ) > $O/golden.log 2>&1; echo "rc=$?" >> $O/golden.log
cp -f tests/golden/full_cfg5_seed0_isdc.json $O/
ls -la /tmp/isdc_golden_ckpt > $O/ckpt.txt 2>&1
hostname > $O/host.txt
