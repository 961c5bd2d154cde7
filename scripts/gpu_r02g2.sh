#!/bin/bash
# config-5 golden, part 2 of 2: resume from the checkpoint after step 3 (same box only) through step 5
O=gpurun_out/r02g2; mkdir -p $O
hostname > $O/host.txt
ls -la /tmp/isdc_golden_ckpt > $O/ckpt.txt 2>&1
if [ -f /tmp/isdc_golden_ckpt/full_cfg5_seed0_isdc.json ]; then
  ( time python scripts/oracle_golden.py 5:0:isdc:5 ) > $O/golden.log 2>&1; echo "rc=$?" >> $O/golden.log
  cp -f tests/golden/full_cfg5_seed0_isdc.json $O/
  timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k cfg5 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
fi
