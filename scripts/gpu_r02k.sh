#!/bin/bash
O=gpurun_out/r02k; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
OMP_NUM_THREADS=4 timeout 900 python -m pytest tests/test_gpu_pfasst.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
