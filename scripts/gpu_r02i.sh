#!/bin/bash
O=gpurun_out/r02i; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python -m pytest tests/test_gpu_pfasst.py tests/test_gpu_mlsdc.py -x -q > $O/pytest_pf.log 2>&1; echo "rc=$?" >> $O/pytest_pf.log
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --extra "" --pfasst 0 > $O/bench5.json 2> $O/bench5.err; echo "rc=$?" >> $O/bench5.err
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
