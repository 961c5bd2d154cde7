#!/bin/bash
# What the driver runs at round end (one GPU): build, smoke, gpu tests, default bench, reference arm.
O=gpurun_out/driver; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/build.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
{ time python bench.py > $O/bench.json 2> $O/bench.err; } 2> $O/bench.time; echo "bench rc=$?" >> $O/bench.err
{ time python bench.py --impl reference > $O/ref.json 2> $O/ref.err; } 2> $O/ref.time; echo "ref rc=$?" >> $O/ref.err
