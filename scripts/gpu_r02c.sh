set -x
O=gpurun_out/r02c; mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python -m pytest tests/test_gpu_mlsdc.py -q -x > $O/pytest_mlsdc.log 2>&1; echo "rc=$?" >> $O/pytest_mlsdc.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 2400 python -m pytest tests -m gpu -q --durations=20 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
