set -x
O=gpurun_out/r02a; mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 900 bash scripts/ncu_classes.sh r02a 5 2500 400
