# quick GPU check: build, selected GPU tests, one bench config.  Usage: bash scripts/gpu_quick2.sh TAG [pytest -k expr] [config]
TAG=${1:-q}; K=${2:-"mlsdc or fullsize_against_oracle_golden[full_cfg5 or steps_bitwise or execution_paths"}; C=${3:-5}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "$K" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --extra "" > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
