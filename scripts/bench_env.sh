# bench one config under several environment settings: bash scripts/bench_env.sh TAG CONFIG "ENV1" "ENV2" ...
TAG=$1; C=$2; shift 2
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
i=0
for E in "$@"; do
  env $E timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --extra "" > $O/bench_$i.json 2> $O/bench_$i.err
  echo "$i: $E rc=$?" >> $O/index.txt; i=$((i+1))
done
