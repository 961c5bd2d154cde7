#!/bin/bash
# ISDC vs SDC on configs 1 and 3 (north star: "reporting both the throughput and the total V-cycle
# count per step"); one bench line each -> gpurun_out/ivs/*.json -> profiles/isdc_vs_sdc_<tag>.md
TAG=${1:-r01}; O=gpurun_out/ivs; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in 1 3; do for m in isdc sdc; do
  python bench.py --config $c --mode $m --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/cfg${c}_$m.json 2> $O/cfg${c}_$m.err
done; done
python - <<PY
import json, glob, os
rows = []
for c in (1, 3):
    r = {}
    for m in ("isdc", "sdc"):
        d = json.loads(open(f"$O/cfg{c}_{m}.json").read().strip().splitlines()[-1])
        r[m] = d
    rows.append((c, r))
out = ["# ISDC vs SDC on one B200 (bench.py, 3 timed steps)", "",
       "| cfg | mode | sweeps/step | V-cycles/step | ms/step | steps/s | V-cycles/s |", "|---|---|---|---|---|---|---|"]
for c, r in rows:
    for m in ("isdc", "sdc"):
        d = r[m]
        out.append(f"| {c} | {m.upper()} | {d['sweeps_per_step']:.0f} | {d['vcycles_per_step']:.0f} | {d['ms_per_step']:.2f} | "
                   f"{d['value']:.4g} | {d['vcycles_per_s']:.4g} |")
    s, i = r["sdc"], r["isdc"]
    out.append(f"| {c} | ISDC saves | | {100*(1-i['vcycles_per_step']/s['vcycles_per_step']):.0f}% of the V-cycles | "
               f"{s['ms_per_step']/i['ms_per_step']:.2f}x faster per step | | |")
open("$O/isdc_vs_sdc_$TAG.md", "w").write("\n".join(out) + "\n")   # copy to profiles/ after the call
print("\n".join(out))
PY
