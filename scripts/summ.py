"""Summarise bench JSON lines: python scripts/summ.py file..."""
import json
import sys

for fn in sys.argv[1:]:
    try:
        d = json.loads(open(fn).read().strip().splitlines()[-1])
    except Exception as e:
        print(fn, "unreadable", e)
        continue
    print(f"{fn}: {d['config']['workload']} steps/s {d['value']:.3f} ms/step {d['ms_per_step']:.1f} "
          f"sweeps {d['sweeps_per_step']:.1f} vcyc/s {d['vcycles_per_s']:.0f} stepGB/s {d['step_alg_GBps']:.0f} "
          f"({d['step_alg_frac_of_peak']:.2f}) launches {d['gpu_launches']} conv {d['converged']}")
    r = d["roofline"]
    print(f"   roofline: {r['achieved']:.0f} GB/s frac {r['frac']:.3f} avg {r['avg_launch_ms']:.4f} ms share {r['share_of_step']:.3f}")
    tot = 0
    for k, v in d["kernels"].items():
        if k.startswith("_"):
            continue
        tot += v["share"]
        print(f"   {k:22s} share {v['share']:.3f} GB/s {v['alg_GBps'] or 0:7.0f} n {v['launches']}")
    print(f"   kernel share total {tot:.3f}; e2e {d['e2e']['value'] if d.get('e2e') else None}; clocks {d['clocks']}")
    if d.get("cpu_baseline"):
        print("   cpu", d["cpu_baseline"])
