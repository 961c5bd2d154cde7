"""Print the key numbers of bench JSON lines: python scripts/show.py file..."""
import json, sys
for fn in sys.argv[1:]:
    try:
        d = json.loads(open(fn).read().strip().splitlines()[-1])
    except Exception as e:
        print(fn, "unreadable", e); continue
    print(f"== {fn}: {d['config']['workload']} value={d['value']:.4g} {d['unit']} ms/step={d['ms_per_step']:.2f} "
          f"sweeps={d.get('sweeps_per_step')} step_alg={d.get('step_alg_GBps', 0):.0f} GB/s "
          f"({d.get('step_alg_frac_of_peak', 0):.3f}) launches={d.get('gpu_launches')} clocks={d.get('clocks', {}).get('sm_mhz')} {d.get('clocks', {}).get('reasons')}")
    r = d["roofline"]
    print(f"   roofline {r.get('kernel')}: achieved={r['achieved']:.0f} frac={r['frac']:.3f} avg_ms={r['avg_launch_ms']:.4f} share={r['share_of_step']:.3f}")
    for k, v in d.get("kernels", {}).items():
        if k.startswith("_"): continue
        print(f"   {k:22s} ms={v['ms']:9.2f} n={v['launches']:6d} alg_GBps={v['alg_GBps'] or 0:8.0f} share={v['share']:.3f}")
    if d.get("e2e"): print("   e2e", d["e2e"]["value"])
