"""Per-kernel/grid totals of an ncu launch list: python scripts/launch_table.py file.csv"""
import csv, collections, sys, io
rows = list(csv.reader(io.StringIO(open(sys.argv[1]).read().split('\n', 0)[0])))
hdr = None; data = collections.defaultdict(dict)
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if not hdr or len(r) != len(hdr): continue
    d = dict(zip(hdr, r))
    key = d["ID"]
    data[key]["name"] = d["Kernel Name"].split("(")[0]
    try: data[key][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    except ValueError: pass
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for k, v in data.items():
    g = v.get("launch__grid_size", 0); t = v.get("gpu__time_duration.sum", 0) / 1e3
    nm = (v["name"][:40], int(g))
    agg[nm][0] += 1; agg[nm][1] += t; tot += t
print(f"total {tot:.1f} us over {len(data)} launches")
for (nm, g), (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{nm:42s} grid={g:7d} n={c:4d} total={t:9.1f}us avg={t/c:8.2f}us share={t/tot:.3f}")
