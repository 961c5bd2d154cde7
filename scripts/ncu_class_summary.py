"""Summarise a per-kernel ncu metric CSV (scripts/ncu_classes.sh) into a committed table.

    python scripts/ncu_class_summary.py gpurun_out/<tag>/ncu_cfg5.csv profiles/<name>.txt "<title>" [WORKLOAD]

With WORKLOAD (e.g. cfg5_advdiff3d_511_M5) it also records, in profiles/ncu_traffic.json, the DRAM
bytes per launch of each kernel class's fine-level launch (bench.py's roofline "traffic").

Groups launches by (kernel, grid) -- the grid tells the multigrid level apart -- and reports per
group: launches, mean duration, DRAM bytes read / written per launch, DRAM throughput %, warps
active %, issue active %, L1/LSU %, shared-memory wavefronts, L2 hit %, fp64 pipe %, registers.
"""
import collections
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# bench.py kernel classes -> kernel-name patterns (the fine level is the launch with the largest grid)
CLASS_PATTERNS = {
    "fine_smoother": [r"f3d::k_smooth2<\d+, 0,", r"f3d::k_smooth2ws<0[,>]"],
    "fine_defect_restrict": [r"f3d::k_restrict", r"f2d::k_smooth2r<0,"],
    "fine_prolong_correct": [r"f3d::k_prolong", r"f2d::k_smooth2<false, 2,", r"f2d::k_smooth2<0, 2,"],
    "residual": [r"k_resid", r"f3d::k_bl<\d+, 1,"],
    "rhs": [r"k_rhs", r"f3d::k_bl<\d+, [02],"],
}

SHORT = {
    "gpu__time_duration.sum": "us",
    "dram__bytes_read.sum": "rdMB",
    "dram__bytes_write.sum": "wrMB",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps%",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1%",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "shwfM",
    "lts__t_sector_hit_rate.pct": "l2hit%",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64%",
    "launch__registers_per_thread": "regs",
}
SCALE = {"gpu__time_duration.sum": 1e-3, "dram__bytes_read.sum": 1e-6, "dram__bytes_write.sum": 1e-6,
         "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": 1e-6}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "usecond": 1e3,
        "nsecond": 1, "msecond": 1e6}


def short_name(k):
    k = k.split("(")[0] if "<" not in k.split("(")[0] else k[: k.index(">") + 1]
    return k.replace("void ", "")


def grid_size(g):
    v = 1
    for x in re.findall(r"\d+", g):
        v *= int(x)
    return v


def main(path, out, title, workload=None):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    hdr, rows = rows[0], rows[1:]
    ix = {h: i for i, h in enumerate(hdr)}
    per = collections.defaultdict(dict)
    for r in rows:
        key = (r[ix["ID"]], short_name(r[ix["Kernel Name"]]), r[ix["Grid Size"]], r[ix["Block Size"]])
        v = r[ix["Metric Value"]].replace(",", "")
        try:
            v = float(v) * UNIT.get(r[ix["Metric Unit"]], 1)
        except ValueError:
            continue
        per[key][r[ix["Metric Name"]]] = v
    groups = collections.OrderedDict()
    for (lid, name, grid, blk), m in per.items():
        groups.setdefault((name, grid, blk), []).append(m)
    tot = sum(sum(m.get("gpu__time_duration.sum", 0) for m in ms) for ms in groups.values())
    lines = [f"# {title}", f"# source: {path}; {len(per)} launches, total {tot / 1e3:.1f} us (cold-cache, serialised)",
             "# per launch means; rdMB/wrMB = DRAM bytes per launch; shwfM = shared-memory LSU wavefronts (millions)"]
    cols = list(SHORT)
    lines.append("%-34s %-14s %5s %6s " % ("kernel", "grid", "n", "share") + " ".join("%8s" % SHORT[c] for c in cols))
    for (name, grid, blk), ms in sorted(groups.items(), key=lambda kv: -sum(m.get("gpu__time_duration.sum", 0) for m in kv[1])):
        share = sum(m.get("gpu__time_duration.sum", 0) for m in ms) / tot
        vals = []
        for c in cols:
            xs = [m[c] for m in ms if c in m]
            v = sum(xs) / len(xs) if xs else float("nan")
            v *= SCALE.get(c, 1)
            vals.append("%8.1f" % v if abs(v) < 1e5 else "%8.3g" % v)
        lines.append("%-34s %-14s %5d %6.3f " % (name[:34], grid, len(ms), share) + " ".join(vals))
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if workload:
        tj = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        db = json.load(open(tj)) if os.path.exists(tj) else {}
        ent = {}
        for cls, pats in CLASS_PATTERNS.items():
            # the fine-level launch of a class is the (kernel, grid) group with the largest total time
            # (grid sizes mix tiles and z chunks; a one-off launch such as the first sweep's RHS from
            # the node fields is not the class's representative)
            cand = [(sum(m.get("gpu__time_duration.sum", 0) for m in ms), name, grid, ms)
                    for (name, grid, blk), ms in groups.items() if any(re.search(p, name) for p in pats)]
            if not cand:
                continue
            gsz, name, grid, ms = max(cand)
            rd = sum(m.get("dram__bytes_read.sum", 0) for m in ms) / len(ms)
            wr = sum(m.get("dram__bytes_write.sum", 0) for m in ms) / len(ms)
            ent[cls] = {"kernel": name, "grid": grid, "dram_bytes_per_launch": rd + wr, "dram_read": rd,
                        "dram_write": wr, "source": f"{os.path.relpath(out, ROOT)} (the class's (kernel, grid) group with the largest total time = fine level)"}
        db[workload] = ent
        json.dump(db, open(tj, "w"), indent=1)
        print("traffic ->", tj, list(ent))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "", sys.argv[4] if len(sys.argv) > 4 else None)
