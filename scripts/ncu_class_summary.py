"""Summarise a per-kernel ncu metric CSV (scripts/ncu_classes.sh) into a committed table.

    python scripts/ncu_class_summary.py gpurun_out/<tag>/ncu_cfg5.csv profiles/<name>.txt "<title>"

Groups launches by (kernel, grid) -- the grid tells the multigrid level apart -- and reports per
group: launches, mean duration, DRAM bytes read / written per launch, DRAM throughput %, warps
active %, issue active %, L1/LSU %, shared-memory wavefronts, L2 hit %, fp64 pipe %, registers.
"""
import collections
import csv
import sys

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


def main(path, out, title):
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


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
