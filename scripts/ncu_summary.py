"""Summarise ncu captures into profiles/ (committed evidence).

    python scripts/ncu_summary.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv \
        --tag r01_cfg3 [--workload cfg3_forced_heat2d_4095_M5]

Writes profiles/<tag>_kernels.txt (per-launch key metrics of the full capture),
profiles/<tag>_launches.txt (per-kernel totals/shares of the launch list) and, with --workload,
updates profiles/ncu_traffic.json with the fine-level smoother's DRAM traffic per launch.
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def to_bytes(v, unit):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--workload")
    ap.add_argument("--kernel-regex", default="k_smooth2")
    ap.add_argument("--cls", default="fine_defect_restrict", help="bench.py profile class of the kernel")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.rep:
        hdr, units, data = raw_rows(a.rep)
        idx = {k: hdr.index(k) for k in KEYS if k in hdr}
        ki = hdr.index("Kernel Name")
        lines = [f"# ncu --set full capture {os.path.basename(a.rep)}; one line per profiled launch"]
        traffic = None
        for r in data:
            name = r[ki]
            fields = []
            for k, i in idx.items():
                fields.append(f"{k}={r[i]} {units[i]}".strip())
            lines.append(name.split("(")[0] + " | " + " | ".join(fields))
            import re
            if a.workload and re.search(a.kernel_regex, name):
                rd = to_bytes(r[idx["dram__bytes_read.sum"]], units[idx["dram__bytes_read.sum"]])
                wr = to_bytes(r[idx["dram__bytes_write.sum"]], units[idx["dram__bytes_write.sum"]])
                grid = float(r[idx["launch__grid_size"]].replace(",", ""))
                if traffic is None or grid > traffic[1]:      # largest grid = the fine level
                    traffic = (rd + wr, grid, name.split("(")[0])
        with open(os.path.join(PROF, f"{a.tag}_kernels.txt"), "w") as f:
            f.write("\n".join(lines) + "\n")
        if a.workload and traffic:
            path = os.path.join(PROF, "ncu_traffic.json")
            d = json.load(open(path)) if os.path.exists(path) else {}
            d[a.workload] = {"class": a.cls, "dram_bytes_per_launch": traffic[0], "kernel": traffic[2],
                             "grid": traffic[1], "source": f"profiles/{a.tag}_kernels.txt (matching launch with the "
                                                           "largest grid = fine level)"}
            json.dump(d, open(path, "w"), indent=1)
    if a.launches:
        rows = list(csv.reader(open(a.launches)))
        hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        h = rows[hi]
        ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
        mi = h.index("Metric Name")
        agg = collections.defaultdict(lambda: [0, 0.0])
        for r in rows[hi + 1:]:
            if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
                continue
            v = float(r[vi].replace(",", ""))
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
            nm = r[ki].split("(")[0]
            agg[nm][0] += 1
            agg[nm][1] += v
        tot = sum(v[1] for v in agg.values())
        lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none launch list ({os.path.basename(a.launches)})",
                 "# cold-cache, serialised launches: compare SHARES, not absolute times",
                 f"# total {tot:.1f} us over {sum(v[0] for v in agg.values())} launches"]
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"{k:48s} launches={v[0]:6d} total_us={v[1]:12.1f} avg_us={v[1] / v[0]:10.2f} share={v[1] / tot:.3f}")
        with open(os.path.join(PROF, f"{a.tag}_launches.txt"), "w") as f:
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
