"""Summarise an ncu --set full report (raw page): one line per launch with the metrics we track.
    python scripts/ncu_rep.py REPORT.ncu-rep"""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
want = [("Kernel Name", "kernel"), ("launch__grid_size", "grid"), ("launch__registers_per_thread", "regs"),
        ("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "rdMB"), ("dram__bytes_write.sum", "wrMB"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shwf"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%")]
idx = [(hdr.index(k) if k in hdr else None, n) for k, n in want]
units = rows[1]
print(" | ".join(n for _, n in idx))
for r in rows[2:]:
    vals = []
    for i, n in idx:
        if i is None:
            vals.append("-"); continue
        v = r[i]
        if n == "kernel":
            v = v.split("(")[0][-40:]
        elif n in ("rdMB", "wrMB"):
            f = float(v); u = units[i]
            f *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(u, 1)
            v = f"{f:.1f}"
        elif n == "us":
            f = float(v); u = units[i]
            f *= {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(u, 1)
            v = f"{f:.1f}"
        vals.append(v)
    print(" | ".join(vals))
