"""Summarise `ncu --set full` captures exported as CSV (raw / source pages; scripts/gpu_r02f.sh) into a
committed text file: duration, DRAM bytes, occupancy, issue, pipes, stall reasons, stall samples by opcode.

    python scripts/ncu_full_summary.py OUT.txt "title" gpurun_out/<tag>/full_<kernel> [...]
"""
import collections
import csv
import sys


def summary(prefix):
    out = []
    rows = list(csv.reader(open(prefix + ".raw.csv")))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    un = dict(zip(hdr, units))
    out.append(f"\n## {d.get('Kernel Name', '')[:100]}")
    out.append(f"  grid {d.get('launch__grid_size')} block {d.get('launch__block_size')} "
               f"regs {d.get('launch__registers_per_thread')}")
    keys = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
            ("dram__bytes_write.sum", "DRAM write"),
            ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput"),
            ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active"),
            ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active"),
            ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe"),
            ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/LSU"),
            ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
            ("lts__t_sector_hit_rate.pct", "L2 hit"), ("smsp__inst_executed.sum", "warp instructions")]
    for k, lab in keys:
        if k in d:
            out.append(f"  {lab:20s} {d[k]} {un.get(k, '')}")
    st = [(h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(v))
          for h, v in d.items() if h.startswith("smsp__average_warps_issue_stalled_")
          and h.endswith("_per_issue_active.ratio") and v]
    st.sort(key=lambda x: -x[1])
    out.append("  stalls (warps per issue): " + ", ".join(f"{a} {b:.2f}" for a, b in st[:8]))
    try:
        rows = list(csv.reader(open(prefix + ".source.csv")))
        ix = {h: i for i, h in enumerate(rows[1])}
        data = rows[2:]
        col = "Warp Stall Sampling (All Samples)"
        tot = sum(int(r[ix[col]] or 0) for r in data) or 1
        byop, cnt = collections.Counter(), collections.Counter()
        for r in data:
            t = r[ix["Source"]].split()
            if not t:
                continue
            op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            byop[op] += int(r[ix[col]] or 0)
            cnt[op] += int(r[ix["Instructions Executed"]] or 0)
        out.append("  stall samples by opcode: " + ", ".join(
            f"{op} {100 * v / tot:.1f}% ({cnt[op] / 1e6:.1f}M inst)" for op, v in byop.most_common(8)))
    except (OSError, KeyError, IndexError):
        pass
    return out


def main(out_path, title, *prefixes):
    lines = [f"# {title}"]
    for p in prefixes:
        try:
            lines += summary(p)
        except (OSError, IndexError):
            lines.append(f"\n## {p}: no capture")
    open(out_path, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:])
