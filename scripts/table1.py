"""Table 1a of the paper on the CUDA path: SDC / fixed-L ISDC / ISDC-capped counts next to the
paper's.  Writes profiles/table1_<tag>.md.   python scripts/table1.py r01"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1401_7824_b200 as pk  # noqa: E402
import synth  # noqa: E402
from synth import Config, FE_NONE, MODE_ISDC, MODE_ISDC_CAPPED, MODE_SDC  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
rows = []
for line in open(os.path.join(ROOT, "tests", "golden", "paper_table1.txt")):
    if line.startswith("#") or not line.strip():
        continue
    f = line.split()
    rows.append((int(f[0]), int(f[1]), [int(x) for x in f[2:6]], f[6]))
n = 63
u0 = torch.from_numpy(synth.sine_mode(n, (1, 1))).cuda()
out = ["# Table 1a on the CUDA path (B200), " + time.strftime("%Y-%m-%d"),
       "",
       "2D heat, u0 = sin(pi x) sin(pi y), h = 1/64, dt = 0.001, L = 2, tol 5e-8 (P:114-117).  Entries are",
       "accumulated V-cycles (sweeps) for one step; 'paper' = Table 1 (P:126-136).  This build's multigrid is",
       "V(2,2) weighted Jacobi (reading R11; the paper's is unspecified, P:213), so cycle counts are",
       "trend-only; SDC sweep counts are the comparable quantity.  ISDC-capped = at most L cycles per node",
       "solve, stopping at the SDC inner tolerance (reading R10).",
       "",
       "| nu | M | SDC paper | SDC ours | ISDC paper | ISDC (fixed L) ours | ISDC-capped ours | savings paper | savings ours (fixed / capped) | source |",
       "|---|---|---|---|---|---|---|---|---|---|"]
for nu, M, (sc, ss, ic, is_), src in rows:
    cfg = Config(0, 2, n, M, 0.001, float(nu), FE_NONE, sweep_tol=5e-8, max_sweeps=100)
    res = {}
    for mode in (MODE_SDC, MODE_ISDC, MODE_ISDC_CAPPED):
        h = pk.ISDC.from_config(cfg, mode=mode)
        h.set_initial(u0, 0)
        st = h.step()
        res[mode] = (st["vcycles"], st["sweeps"])
    s_ours = res[MODE_SDC][0]
    sav = lambda c: f"{100.0 * (1 - c / s_ours):.0f}%"   # noqa: E731
    out.append(f"| {nu} | {M} | {sc} ({ss}) | {res[MODE_SDC][0]} ({res[MODE_SDC][1]}) | {ic} ({is_}) | "
               f"{res[MODE_ISDC][0]} ({res[MODE_ISDC][1]}) | {res[MODE_ISDC_CAPPED][0]} ({res[MODE_ISDC_CAPPED][1]}) | "
               f"{100.0 * (1 - ic / sc):.0f}% | {sav(res[MODE_ISDC][0])} / {sav(res[MODE_ISDC_CAPPED][0])} | {src} |")
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
path = os.path.join(ROOT, "profiles", f"table1_{tag}.md")
open(path, "w").write("\n".join(out) + "\n")
print("\n".join(out))
