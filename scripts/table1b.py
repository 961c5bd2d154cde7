"""Table 1b of the paper on the CUDA path (NEXT f3): viscous Burgers, periodic, WENO5 advection.
SDC / fixed-L ISDC / ISDC-capped counts next to the paper's, plus the device time of
each step.  Writes profiles/table1b_<tag>.md.   python scripts/table1b.py r01"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1401_7824_b200 as pk  # noqa: E402
import synth  # noqa: E402
from synth import MODE_ISDC, MODE_ISDC_CAPPED, MODE_SDC  # noqa: E402

PAPER = {  # (nu, M): (SDC cycles, SDC sweeps, ISDC cycles, ISDC sweeps, source line)
    (0.1, 3): (21, 8, 21, 8, "P:144"), (0.1, 5): (26, 6, 26, 6, "P:145"), (0.1, 7): (33, 5, 33, 5, "P:146"),
    (1.0, 3): (97, 17, 66, 17, "P:148"), (1.0, 5): (140, 17, 117, 17, "P:149"), (1.0, 7): (160, 15, 143, 15, "P:150"),
    (10.0, 3): (207, 25, 100, 25, "P:152"), (10.0, 5): (523, 38, 298, 38, "P:153"),
    (10.0, 7): (902, 50, 578, 50, "P:154"),
}

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
out = ["# Table 1b on the CUDA path (B200), " + time.strftime("%Y-%m-%d"),
       "",
       "2D viscous Burgers on [-1,1)^2, periodic, u0 = exp(-(x^2+y^2)/0.01), WENO5-JS advection on Lax-Friedrichs",
       "split fluxes, compact 4th-order diffusion, h = 1/64 (n = 128, reading R30), dt = 0.001, L = 2, tol 5e-8",
       "(P:106-117, P:158).  Entries: accumulated V-cycles (sweeps) of one step; 'paper' = Table 1b (P:140-156).",
       "This build's multigrid is V(2,2) weighted Jacobi on the periodic hierarchy down to 4x4 (reading R11/R31;",
       "the paper's is unspecified, P:213): cycle counts are trend-only.  Every entry equals the CPU oracle bit",
       "for bit (tests/test_gpu_burgers.py).  ms = device time of the step (CUDA events, after one warm-up step).",
       "",
       "| nu | M | SDC paper | SDC ours | ISDC paper | ISDC (fixed L) ours | ISDC-capped ours | savings paper | savings ours (fixed / capped) | ms SDC / ISDC | source |",
       "|---|---|---|---|---|---|---|---|---|---|---|"]
for (nu, M), (sc, ss, ic, is_, src) in sorted(PAPER.items()):
    cfg = synth.burgers_config(nu, M)
    u0 = torch.from_numpy(synth.burgers_initial(cfg.n)).cuda()
    res, ms = {}, {}
    for mode in (MODE_SDC, MODE_ISDC, MODE_ISDC_CAPPED):
        h = pk.ISDC.from_config(cfg, mode=mode)
        h.set_initial(u0, 0)
        h.step()                                   # warm-up (graph capture)
        h.set_initial(u0, 0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(h.stream)
        st = h.step()
        e1.record(h.stream)
        torch.cuda.synchronize()
        res[mode] = (st["vcycles"], st["sweeps"])
        ms[mode] = e0.elapsed_time(e1)
    s_ours = res[MODE_SDC][0]
    sav = lambda c: f"{100.0 * (1 - c / s_ours):.0f}%"   # noqa: E731
    out.append(f"| {nu:g} | {M} | {sc} ({ss}) | {res[MODE_SDC][0]} ({res[MODE_SDC][1]}) | {ic} ({is_}) | "
               f"{res[MODE_ISDC][0]} ({res[MODE_ISDC][1]}) | {res[MODE_ISDC_CAPPED][0]} ({res[MODE_ISDC_CAPPED][1]}) | "
               f"{100.0 * (1 - ic / sc):.0f}% | {sav(res[MODE_ISDC][0])} / {sav(res[MODE_ISDC_CAPPED][0])} | "
               f"{ms[MODE_SDC]:.2f} / {ms[MODE_ISDC]:.2f} | {src} |")
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
path = os.path.join(ROOT, "profiles", f"table1b_{tag}.md")
open(path, "w").write("\n".join(out) + "\n")
print("\n".join(out))
