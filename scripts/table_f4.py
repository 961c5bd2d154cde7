"""NEXT f4 on the paper's Table-1a problems: single-level ISDC vs ISDC sweeps inside MLSDC
(reading R32) vs PFASST blocks of 4 slices (reading R33), on the CUDA path
(bitwise equal to the oracle by tests/test_gpu_mlsdc.py and tests/test_gpu_pfasst.py).  Writes
profiles/table_f4_<tag>.md.

    python scripts/table_f4.py r02
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1401_7824_b200 as pk  # noqa: E402
from paper_1401_7824_b200 import pfasst  # noqa: E402
import synth  # noqa: E402
from synth import Config, FE_NONE, MODE_ISDC  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
n, P = 63, 4
u0n = synth.sine_mode(n, (1, 1))
u0 = torch.from_numpy(u0n).cuda()
out = ["# NEXT f4 on the paper's Table-1a problems (B200), " + time.strftime("%Y-%m-%d"), "",
       "2D heat, u0 = sin(pi x) sin(pi y), h = 1/64, dt = 0.001, L = 2 V(2,2) cycles per node solve, tol 5e-8",
       "(P:114-117).  Per time step (PFASST: per slice of a block of 4 consecutive steps): fine sweeps /",
       "iterations, fine V-cycles, coarse V-cycles (MLSDC / PFASST: the coarse level n = 31, one coarse ISDC",
       "sweep per iteration; PFASST with the pipelined coarse predictor).  P:204: MLSDC moves work to the",
       "coarse level;",
       "P:208-209: PFASST runs one sweep per level and iteration on all slices at once, so its iterations",
       "are the parallel critical path.", "",
       "| nu | M | ISDC sweeps (V-cycles) | MLSDC fine sweeps (fine V / coarse V) | PFASST iterations (fine V / coarse V per slice) | serial steps' fine sweeps vs PFASST iterations |",
       "|---|---|---|---|---|---|"]
for nu in (1, 10, 100):
    for M in (3, 5, 7):
        cfg = Config(0, 2, n, M, 0.001, float(nu), FE_NONE, sweep_tol=5e-8, max_sweeps=100)
        h = pk.ISDC.from_config(cfg, mode=MODE_ISDC)
        h.set_initial(u0, 0)
        si = h.step()
        hm = pk.ISDC.from_config(cfg, mode=MODE_ISDC, mlsdc_levels=2, coarse_sweeps=1)
        hm.set_initial(u0, 0)
        sm = hm.step()
        hs = [pk.ISDC.from_config(cfg, mode=MODE_ISDC, mlsdc_levels=2, coarse_sweeps=1) for _ in range(P)]
        sl = [pfasst.CudaSlice(hs[p], u0, p) for p in range(P)]
        res = pfasst.run_block_local(sl, max_iters=cfg.max_sweeps, fixed_iters=0, tol=cfg.sweep_tol, predictor=True)
        # the same 4 steps serially (single-level ISDC)
        hser = pk.ISDC.from_config(cfg, mode=MODE_ISDC)
        hser.set_initial(u0, 0)
        ser = sum(hser.step()["sweeps"] for _ in range(P))
        it = res[0].iterations
        fv = sum(r.vcycles for r in res) / P
        cv = sum(r.coarse_vcycles for r in res) / P
        out.append(f"| {nu} | {M} | {si['sweeps']} ({si['vcycles']}) | {sm['sweeps']} ({sm['vcycles']} / {sm['coarse_vcycles']}) | "
                   f"{it} ({fv:.0f} / {cv:.0f}) | {ser} vs {it} |")
path = os.path.join(ROOT, "profiles", f"table_f4_{tag}.md")
open(path, "w").write("\n".join(out) + "\n")
print("\n".join(out))
