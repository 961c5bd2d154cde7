"""Weighted (default, R15) vs the paper's unweighted residual (residual_kind 1)
in the stop test of the 2D configs: sweeps, V-cycles, W-cycles and device time per step on the GPU.
Writes profiles/residual_kinds_r02.md (answers ADVICE r1: report the unweighted counts beside the
weighted ones).  3D has no unweighted form (R15: the V-cycle on B_h stalls in 3D)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1401_7824_b200 as pk  # noqa: E402

rows = []
for cid in (2, 3):
    cfg, u0, G = synth.problem_inputs(cid, 0)
    for kind in (0, 1):
        h = pk.ISDC.from_config(cfg, None if G is None else torch.from_numpy(G), mode=synth.MODE_ISDC,
                                residual_kind=kind)
        h.set_initial(torch.from_numpy(u0).cuda(), 0)
        h.step()                                   # warm-up (graph capture)
        h.set_initial(torch.from_numpy(u0).cuda(), 0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(h.stream)
        sts = [h.step() for _ in range(cfg.steps)]
        e1.record(h.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / cfg.steps
        rows.append((cid, kind, [s["sweeps"] for s in sts], sum(s["vcycles"] for s in sts) / cfg.steps,
                     sum(s["wcycles"] for s in sts) / cfg.steps, ms))
        del h
        torch.cuda.empty_cache()
out = ["# Weighted vs unweighted residual in the stop test (2D configs, ISDC, seed 0, one B200)", "",
       "residual_kind 0 = weighted ||B_h r||_inf (DESIGN.md R15, the default); 1 = the paper's unweighted",
       "||r||_inf = ||W^-1 r~||_inf (P:78, P:87-88; W^-1 by V-cycles on B_h, counted apart as W-cycles, P:165).", "",
       "| config | residual | sweeps per step | V-cycles per step | W-cycles per step | ms per step |", "|---|---|---|---|---|---|"]
for cid, kind, sw, vc, wc, ms in rows:
    out.append(f"| {cid} | {'unweighted' if kind else 'weighted'} | {', '.join(map(str, sw))} | {vc:.1f} | {wc:.1f} | {ms:.2f} |")
open(os.path.join(ROOT, "profiles", "residual_kinds_r02.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
