"""Per-class device time of one Burgers ISDC step (Table 1b problem), CUDA events on every launch.
    python scripts/burgers_profile.py [nu] [M]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1401_7824_b200 as pk  # noqa: E402
import synth  # noqa: E402

nu = float(sys.argv[1]) if len(sys.argv) > 1 else 10.0
M = int(sys.argv[2]) if len(sys.argv) > 2 else 7
cfg = synth.burgers_config(nu, M)
u0 = torch.from_numpy(synth.burgers_initial(cfg.n)).cuda()
for mode in (pk.MODE_ISDC, pk.MODE_SDC):
    h = pk.ISDC.from_config(cfg, mode=mode)
    h.set_initial(u0, 0)
    h.step()
    h.set_initial(u0, 0)
    l0 = h.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(h.stream)
    st = h.step()
    e1.record(h.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    nl = h.launches - l0
    h.set_initial(u0, 0)
    h.profile(2)
    h.profile_reset()
    h.step()
    prof = h.profile_get()
    h.profile(0)
    print(f"mode {mode}: {ms:.2f} ms/step, {st['sweeps']} sweeps, {st['vcycles']} V-cycles, {nl} launches "
          f"({1000 * ms / max(nl, 1):.2f} us/launch)")
    for k, (t, n, b) in prof.items():
        if n:
            print(f"   {k:22s} {t:8.2f} ms  {n:6d} launches  {1000 * t / n:7.2f} us/launch")
