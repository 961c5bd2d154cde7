"""Debug: compare 2D V-cycles with ISDC_FUSE2D=1 vs 0 at several sizes (bitwise)."""
import os, sys, subprocess
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch, synth
    import paper_1401_7824_b200 as pk
    n = int(sys.argv[2]); out = sys.argv[3]
    cfg = synth.Config(0, 2, n, 5, 0.01, 0.1, synth.FE_NONE)
    h = pk.ISDC.from_config(cfg)
    b = synth.random_field(n, 2, 21); u = torch.from_numpy(synth.random_field(n, 2, 22)).cuda()
    d = []
    for m in range(2):
        d.append(h.vcycle(m, b, u))
    np.save(out, u.cpu().numpy()); print(d)
    sys.exit(0)
for n in (127, 255, 511, 1023, 2047, 4095):
    outs = []
    for f in ("0", "1"):
        env = dict(os.environ, ISDC_FUSE2D=f)
        fn = f"/tmp/fz_{n}_{f}.npy"
        r = subprocess.run([sys.executable, __file__, "child", str(n), fn], env=env, capture_output=True, text=True, timeout=600)
        outs.append(np.load(fn) if r.returncode == 0 else None)
        if r.returncode: print(r.stderr[-500:])
    a, b = outs
    if a is None or b is None: print(n, "failed"); continue
    diff = np.argwhere(a != b)
    print(n, "equal" if len(diff) == 0 else f"{len(diff)} diffs, first {diff[:5].tolist()}, maxabs {np.abs(a-b).max():.3e}", flush=True)
