"""Debug: compare V-cycles with fused kernels on vs off (ISDC_FUSE2D / ISDC_FUSE3D) at several sizes (bitwise)."""
import os, sys, subprocess
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch, synth
    import paper_1401_7824_b200 as pk
    n = int(sys.argv[2]); out = sys.argv[3]; dim = int(sys.argv[4])
    cfg = synth.Config(0, dim, n, 5, 0.01, 0.1, synth.FE_NONE)
    h = pk.ISDC.from_config(cfg)
    b = synth.random_field(n, dim, 21); u = torch.from_numpy(synth.random_field(n, dim, 22)).cuda()
    d = []
    for m in range(2):
        d.append(h.vcycle(m, b, u))
    np.save(out, u.cpu().numpy()); print(d)
    sys.exit(0)
for dim, n in [(2, 127), (2, 255), (2, 511), (2, 1023), (2, 2047), (2, 4095), (3, 63), (3, 127), (3, 255), (3, 511)]:
    outs = []
    for f in ("0", "1"):
        env = dict(os.environ, ISDC_FUSE2D=f, ISDC_FUSE3D=f)   # fused paths on (1) / off (0)
        fn = f"/tmp/fz_{dim}_{n}_{f}.npy"
        r = subprocess.run([sys.executable, __file__, "child", str(n), fn, str(dim)], env=env, capture_output=True, text=True, timeout=600)
        outs.append(np.load(fn) if r.returncode == 0 else None)
        if r.returncode: print(r.stderr[-500:])
    a, b = outs
    if a is None or b is None: print(n, "failed"); continue
    diff = np.argwhere(a != b)
    print(dim, n, "equal" if len(diff) == 0 else f"{len(diff)} diffs, first {diff[:5].tolist()}, maxabs {np.abs(a-b).max():.3e}", flush=True)
