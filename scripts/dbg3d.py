"""Debug helper: run 3D V-cycles through the C-ABI with individual fast kernels masked (env)."""
import os, sys, subprocess
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch, synth
    import paper_1401_7824_b200 as pk
    n = int(sys.argv[2])
    cfg = synth.Config(0, 3, n, 3, 0.01, 1.0, synth.FE_NONE)
    h = pk.ISDC.from_config(cfg)
    b = synth.random_field(n, 3, 21); u = torch.from_numpy(synth.random_field(n, 3, 22)).cuda()
    d0, d1 = h.vcycle(0, b, u)
    torch.cuda.synchronize()
    print("ok", d0, d1, float(u.abs().max()))
    sys.exit(0)
for n in (31, 63):
    for mask in ("0", "1", "2", "4", "7"):
        env = dict(os.environ, ISDC_FAST3D_MASK=mask, CUDA_LAUNCH_BLOCKING="1", ISDC_NO_GRAPHS="1")
        r = subprocess.run([sys.executable, __file__, "child", str(n)], env=env, capture_output=True, text=True, timeout=300)
        print(n, mask, r.returncode, (r.stdout.strip() or r.stderr.strip().splitlines()[-1])[:300], flush=True)
