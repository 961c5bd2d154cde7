"""Write full-size oracle reference results for the GPU parity tests (tests/golden/full_*.json).

Calls only oracle/ (and the seeded input generator synth/).  Records, per time step, the sweep and
V-cycle counts, every residual (as exact float.hex strings) and, for the final solution, a SHA-256
of its little-endian fp64 bytes plus exact samples at fixed points.

    python scripts/oracle_golden.py 2 3 4 5          # configs to run (slow: minutes to ~1 h)
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")

# (config, seed, mode, steps): config 5 is limited to its first step (oracle cost)
JOBS = {
    2: [(2, 0, synth.MODE_ISDC, 10)],
    3: [(3, 0, synth.MODE_ISDC, 1), (3, 0, synth.MODE_SDC, 1)],
    4: [(4, 0, synth.MODE_ISDC, 1)],
    5: [(5, 0, synth.MODE_ISDC, 1)],
}


def sample_points(n, dim, count=64, seed=1234):
    rng = np.random.default_rng(seed)
    return rng.integers(0, n, size=(count, dim)).tolist()


def run(cid, seed, mode, steps):
    cfg, u0, G = synth.problem_inputs(cid, seed)
    prob = oracle.Problem(cfg, G, mode=mode)
    u = u0
    rec = dict(config=cid, seed=seed, mode=int(mode), steps=[], n=cfg.n, dim=cfg.dim,
               threads=oracle.num_threads())
    t0 = time.time()
    for s in range(steps):
        u, st = oracle.step(prob, u, float(s) * cfg.dt)
        rec["steps"].append(dict(sweeps=st["sweeps"], vcycles=st["vcycles"], converged=st["converged"],
                                 cap_hits=st["cap_hits"], res_hist=[float(x).hex() for x in st["res_hist"]],
                                 node_cycles=st["node_cycles"].tolist(), seconds=st["seconds"]))
        print(f"cfg {cid} mode {mode} step {s}: {st['sweeps']} sweeps, {st['vcycles']} cycles, "
              f"res {st['res_hist'][-1]:.3e}, {st['seconds']:.1f}s", flush=True)
    pts = sample_points(cfg.n, cfg.dim)
    rec["samples"] = [[p, float(u[tuple(reversed(p))]).hex()] for p in pts]   # p = (x, y[, z])
    rec["sha256"] = hashlib.sha256(np.ascontiguousarray(u, dtype="<f8").tobytes()).hexdigest()
    rec["max_abs"] = float(np.abs(u).max()).hex()
    rec["seconds"] = time.time() - t0
    name = f"full_cfg{cid}_seed{seed}_{'sdc' if mode else 'isdc'}.json"
    with open(os.path.join(OUT, name), "w") as f:
        json.dump(rec, f, indent=1)
    print("wrote", name, flush=True)


if __name__ == "__main__":
    cids = [int(a) for a in sys.argv[1:]] or [2, 3, 4, 5]
    for c in cids:
        for job in JOBS[c]:
            run(*job)
