"""Write full-size oracle reference results for the GPU parity tests (tests/golden/full_*.json).

Calls only oracle/ (and the seeded input generator synth/).  Records, per time step, the sweep and
V-cycle counts, every residual (as exact float.hex strings), the SHA-256 of that step's end value
u_M, and, for the final solution, exact samples at fixed points.

    python scripts/oracle_golden.py 2 3 4 5              # all jobs of these configs (minutes to hours)
    python scripts/oracle_golden.py 5:0:isdc:5            # one job: config:seed:mode:steps

Long jobs checkpoint after every step under $ISDC_GOLDEN_CKPT (default /tmp/isdc_golden_ckpt) and
resume from the last finished step (the oracle is deterministic, so a resumed run writes the same
bits as an uninterrupted one).
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
CKPT = os.environ.get("ISDC_GOLDEN_CKPT", "/tmp/isdc_golden_ckpt")

# (config, seed, mode, steps) -- every seed of SURVEY §8(d1) and the whole bench trajectory
JOBS = {
    2: [(2, s, synth.MODE_ISDC, 10) for s in (0, 1, 2)],
    3: [(3, 0, synth.MODE_ISDC, 1), (3, 0, synth.MODE_SDC, 1)],
    4: [(4, s, synth.MODE_ISDC, 1) for s in (0, 1, 2)],
    5: [(5, 0, synth.MODE_ISDC, 5)],
}


def sample_points(n, dim, count=64, seed=1234):
    rng = np.random.default_rng(seed)
    return rng.integers(0, n, size=(count, dim)).tolist()


def sha(u):
    return hashlib.sha256(np.ascontiguousarray(u, dtype="<f8").tobytes()).hexdigest()


def run(cid, seed, mode, steps):
    name = f"full_cfg{cid}_seed{seed}_{'sdc' if mode else 'isdc'}"
    cfg, u0, G = synth.problem_inputs(cid, seed)
    prob = oracle.Problem(cfg, G, mode=mode)
    os.makedirs(CKPT, exist_ok=True)
    ck_json, ck_u = os.path.join(CKPT, name + ".json"), os.path.join(CKPT, name + ".npy")
    rec = dict(config=cid, seed=seed, mode=int(mode), steps=[], n=cfg.n, dim=cfg.dim,
               threads=oracle.num_threads(), seconds=0.0)
    u = u0
    if os.path.exists(ck_json) and os.path.exists(ck_u):
        rec = json.load(open(ck_json))
        u = np.load(ck_u)
        assert sha(u) == rec["steps"][-1]["sha256"]
        print(f"{name}: resuming after step {len(rec['steps'])}", flush=True)
    for s in range(len(rec["steps"]), steps):
        t0 = time.time()
        u, st = oracle.step(prob, u, float(s) * cfg.dt)
        rec["steps"].append(dict(sweeps=st["sweeps"], vcycles=st["vcycles"], converged=st["converged"],
                                 cap_hits=st["cap_hits"], res_hist=[float(x).hex() for x in st["res_hist"]],
                                 node_cycles=st["node_cycles"].tolist(), seconds=st["seconds"],
                                 sha256=sha(u)))
        rec["seconds"] += time.time() - t0
        np.save(ck_u + ".tmp.npy", u)
        os.replace(ck_u + ".tmp.npy", ck_u)
        with open(ck_json + ".tmp", "w") as f:
            json.dump(rec, f)
        os.replace(ck_json + ".tmp", ck_json)
        print(f"cfg {cid} seed {seed} mode {mode} step {s}: {st['sweeps']} sweeps, {st['vcycles']} cycles, "
              f"res {st['res_hist'][-1]:.3e}, {st['seconds']:.1f}s", flush=True)
        write(name, rec, cfg, u)      # after every step: a long job's finished steps are usable at once


def write(name, rec, cfg, u):
    pts = sample_points(cfg.n, cfg.dim)
    rec["samples"] = [[p, float(u[tuple(reversed(p))]).hex()] for p in pts]   # p = (x, y[, z])
    rec["sha256"] = sha(u)
    rec["max_abs"] = float(np.abs(u).max()).hex()
    with open(os.path.join(OUT, name + ".json"), "w") as f:
        json.dump(rec, f, indent=1)
    print("wrote", name, flush=True)


if __name__ == "__main__":
    args = sys.argv[1:] or ["2", "3", "4", "5"]
    for a in args:
        if ":" in a:
            c, s, m, k = a.split(":")
            run(int(c), int(s), synth.MODE_SDC if m == "sdc" else synth.MODE_ISDC, int(k))
        else:
            for job in JOBS[int(a)]:
                run(*job)
