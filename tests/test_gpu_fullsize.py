"""Full-size parity (BASELINE.json sizes, the launch configuration bench.py times): the CUDA path
against oracle results stored by scripts/oracle_golden.py (a committed script that calls only
oracle/).  Checked: sweep / V-cycle / per-node cycle counts, every residual of every sweep
(exact bits), the final solution's SHA-256 and exact samples at fixed points."""
import glob
import hashlib
import json
import os

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

GOLD = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "full_cfg*.json")))


@pytest.mark.parametrize("path", GOLD, ids=[os.path.basename(p)[:-5] for p in GOLD])
def test_fullsize_against_oracle_golden(path):
    assert torch.cuda.is_available()
    import paper_1401_7824_b200 as pk
    rec = json.load(open(path))
    cfg, u0, G = synth.problem_inputs(rec["config"], rec["seed"])
    h = pk.ISDC.from_config(cfg, None if G is None else torch.from_numpy(G), mode=rec["mode"])
    h.set_initial(torch.from_numpy(u0).cuda(), 0)
    for s, ref in enumerate(rec["steps"]):
        st = h.step()
        assert st["sweeps"] == ref["sweeps"], (s, st["sweeps"], ref["sweeps"])
        assert st["vcycles"] == ref["vcycles"]
        assert st["converged"] == ref["converged"]
        assert st["node_cycles"].tolist() == ref["node_cycles"]
        got = [float(x).hex() for x in st["res_hist"]]
        assert got == ref["res_hist"], (s, got[-3:], ref["res_hist"][-3:])
        r_gpu = np.array([float.fromhex(x) for x in got])
        r_ref = np.array([float.fromhex(x) for x in ref["res_hist"]])
        assert np.all(np.abs(r_gpu - r_ref) <= 1e-9 * np.abs(r_ref))   # the north-star bar (implied)
        if "sha256" in ref:   # the end value u_M of every step of the trajectory
            u_s = h.solution(0).cpu().numpy()
            assert hashlib.sha256(np.ascontiguousarray(u_s, dtype="<f8").tobytes()).hexdigest() == ref["sha256"], s
    u = h.solution(0).cpu().numpy()
    for p, hx in rec["samples"]:
        assert float(u[tuple(reversed(p))]).hex() == hx, p
    assert float(np.abs(u).max()).hex() == rec["max_abs"]
    assert hashlib.sha256(np.ascontiguousarray(u, dtype="<f8").tobytes()).hexdigest() == rec["sha256"]
