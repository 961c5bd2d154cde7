"""The PFASST driver's schedule (paper_1401_7824_b200/pfasst.py; NEXT f4b, R33)
on the CPU: the product's per-slice program, run by both transports over the ORACLE's slice phases
(oracle.PfasstSlice -- test infrastructure), must reproduce the oracle's serial emulation
ora_pfasst_block bit for bit:

* run_block_local: every slice in this process (the one-GPU mode);
* run_block_dist: one slice per rank of a world_size-2 / -3 gloo group (the multi-GPU mode, whose
  GPU runs use NCCL with the same calls): isend/irecv of the end values, all_reduce(MAX) stop test.

A schedule that received a value one stage early or late, dropped the forward transfer, or stopped
slices at different iterations would change the bits.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import synth  # noqa: E402
from synth import Config, FE_CUBIC, FE_FORCING, FE_NONE  # noqa: E402
from paper_1401_7824_b200 import pfasst  # noqa: E402

CASES = {
    "cubic_pred_fixed": (Config(0, 2, 15, 3, 0.01, 1.0, FE_CUBIC, fixed_sweeps=4), True, 1),
    "none_nopred_tol": (Config(0, 2, 15, 5, 0.02, 1.0, FE_NONE, sweep_tol=1e-12, max_sweeps=200), False, 2),
    "forcing_pred_tol": (Config(0, 2, 15, 3, 0.01, 0.5, FE_FORCING, sweep_tol=1e-11, max_sweeps=200), True, 1),
}


def _problem(ora, name):
    cfg, pred, cs = CASES[name]
    u0 = synth.initial_condition(2, 1, cfg.n) * (0.5 if cfg.fe == FE_CUBIC else 1.0)
    G = None
    if cfg.fe == FE_FORCING:
        x = synth.grid_x(cfg.n)
        G = np.outer(np.sin(2 * np.pi * x), np.sin(2 * np.pi * x))
    return cfg, ora.Problem(cfg, G), u0, pred, cs


def _kw(cfg, pred):
    return dict(max_iters=cfg.max_sweeps, fixed_iters=cfg.fixed_sweeps, tol=cfg.sweep_tol, predictor=pred)


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("P", [1, 3])
def test_local_transport_matches_oracle_block(ora, name, P):
    cfg, prob, u0, pred, cs = _problem(ora, name)
    step0 = 2
    ue, st = ora.pfasst_block(prob, u0, P, step0=step0, coarse_sweeps=cs, predictor=pred)
    slices = [ora.PfasstSlice(prob, u0, step0 + p, coarse_sweeps=cs) for p in range(P)]
    out = pfasst.run_block_local(slices, **_kw(cfg, pred))
    assert all(o.iterations == st["iterations"] for o in out)
    assert all(o.converged == st["converged"] for o in out)
    hist = np.array([o.res_hist for o in out]).T
    assert np.array_equal(hist, st["res_hist"])
    for p in range(P):
        assert np.array_equal(slices[p].end(), ue[p])
    assert sum(o.vcycles for o in out) == st["vcycles"]
    assert sum(o.coarse_vcycles for o in out) == st["coarse_vcycles"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    cfg, prob, u0, pred, cs = _problem(oracle, name)
    sl = oracle.PfasstSlice(prob, u0, 5 + rank, coarse_sweeps=cs)
    res = pfasst.run_block_dist(sl, **_kw(cfg, pred), nbytes=lambda t: int(np.asarray(t).nbytes))
    q.put((rank, res.iterations, res.converged, list(res.res_hist), sl.end(), res.vcycles, res.coarse_vcycles,
           res.sent, res.recv))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,name", [(2, "cubic_pred_fixed"), (3, "forcing_pred_tol"), (2, "none_nopred_tol")])
def test_gloo_ranks_match_oracle_block(ora, world, name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=300) for _ in range(world)), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg, prob, u0, pred, cs = _problem(ora, name)
    ue, st = ora.pfasst_block(prob, u0, world, step0=5, coarse_sweeps=cs, predictor=pred)
    for rank, it, conv, hist, end, vc, cvc, sent, recv in out:
        assert it == st["iterations"] and conv == st["converged"]
        assert np.array_equal(np.array(hist), st["res_hist"][:, rank])
        assert np.array_equal(end, ue[rank])
    assert sum(o[5] for o in out) == st["vcycles"] and sum(o[6] for o in out) == st["coarse_vcycles"]
    # forward transfer only: the last slice sends nothing, slice 0 receives nothing
    assert out[-1][7] == 0 and out[0][8] == 0 and out[0][7] == out[1][8]
