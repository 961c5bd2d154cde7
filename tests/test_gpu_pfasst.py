"""GPU parity of PFASST with ISDC sweeps (NEXT f4b, R33): P slice handles
(MLSDC handles, include/isdc.h isdc_pfasst_*) scheduled by the product driver
(paper_1401_7824_b200/pfasst.py, one-GPU transport) against the oracle's serial emulation
ora_pfasst_block on identical seeded inputs -- iterations, every slice's residual history, the
V-cycle counts and every slice's end value bit for bit."""
import numpy as np
import pytest

import synth
from synth import Config, FE_ADVECTION, FE_CUBIC, FE_FORCING, FE_NONE, MODE_ISDC

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def gpu():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    import paper_1401_7824_b200 as pk
    pk.lib()
    return pk


CASES = [  # (dim, n, M, fe, P, predictor, coarse_sweeps, fixed, nu, dt)
    (2, 15, 3, FE_NONE, 1, False, 1, 0, 1.0, 0.02),
    (2, 31, 3, FE_NONE, 4, True, 1, 0, 1.0, 0.02),
    (2, 63, 5, FE_FORCING, 3, True, 2, 0, 0.1, 0.01),
    (2, 127, 5, FE_CUBIC, 4, False, 1, 0, 1e-3, 0.005),
    (2, 255, 3, FE_FORCING, 2, True, 1, 5, 0.1, 0.01),
    (3, 15, 3, FE_NONE, 3, True, 1, 0, 1.0, 0.01),
    (3, 63, 5, FE_ADVECTION, 2, True, 1, 0, 0.01, 0.002),
]


@pytest.mark.parametrize("dim,n,M,fe,P,pred,cs,fixed,nu,dt", CASES)
def test_pfasst_block_bitwise(gpu, ora, dim, n, M, fe, P, pred, cs, fixed, nu, dt):
    from paper_1401_7824_b200 import pfasst
    cfg = Config(0, dim, n, M, dt, nu, fe, fe_a=(1.0, 0.5, 0.25), fixed_sweeps=fixed, sweep_tol=1e-10,
                 max_sweeps=100)
    G = synth.forcing_field(n, dim) if fe == FE_FORCING else None
    u0 = synth.initial_condition(5 if dim == 3 else 3, 0, n) if fe != FE_CUBIC else synth.initial_condition(2, 0, n)
    step0 = 1
    slices = []
    for p in range(P):
        h = gpu.ISDC.from_config(cfg, None if G is None else torch.from_numpy(G), mode=MODE_ISDC, mlsdc_levels=2,
                                 coarse_sweeps=cs)
        slices.append(pfasst.CudaSlice(h, torch.from_numpy(u0).cuda(), step0 + p))
    out = pfasst.run_block_local(slices, max_iters=cfg.max_sweeps, fixed_iters=fixed, tol=cfg.sweep_tol,
                                 predictor=pred)
    ue, st = ora.pfasst_block(ora.Problem(cfg, G), u0, P, step0=step0, coarse_sweeps=cs, predictor=pred)
    assert all(o.iterations == st["iterations"] and o.converged == st["converged"] for o in out)
    hist = np.array([o.res_hist for o in out]).T
    assert np.array_equal(hist, st["res_hist"]), (hist[-1], st["res_hist"][-1])
    assert sum(o.vcycles for o in out) == st["vcycles"]
    assert sum(o.coarse_vcycles for o in out) == st["coarse_vcycles"]
    for p in range(P):
        assert np.array_equal(slices[p].end().cpu().numpy(), ue[p]), p


def test_pfasst_needs_mlsdc_handle(gpu):
    from paper_1401_7824_b200 import pfasst
    cfg = Config(0, 2, 31, 3, 0.01, 1.0, FE_NONE)
    h = gpu.ISDC.from_config(cfg, mode=MODE_ISDC)
    with pytest.raises(ValueError):
        pfasst.CudaSlice(h, torch.zeros(31, 31, dtype=torch.float64, device="cuda"), 0)
    with pytest.raises(gpu.IsdcError) as ei:
        h.pfasst_restrict()
    assert ei.value.status == 1


def _dist_worker(rank, world, port, q):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1401_7824_b200 as pk
    from paper_1401_7824_b200 import pfasst
    cfg, G, u0 = _dist_case()
    h = pk.ISDC.from_config(cfg, torch.from_numpy(G), mode=MODE_ISDC, mlsdc_levels=2, coarse_sweeps=1)
    sl = pfasst.CudaSlice(h, torch.from_numpy(u0).cuda(), 1 + rank)
    res = pfasst.run_block_dist(sl, max_iters=cfg.max_sweeps, fixed_iters=0, tol=cfg.sweep_tol, predictor=True)
    q.put((rank, res.iterations, list(res.res_hist), sl.end().cpu().numpy()))
    dist.barrier()
    dist.destroy_process_group()


def _dist_case():
    n = 63
    cfg = Config(0, 2, n, 3, 0.01, 0.1, FE_FORCING, sweep_tol=1e-10, max_sweeps=100)
    return cfg, synth.forcing_field(n, 2), synth.initial_condition(3, 0, n)


def test_pfasst_dist_transport_with_cuda_slices(gpu, ora):
    """The multi-rank transport (run_block_dist: isend/recv of end values, all_reduce MAX) driving
    CUDA slices, one per process: two processes on this GPU exchange through host memory over gloo
    (no kernel waits on another process), bit for bit the oracle block."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=600) for _ in range(2)), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg, G, u0 = _dist_case()
    ue, st = ora.pfasst_block(ora.Problem(cfg, G), u0, 2, step0=1, coarse_sweeps=1, predictor=True)
    for rank, it, hist, end in out:
        assert it == st["iterations"]
        assert np.array_equal(np.array(hist), st["res_hist"][:, rank])
        assert np.array_equal(end, ue[rank])
