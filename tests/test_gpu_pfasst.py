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
