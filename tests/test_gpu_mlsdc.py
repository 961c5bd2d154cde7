"""GPU parity of two-level MLSDC with ISDC sweeps (NEXT f4, R32): the CUDA path
(fine handle + coarse handle, transfer / FAS kernels of kernels_mlsdc.cuh) against the oracle's
ora_mlsdc_step on identical seeded inputs -- counts, every residual and the solution bit for bit."""
import numpy as np
import pytest

import synth
from synth import Config, FE_ADVECTION, FE_CUBIC, FE_FORCING, FE_NONE, MODE_ISDC, MODE_SDC

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def gpu():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    import paper_1401_7824_b200 as pk
    pk.lib()
    return pk


CASES = [  # (dim, n, M, fe, coarse_sweeps, fixed_sweeps, nu, dt)
    (2, 7, 3, FE_NONE, 1, 0, 1.0, 0.01),            # the coarse level is the single 3^2 exact solve
    (2, 63, 3, FE_NONE, 1, 0, 10.0, 0.001),         # Table-1a type problem
    (2, 127, 5, FE_FORCING, 2, 0, 0.1, 0.01),       # fast 2D kernels on both levels (63 coarse)
    (2, 255, 5, FE_CUBIC, 1, 0, 1e-3, 0.005),
    (2, 63, 5, FE_NONE, 0, 4, 1.0, 0.01),           # no coarse sweep: plain ISDC
    (3, 15, 3, FE_NONE, 1, 0, 1.0, 0.01),
    (3, 63, 5, FE_ADVECTION, 1, 0, 0.01, 0.002),    # stored CD4 f^E on both levels (fast 3D fine, 31 coarse)
    (3, 63, 3, FE_NONE, 2, 3, 1.0, 0.01),
]


@pytest.mark.parametrize("dim,n,M,fe,cs,fixed,nu,dt", CASES)
def test_mlsdc_steps_bitwise(gpu, ora, dim, n, M, fe, cs, fixed, nu, dt):
    cfg = Config(0, dim, n, M, dt, nu, fe, fe_a=(1.0, 0.5, 0.25), fixed_sweeps=fixed, sweep_tol=1e-10, max_sweeps=100)
    G = synth.forcing_field(n, dim) if fe == FE_FORCING else None
    u0 = synth.initial_condition(5 if dim == 3 else 3, 0, n) if fe != FE_CUBIC else synth.initial_condition(2, 0, n)
    h = gpu.ISDC.from_config(cfg, None if G is None else torch.from_numpy(G), mode=MODE_ISDC, mlsdc_levels=2,
                             coarse_sweeps=cs)
    prob = ora.Problem(cfg, G)
    h.set_initial(torch.from_numpy(u0).cuda(), 0)
    u_ref = u0.copy()
    for s in range(2):
        st = h.step()
        u_ref, st_ref = ora.mlsdc_step(prob, u_ref, float(s) * dt, coarse_sweeps=cs)
        assert st["sweeps"] == st_ref["sweeps"] and st["vcycles"] == st_ref["vcycles"], (s, st["sweeps"], st_ref["sweeps"])
        assert st["coarse_vcycles"] == st_ref["coarse_vcycles"]
        assert st["converged"] == st_ref["converged"]
        assert np.array_equal(st["res_hist"], st_ref["res_hist"]), (s, st["res_hist"][-3:], st_ref["res_hist"][-3:])
        assert np.array_equal(h.solution(0).cpu().numpy(), u_ref)


def test_mlsdc_rejects_unsupported(gpu):
    cfg = Config(0, 2, 63, 3, 0.01, 1.0, FE_NONE)
    with pytest.raises(gpu.IsdcError) as ei:
        gpu.ISDC.from_config(cfg, mode=MODE_SDC, mlsdc_levels=2)
    assert ei.value.status == 2
