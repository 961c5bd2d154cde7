"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle on identical seeded inputs.

The bar (north_star): u within 1e-11 relative max-norm after every step, each
reported residual within 1e-9 relative, identical sweep and V-cycle counts.  The canonical
arithmetic contract makes both sides bit-identical, so most checks below are exact equality
(``==`` on values; the sign of a zero is the only freedom).
"""
import dataclasses

import numpy as np
import pytest

import synth
from synth import FE_ADVECTION, FE_CUBIC, FE_FORCING, FE_NONE, MODE_ISDC, MODE_ISDC_CAPPED, MODE_SDC

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def gpu():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    import paper_1401_7824_b200 as pk
    pk.lib()  # raises when the library is missing: no fallback
    return pk


def rel(a, b):
    den = max(np.abs(b).max(), 1e-300)
    return np.abs(np.asarray(a) - np.asarray(b)).max() / den


def make(gpu, cfg, G=None, mode=MODE_ISDC, **kw):
    return gpu.ISDC.from_config(cfg, None if G is None else torch.from_numpy(G), mode=mode, **kw)


# ------------------------------------------------------------------------------------ tables
@pytest.mark.parametrize("M", [2, 3, 4, 5, 7, 8])
def test_tables_bitwise(gpu, ora, M):
    cfg = synth.Config(0, 2, 7, M, 0.01, 1.0, FE_NONE)
    h = make(gpu, cfg)
    for a, b in zip(h.tables(), ora.tables(M)):
        assert np.array_equal(a, b)


# --------------------------------------------------------------------------------- V-cycle
@pytest.mark.parametrize("dim,n,M,dt,nu", [(2, 63, 3, 0.01, 1.0), (2, 127, 5, 0.01, 0.1), (2, 255, 5, 0.005, 1e-3),
                                           (3, 15, 3, 0.01, 1.0), (3, 31, 5, 0.002, 0.01), (3, 63, 3, 0.01, 1.0),
                                           (3, 127, 3, 0.01, 1.0), (3, 127, 5, 0.002, 0.01)])
def test_vcycle_bitwise(gpu, ora, dim, n, M, dt, nu):
    cfg = synth.Config(0, dim, n, M, dt, nu, FE_NONE)
    h = make(gpu, cfg)
    tau, Q, S, dtau = ora.tables(M)
    b = synth.random_field(n, dim, 21)
    u0 = synth.random_field(n, dim, 22)
    for m in range(M - 1):
        gamma = nu * (dt * dtau[m])
        u_ref = u0.copy()
        u_dev = torch.from_numpy(u0.copy()).cuda()
        for cyc in range(3):
            d0_ref = ora.defect_norm(b, u_ref, gamma)
            u_ref = ora.vcycle(b, u_ref, gamma)
            d1_ref = ora.defect_norm(b, u_ref, gamma)
            d0, d1 = h.vcycle(m, b, u_dev)
            assert d0 == d0_ref and d1 == d1_ref, (m, cyc, d0, d0_ref, d1, d1_ref)
            assert np.array_equal(u_dev.cpu().numpy(), u_ref), (m, cyc, rel(u_dev.cpu().numpy(), u_ref))


# ----------------------------------------------------------------------------- RHS / residual
FE_CASES = [(2, FE_NONE), (2, FE_CUBIC), (2, FE_FORCING), (2, FE_ADVECTION), (3, FE_NONE), (3, FE_CUBIC),
            (3, FE_FORCING), (3, FE_ADVECTION)]


@pytest.mark.parametrize("dim,fe", FE_CASES)
def test_rhs_and_residual_bitwise(gpu, ora, dim, fe):
    n = 31 if dim == 3 else 63
    M = 5
    cfg = synth.Config(0, dim, n, M, 0.01, 0.3, fe, fe_a=(1.0, -0.5, 0.25))
    G = synth.forcing_field(n, dim) if fe == FE_FORCING else None
    h = make(gpu, cfg, G)
    prob = ora.Problem(cfg, G)
    uold = [synth.random_field(n, dim, 30 + j) for j in range(M)]
    unew = [synth.random_field(n, dim, 40 + j) for j in range(M)]
    step_index = 3
    tn = float(step_index) * cfg.dt
    for m in range(M - 1):
        b = h.rhs(m, uold, unew[m], step_index).cpu().numpy()
        assert np.array_equal(b, ora.rhs(prob, tn, m, uold, unew)), m
    h.set_state(uold, step_index)
    r, per = h.residual()
    r_ref, per_ref = ora.residual(prob, tn, uold)
    assert r == r_ref and np.array_equal(per, per_ref)


# ------------------------------------------------------------------------------------- sweep
@pytest.mark.parametrize("dim,fe,mode,n", [(2, FE_NONE, MODE_ISDC, 127), (2, FE_CUBIC, MODE_SDC, 127),
                                           (2, FE_FORCING, MODE_ISDC, 127), (3, FE_ADVECTION, MODE_ISDC, 31),
                                           (3, FE_NONE, MODE_SDC, 31), (3, FE_NONE, MODE_ISDC, 63),
                                           (3, FE_ADVECTION, MODE_ISDC, 63), (3, FE_CUBIC, MODE_SDC, 63),
                                           (2, FE_FORCING, MODE_ISDC_CAPPED, 127), (3, FE_NONE, MODE_ISDC_CAPPED, 63)])
def test_sweep_bitwise(gpu, ora, dim, fe, mode, n):
    M = 5 if fe != FE_NONE else 3
    cfg = synth.Config(0, dim, n, M, 0.01, 0.5, fe, fe_a=(1.0, 0.5, 0.25))
    G = synth.forcing_field(n, dim) if fe == FE_FORCING else None
    h = make(gpu, cfg, G, mode=mode)
    prob = ora.Problem(cfg, G, mode=mode)
    state = [0.5 * synth.random_field(n, dim, 50 + j) for j in range(M)]
    h.set_state(state, 1)
    for k in range(3):
        per, mx, cyc = h.sweep()
        state, cyc_ref = ora.sweep(prob, 1 * cfg.dt, state)
        assert cyc == cyc_ref
        r_ref, per_ref = ora.residual(prob, 1 * cfg.dt, state)
        assert mx == r_ref and np.array_equal(per, per_ref)
        for j in range(M):
            assert np.array_equal(h.solution(j).cpu().numpy(), state[j]), (k, j)


# -------------------------------------------------------------------------------------- steps
STEP_CASES = [
    (1, 0, None, MODE_ISDC), (1, 1, None, MODE_ISDC), (1, 2, None, MODE_ISDC),
    (1, 0, None, MODE_SDC), (1, 1, None, MODE_SDC), (1, 2, None, MODE_SDC),
    (2, 0, 127, MODE_ISDC), (2, 1, 127, MODE_ISDC), (2, 2, 127, MODE_ISDC),
    (3, 0, 255, MODE_ISDC), (3, 0, 255, MODE_SDC),
    (4, 0, 31, MODE_ISDC), (4, 1, 31, MODE_ISDC), (4, 2, 31, MODE_ISDC),
    (5, 0, 31, MODE_ISDC), (5, 0, 63, MODE_ISDC),
    (2, 0, 127, MODE_ISDC_CAPPED), (4, 0, 31, MODE_ISDC_CAPPED),
]


@pytest.mark.parametrize("cid,seed,n,mode", STEP_CASES)
def test_steps_bitwise(gpu, ora, cid, seed, n, mode):
    cfg, u0, G = synth.problem_inputs(cid, seed, n)
    steps = min(cfg.steps, 3)
    h = make(gpu, cfg, G, mode=mode)
    prob = ora.Problem(cfg, G, mode=mode)
    h.set_initial(torch.from_numpy(u0).cuda(), 0)
    u_ref = u0.copy()
    for s in range(steps):
        st = h.step()
        u_ref, st_ref = ora.step(prob, u_ref, float(s) * cfg.dt)
        assert st["sweeps"] == st_ref["sweeps"] and st["vcycles"] == st_ref["vcycles"]
        assert st["converged"] == st_ref["converged"]
        assert np.array_equal(st["node_cycles"], st_ref["node_cycles"])
        assert np.array_equal(st["res_hist"], st_ref["res_hist"])
        u = h.solution(0).cpu().numpy()
        assert rel(u, u_ref) <= 1e-11
        assert np.array_equal(u, u_ref)
        if mode == MODE_ISDC:
            assert st["vcycles"] == st["sweeps"] * (cfg.M - 1) * cfg.L


def test_determinism(gpu):
    cfg, u0, G = synth.problem_inputs(2, 0, 255)
    outs = []
    for _ in range(2):
        h = make(gpu, cfg, G)
        h.set_initial(torch.from_numpy(u0).cuda(), 0)
        st = h.step()
        outs.append((h.solution(0).cpu().numpy(), st["res_hist"]))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_host_entry_points(gpu, ora):
    cfg, u0, G = synth.problem_inputs(1, 0)
    h = make(gpu, cfg)
    h.set_initial(u0, 0)               # host numpy -> isdc_set_initial_host
    h.step()
    out = h.solution_host(-1)
    ref, _ = ora.step(ora.Problem(cfg), u0, 0.0)
    assert np.array_equal(out, ref)


def test_errors(gpu):
    with pytest.raises(gpu.IsdcError):
        gpu.ISDC(2, 62, 3, 0.01, 1.0)          # n + 1 not a power of two
    with pytest.raises(gpu.IsdcError):
        gpu.ISDC(4, 63, 3, 0.01, 1.0)          # bad dimension
    with pytest.raises(gpu.IsdcError):
        gpu.ISDC(2, 63, 9, 0.01, 1.0)          # M unsupported
    with pytest.raises(gpu.IsdcError):
        gpu.ISDC(2, 63, 3, -0.01, 1.0)         # dt <= 0
    with pytest.raises(gpu.IsdcError):
        gpu.ISDC(2, 63, 3, 0.01, 1.0, fe=FE_FORCING, G=None) if False else gpu.ISDC(2, 63, 3, 0.01, 1.0, L=0)


# ------------------------------------------------------------ unweighted residual (NEXT f2)
@pytest.mark.parametrize("cid,n,mode", [(1, 63, MODE_ISDC), (2, 127, MODE_ISDC), (3, 255, MODE_ISDC),
                                        (1, 63, MODE_SDC), (2, 255, MODE_ISDC_CAPPED)])
def test_unweighted_residual_steps_bitwise(gpu, ora, cid, n, mode):
    """residual_kind 1: ||W^{-1} r~|| with W^{-1} by V-cycles on B_h -- every
    residual, count (sweeps, V-cycles, W-cycles) and the solution equal the oracle's bits."""
    cfg, u0, G = synth.problem_inputs(cid, 0, n)
    h = make(gpu, cfg, G, mode=mode, residual_kind=1, w_tol=1e-6, w_cap=50)
    prob = ora.Problem(cfg, G, mode=mode, res_kind=1, w_tol=1e-6, w_cap=50)
    h.set_initial(torch.from_numpy(u0).cuda(), 0)
    st = h.step()
    u_ref, st_ref = ora.step(prob, u0, 0.0)
    assert st["sweeps"] == st_ref["sweeps"] and st["vcycles"] == st_ref["vcycles"]
    assert st["wcycles"] == st_ref["wcycles"] and st["wcycles"] > 0
    assert np.array_equal(st["res_hist"], st_ref["res_hist"])
    assert np.array_equal(h.solution(0).cpu().numpy(), u_ref)


@pytest.mark.parametrize("n", [63, 127])
def test_config5_whole_trajectory_bitwise(gpu, ora, n):
    """All five steps of config 5's trajectory (the one bench.py times) at reduced size, step by
    step against the oracle: counts, residual bits and the end value of every step.  (At 511^3 the
    stored oracle results cover the same five steps, tests/test_gpu_fullsize.py.)"""
    cfg, u0, G = synth.problem_inputs(5, 0, n)
    assert cfg.steps == 5
    h = make(gpu, cfg, G, mode=MODE_ISDC)
    prob = ora.Problem(cfg, G, mode=MODE_ISDC)
    h.set_initial(torch.from_numpy(u0).cuda(), 0)
    u_ref = u0.copy()
    for s in range(cfg.steps):
        st = h.step()
        u_ref, st_ref = ora.step(prob, u_ref, float(s) * cfg.dt)
        assert st["sweeps"] == st_ref["sweeps"] and st["vcycles"] == st_ref["vcycles"], s
        assert st["converged"] == st_ref["converged"]
        assert np.array_equal(st["node_cycles"], st_ref["node_cycles"])
        assert np.array_equal(st["res_hist"], st_ref["res_hist"]), s
        assert np.array_equal(h.solution(0).cpu().numpy(), u_ref), s


# ------------------------------------------------ alternative execution paths (same bits)
@pytest.mark.parametrize("env,mode", [({"ISDC_DEVICE_SDC": "0"}, MODE_SDC), ({"ISDC_DEVICE_SDC": "0"}, MODE_ISDC_CAPPED),
                                      ({"ISDC_NO_GRAPHS": "1"}, MODE_ISDC), ({"ISDC_NO_GRAPHS": "1"}, MODE_SDC),
                                      ({"ISDC_GENERIC_KERNELS": "1"}, MODE_ISDC), ({"ISDC_FOLDS": "0"}, MODE_ISDC),
                                      ({"ISDC_STEP_GRAPH": "0"}, MODE_ISDC), ({"ISDC_TAIL_FUSE": "0"}, MODE_ISDC),
                                      ({"ISDC_STREAM2D": "0"}, MODE_ISDC), ({"ISDC_FUSE2D": "0"}, MODE_ISDC),
                                      ({"ISDC_FAST3D_MASK": "0x1"}, MODE_ISDC), ({"ISDC_FAST3D_MASK": "0x6"}, MODE_ISDC),
                                      ({"ISDC_FAST3D_MASK": "0x18"}, MODE_ISDC), ({"ISDC_WS3D": "0"}, MODE_ISDC),
                                      ({"ISDC_FUSE3D": "1"}, MODE_ISDC), ({"ISDC_WS3D_MIN": "31"}, MODE_ISDC),
                                      ({"ISDC_RESID2D_TMA": "0"}, MODE_ISDC), ({"ISDC_CTAIL": "0"}, MODE_ISDC),
                                      ({"ISDC_CTAIL": "0"}, MODE_SDC), ({"ISDC_CTAIL": "2"}, MODE_ISDC),
                                      ({"ISDC_CTAIL": "2"}, MODE_SDC),
                                      ({"ISDC_RHS128": "1"}, MODE_ISDC), ({"ISDC_SHIFT3D": "0"}, MODE_ISDC), ({"ISDC_WS_NS": "6"}, MODE_ISDC),
                                      ({"ISDC_WS_NS": "10"}, MODE_ISDC)])
def test_execution_paths_bitwise(gpu, ora, monkeypatch, env, mode):
    """Host-side node-solve tests, un-captured sweeps, sweep-by-sweep steps, the generic kernels, the
    fold-free RHS, the unfused tail, the tile-based 2D RHS / residual, the unfused 2D transfers and
    every subset of the fast 3D kernels (mask bits: 1 smoother, 2 restriction, 4 prolongation, 8 RHS,
    16 residual, 32 four-node residual), the 4 x 8 single-group 3D smoother, the 3D prolongation fused
    into the warp-specialised post-smoother and the warp-specialised smoother on 31^3, and the coarse
    levels without the cluster tail (ISDC_CTAIL=0) or with it in 2D too (ISDC_CTAIL=2), and the fold
    RHS with 128-bit loads (ISDC_RHS128=1) produce the
    oracle's bits too (the environment is read when the handle is created)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for cid, n in ((2, 127), (4, 31), (5, 63)):
        cfg, u0, G = synth.problem_inputs(cid, 0, n)
        h = make(gpu, cfg, G, mode=mode)
        h.set_initial(torch.from_numpy(u0).cuda(), 0)
        st = h.step()
        u_ref, st_ref = ora.step(ora.Problem(cfg, G, mode=mode), u0, 0.0)
        assert st["sweeps"] == st_ref["sweeps"] and st["vcycles"] == st_ref["vcycles"]
        assert np.array_equal(st["node_cycles"], st_ref["node_cycles"])
        assert np.array_equal(st["res_hist"], st_ref["res_hist"])
        assert np.array_equal(h.solution(0).cpu().numpy(), u_ref)


# --------------------------------------------------------------------------- edge cases
EDGE = [  # (dim, n, M, L, nu1, nu2, guess, mode, fe)
    (2, 3, 2, 2, 2, 2, 0, MODE_ISDC, FE_NONE),         # a single level: the exact coarse solve only
    (3, 3, 3, 1, 2, 2, 0, MODE_SDC, FE_NONE),
    (2, 7, 8, 1, 1, 0, 0, MODE_ISDC, FE_CUBIC),        # M = 8 (the maximum), L = 1, V(1,0)
    (2, 63, 2, 3, 0, 2, 0, MODE_ISDC, FE_FORCING),     # M = 2, V(0,2): no pre-smoothing
    (2, 127, 5, 2, 3, 1, 0, MODE_ISDC, FE_NONE),       # V(3,1): an extra unfused pre-sweep on the fast levels
    (3, 31, 3, 2, 1, 3, 0, MODE_ISDC, FE_ADVECTION),   # odd sweep counts in 3D
    (2, 127, 3, 2, 2, 2, 2, MODE_SDC, FE_NONE),        # initial guess u_m^{k+1} (P:187 ablation)
    (2, 63, 3, 2, 2, 2, 1, MODE_SDC, FE_NONE),         # zero initial guess
    (3, 15, 3, 2, 2, 2, 2, MODE_SDC, FE_NONE),
]


@pytest.mark.parametrize("dim,n,M,L,nu1,nu2,guess,mode,fe", EDGE)
def test_edge_cases_bitwise(gpu, ora, dim, n, M, L, nu1, nu2, guess, mode, fe):
    cfg = synth.Config(0, dim, n, M, 0.01, 0.7, fe, fe_a=(1.0, -0.5, 0.25), L=L, nu1=nu1, nu2=nu2,
                       sweep_tol=1e-9, max_sweeps=60)
    G = synth.forcing_field(n, dim) if fe == FE_FORCING else None
    u0 = synth.random_field(n, dim, 77)
    h = make(gpu, cfg, G, mode=mode, guess=guess)
    h.set_initial(torch.from_numpy(u0).cuda(), 0)
    prob = ora.Problem(cfg, G, mode=mode, guess=guess)
    u_ref = u0.copy()
    for s in range(2):
        st = h.step()
        u_ref, st_ref = ora.step(prob, u_ref, float(s) * cfg.dt)
        assert st["sweeps"] == st_ref["sweeps"] and st["vcycles"] == st_ref["vcycles"]
        assert st["converged"] == st_ref["converged"]
        assert np.array_equal(st["node_cycles"], st_ref["node_cycles"])
        assert np.array_equal(st["res_hist"], st_ref["res_hist"])
        assert np.array_equal(h.solution(0).cpu().numpy(), u_ref)


# ------------------------------------------------------------- non-finite detection (errors)
@pytest.mark.parametrize("cid,n,mode,bad", [(1, 63, MODE_ISDC, np.nan), (2, 127, MODE_ISDC, np.inf),
                                            (3, 127, MODE_SDC, np.nan), (4, 31, MODE_ISDC, -np.inf),
                                            (5, 31, MODE_ISDC, np.nan), (2, 127, MODE_ISDC_CAPPED, np.nan)])
def test_nonfinite_input_raises(gpu, cid, n, mode, bad):
    """A NaN / Inf in u0 propagates into the residual (or the SDC defect test) and the step returns
    ISDC_ERR_NONFINITE (include/isdc.h) instead of a silent result, on every execution path: the
    fixed-sweep step graph (cfg 1), the tolerance-stopped step graph (cfgs 2, 4, 5), the device SDC /
    capped node-solve loop (cfg 3 SDC, cfg 2 capped)."""
    cfg, u0, G = synth.problem_inputs(cid, 0, n)
    u0 = u0.copy()
    u0[(n // 3,) * cfg.dim] = bad
    h = make(gpu, cfg, G, mode=mode)
    h.set_initial(torch.from_numpy(u0).cuda(), 0)
    with pytest.raises(gpu.IsdcError) as ei:
        h.step()
    assert ei.value.status == 4, str(ei.value)
    # residual_norm on the spread state of a poisoned u0 reports it too
    h.set_initial(torch.from_numpy(u0).cuda(), 0)
    with pytest.raises(gpu.IsdcError) as ei:
        h.residual()
    assert ei.value.status == 4


def test_binding_rejects_bad_shapes(gpu):
    cfg = synth.Config(0, 2, 63, 3, 0.01, 1.0, FE_NONE)
    h = make(gpu, cfg)
    b = synth.random_field(63, 2, 1)
    with pytest.raises(ValueError):
        h.vcycle(0, b, torch.zeros(31, 31, dtype=torch.float64, device="cuda"))   # would be an OOB write
    with pytest.raises(ValueError):
        h.set_initial(torch.zeros(62, 63, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        h.solution(0, out=torch.zeros(63, 64, dtype=torch.float64, device="cuda"))


def test_handle_on_side_stream_matches_default(gpu, ora):
    """A handle bound to a non-default stream (temporaries recorded on it) gives the same bits."""
    cfg, u0, G = synth.problem_inputs(2, 0, 127)
    side = torch.cuda.Stream()
    h = gpu.ISDC.from_config(cfg, None, mode=MODE_ISDC, stream=side)
    h.set_initial(torch.from_numpy(u0).cuda(), 0)
    st = h.step()
    u_ref, st_ref = ora.step(ora.Problem(cfg, G), u0, 0.0)
    assert st["sweeps"] == st_ref["sweeps"]
    assert np.array_equal(h.solution(0).cpu().numpy(), u_ref)


def test_handles_with_different_tail_sizes_coexist(gpu, ora):
    """creating a small 3D handle must not break a larger one created earlier (the
    kernels' shared-memory limits are set once per device to the maximum)."""
    cfg_big, u_big, _ = synth.problem_inputs(4, 0, 63)
    big = make(gpu, cfg_big)
    small = make(gpu, synth.Config(0, 3, 7, 3, 0.01, 1.0, FE_NONE))
    small.set_initial(torch.from_numpy(synth.random_field(7, 3, 3)).cuda(), 0)
    small.step()
    big.set_initial(torch.from_numpy(u_big).cuda(), 0)
    st = big.step()
    u_ref, st_ref = ora.step(ora.Problem(cfg_big), u_big, 0.0)
    assert st["sweeps"] == st_ref["sweeps"]
    assert np.array_equal(big.solution(0).cpu().numpy(), u_ref)
