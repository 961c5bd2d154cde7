"""Pins of the oracle's MLSDC with ISDC sweeps (NEXT f4; reading R32).

Independent references:
* 4th-order interpolation (the coarse-correction prolongation P4): exact on cubic polynomials away
  from the boundary and on odd-symmetric cubics at it (the odd reflection), error ratio ~16 per
  halving of h on a smooth function (bilinear: ~4), injection at the coincident points;
* the fixed point: a converged MLSDC step equals the FINE collocation solution (closed form per
  sine mode, (I - zQ)^{-1} 1 / diagonal Pade) -- which is what the FAS correction guarantees;
* FAS consistency: one coarse correction leaves the exact fine collocation solution unchanged, while
  the same correction WITHOUT the FAS term moves it (negative control);
* no coarse sweep = plain ISDC, bit for bit (the restriction / correction plumbing adds exact zeros);
* an independent numpy re-composition of the MLSDC iteration from separately pinned primitives
  (oracle.rhs, oracle.vcycle, apply_B / apply_L, restrict, inject, prolong4_add) reproduces the C
  iteration's residual history and solution;
* behaviour: with exact node solves MLSDC needs fewer fine sweeps than SDC on the paper's heat
  problem -- the point of moving work to the coarse level.
"""
import math

import numpy as np
import pytest

import synth
from synth import Config, FE_ADVECTION, FE_CUBIC, FE_FORCING, FE_NONE, MODE_ISDC


def grid(n):
    return synth.grid_x(n)


# --------------------------------------------------------------------------------- P4 interpolation
def test_prolong4_injection_and_cubic_exactness(ora):
    nc = 15
    nf = 2 * nc + 1
    e = synth.random_field(nc, 2, 3)
    Pe = ora.prolong4_add(e, np.zeros((nf, nf)))
    np.testing.assert_array_equal(Pe[1::2, 1::2], e)          # coincident points are injected
    xc, xf = grid(nc), grid(nf)
    # interior: any cubic in x times any cubic in y is reproduced where the 4-point stencils stay inside
    g = lambda x: 1.0 - 2.0 * x + 3.0 * x ** 2 - 5.0 * x ** 3
    h = lambda y: 0.5 + y - 4.0 * y ** 3
    fc = np.outer(h(xc), g(xc))
    ff = np.outer(h(xf), g(xf))
    Pf = ora.prolong4_add(fc, np.zeros((nf, nf)))
    sl = slice(3, nf - 3)
    np.testing.assert_allclose(Pf[sl, sl], ff[sl, sl], atol=1e-13)
    # boundary: the odd reflection is exact for cubics odd about the boundary point (x = 0 and x = 1)
    g0 = lambda x: x - 2.0 * x ** 3                 # odd about x = 0
    g1 = lambda x: (1 - x) - 3.0 * (1 - x) ** 3     # odd about x = 1
    for gg, side in ((g0, slice(0, nf // 2)), (g1, slice(nf // 2, nf))):
        fc = np.outer(np.ones(nc), gg(xc))
        ff = np.outer(np.ones(nf), gg(xf))
        Pf = ora.prolong4_add(fc, np.zeros((nf, nf)))
        np.testing.assert_allclose(Pf[nf // 2, side], ff[nf // 2, side], atol=1e-13)


def test_prolong4_order_and_3d(ora):
    """Interpolating a smooth function that is odd about the boundary (as solutions of the Dirichlet
    heat problem are: u = 0 and Delta u = u_t / nu = 0 there, so every even derivative vanishes):
    error ratio ~16 per halving (bilinear ~4); 3D too."""
    f = lambda x, y: np.sin(math.pi * x) * np.sin(2 * math.pi * y) + 0.5 * np.sin(3 * math.pi * x) * np.sin(math.pi * y)
    errs4, errs2 = [], []
    for nc in (15, 31, 63):
        nf = 2 * nc + 1
        xc, xf = grid(nc), grid(nf)
        fc = f(xc[None, :], xc[:, None])
        ff = f(xf[None, :], xf[:, None])
        errs4.append(np.abs(ora.prolong4_add(fc, np.zeros((nf, nf))) - ff).max())
        errs2.append(np.abs(ora.prolong_add(fc, np.zeros((nf, nf))) - ff).max())
    r4 = [errs4[i] / errs4[i + 1] for i in range(2)]
    r2 = [errs2[i] / errs2[i + 1] for i in range(2)]
    assert all(12 < r < 20 for r in r4), r4
    assert all(3 < r < 5 for r in r2), r2
    # 3D: separable cubic reproduced in the interior, coincident points injected
    nc = 7
    nf = 2 * nc + 1
    xc, xf = grid(nc), grid(nf)
    cub = lambda x: 0.3 + x - x ** 3
    fc = cub(xc)[:, None, None] * cub(xc)[None, :, None] * cub(xc)[None, None, :]
    ff = cub(xf)[:, None, None] * cub(xf)[None, :, None] * cub(xf)[None, None, :]
    Pf = ora.prolong4_add(fc, np.zeros((nf,) * 3))
    np.testing.assert_array_equal(Pf[1::2, 1::2, 1::2], fc)
    sl = slice(3, nf - 3)
    np.testing.assert_allclose(Pf[sl, sl, sl], ff[sl, sl, sl], atol=1e-13)


# ------------------------------------------------------------------------------------- MLSDC
def sym(ks, n):
    h = 1.0 / (n + 1)
    c = [math.cos(k * math.pi * h) for k in ks]
    if len(ks) == 2:
        return (-20 + 8 * c[0] + 8 * c[1] + 4 * c[0] * c[1]) / (6 * h * h), (8 + 2 * c[0] + 2 * c[1]) / 12
    s = sum(c); pr = c[0] * c[1] + c[0] * c[2] + c[1] * c[2]
    return (-24 + 4 * s + 4 * pr) / (6 * h * h), (6 + 2 * s) / 12


@pytest.mark.parametrize("ks,M,nu,cs", [((1, 2), 3, 1.0, 1), ((2, 1), 5, 10.0, 2), ((1, 1, 2), 3, 1.0, 1)])
def test_mlsdc_converges_to_fine_collocation_solution(ora, ks, M, nu, cs):
    n = 15
    dim = len(ks)
    cfg = Config(0, dim, n, M, 0.02, nu, FE_NONE, sweep_tol=1e-13, max_sweeps=200)
    u0 = synth.sine_mode(n, ks)
    u, st = ora.mlsdc_step(ora.Problem(cfg), u0, 0.0, coarse_sweeps=cs)
    assert st["converged"] and st["coarse_vcycles"] > 0
    lL, lB = sym(ks, n)
    z = cfg.dt * nu * lL / lB
    tau, Q, S, dtau = ora.tables(M)
    coll = np.linalg.solve(np.eye(M) - z * Q, np.ones(M))
    np.testing.assert_allclose(u, coll[-1] * u0, atol=1e-12)


def test_fas_consistency_and_negative_control(ora):
    """At the fine collocation solution u* the FAS-corrected coarse problem is solved by R u*, so the
    correction leaves u* unchanged (to rounding); dropping the FAS term moves u* by the difference
    between the coarse and fine collocation solutions."""
    n, M, nu, ks = 31, 5, 5.0, (2, 3)
    cfg = Config(0, 2, n, M, 0.01, nu, FE_NONE)
    phi = synth.sine_mode(n, ks)
    lL, lB = sym(ks, n)
    tau, Q, S, dtau = ora.tables(M)
    coll = np.linalg.solve(np.eye(M) - cfg.dt * nu * lL / lB * Q, np.ones(M))
    ustar = [c * phi for c in coll]
    prob = ora.Problem(cfg)
    for cs in (1, 4):
        u, cv = ora.mlsdc_correction(prob, 0.0, ustar, coarse_sweeps=cs)
        assert cv == cs * (M - 1) * cfg.L
        for j in range(M):
            np.testing.assert_allclose(u[j], ustar[j], atol=1e-13)
        u_nofas, _ = ora.mlsdc_correction(prob, 0.0, ustar, coarse_sweeps=cs, fas=False)
        assert max(np.abs(u_nofas[j] - ustar[j]).max() for j in range(M)) > 1e-8


@pytest.mark.parametrize("fe,dim", [(FE_NONE, 2), (FE_FORCING, 2), (FE_ADVECTION, 3)])
def test_no_coarse_sweep_is_plain_isdc(ora, fe, dim):
    n = 15
    cfg = Config(0, dim, n, 5, 0.01, 0.5, fe, fe_a=(1.0, -0.5, 0.25), fixed_sweeps=4)
    G = synth.forcing_field(n, dim) if fe == FE_FORCING else None
    u0 = synth.random_field(n, dim, 5)
    prob = ora.Problem(cfg, G)
    u1, s1 = ora.step(prob, u0, 0.02)
    u2, s2 = ora.mlsdc_step(prob, u0, 0.02, coarse_sweeps=0)
    assert np.array_equal(u1, u2) and np.array_equal(s1["res_hist"], s2["res_hist"])
    assert s2["coarse_vcycles"] == 0


def numpy_mlsdc(ora, cfg, u0, coarse_sweeps, nsweeps):
    """Re-composition of the MLSDC iteration (R32) from separately pinned oracle primitives; f^E = 0."""
    M, n, nu, dt = cfg.M, cfg.n, cfg.nu, cfg.dt
    nc = (n - 1) // 2
    tau, Q, S, dtau = ora.tables(M)

    def res_fields(u):
        return [None] + [ora.apply_B(u[m] - u[0]) - ora.apply_L(sum((nu * dt * Q[m, j]) * u[j] for j in range(M)))
                         for m in range(1, M)]

    def sweep(uold, nn, fas=None):
        prob = ora.Problem(Config(0, cfg.dim, nn, M, dt, nu, FE_NONE))
        unew = [uold[0]] + [None] * (M - 1)
        for m in range(M - 1):
            b = ora.rhs(prob, 0.0, m, uold, [unew[j] if unew[j] is not None else uold[j] for j in range(M)])
            if fas is not None:
                b = b + (fas[m + 1] - (0.0 if m == 0 else fas[m]))
            x = uold[m + 1].copy()
            for _ in range(cfg.L):
                x = ora.vcycle(b, x, nu * (dt * dtau[m]))
            unew[m + 1] = x
        return unew

    u, hist = [u0] * M, []
    for k in range(nsweeps):
        u = sweep(u, n)
        rf = res_fields(u)
        hist.append(max(np.abs(x).max() for x in rf[1:]))
        if k + 1 == nsweeps:
            break
        Ub = [ora.inject(x) for x in u]
        rH = res_fields(Ub)
        fas = [None] + [rH[m] - ora.restrict(rf[m]) for m in range(1, M)]
        U = [x.copy() for x in Ub]
        for _ in range(coarse_sweeps):
            U = sweep(U, nc, fas)
        u = [u[0]] + [ora.prolong4_add(U[j] - Ub[j], u[j]) for j in range(1, M)]
    return u[-1], np.array(hist)


@pytest.mark.parametrize("M,cs", [(3, 1), (5, 2)])
def test_mlsdc_matches_recomposition_from_pinned_primitives(ora, M, cs):
    n, K = 31, 4
    cfg = Config(0, 2, n, M, 0.005, 3.0, FE_NONE, fixed_sweeps=K)
    u0 = synth.initial_condition(1, 0, n)
    u, st = ora.mlsdc_step(ora.Problem(cfg), u0, 0.0, coarse_sweeps=cs)
    u_ref, hist = numpy_mlsdc(ora, cfg, u0, cs, K)
    np.testing.assert_allclose(st["res_hist"], hist, rtol=1e-12)
    np.testing.assert_allclose(u, u_ref, atol=1e-13 * np.abs(u_ref).max())


def test_mlsdc_saves_fine_sweeps_with_exact_solves(ora):
    """MLSDC shifts work to the coarse level.  With exact node solves on both levels (SDC
    limit, here L = 30 V-cycles) it needs fewer FINE sweeps than single-level SDC on the paper's heat
    problem (u0 = sin(pi x) sin(pi y), dt = 1e-3, tol 5e-8)."""
    n = 63
    u0 = synth.sine_mode(n, (1, 1))
    fewer = 0
    for nu, M in ((1.0, 5), (10.0, 5), (1.0, 3)):
        cfg = Config(0, 2, n, M, 0.001, nu, FE_NONE, sweep_tol=5e-8, max_sweeps=60, L=30)
        _, s1 = ora.step(ora.Problem(cfg), u0, 0.0)
        _, s2 = ora.mlsdc_step(ora.Problem(cfg), u0, 0.0, coarse_sweeps=1)
        assert s1["converged"] and s2["converged"]
        assert s2["sweeps"] <= s1["sweeps"]
        fewer += s2["sweeps"] < s1["sweeps"]
    assert fewer >= 2


def test_mlsdc_nonlinear_fixed_point(ora):
    """Allen-Cahn f^E = u - u^3: the converged MLSDC step equals the converged single-level ISDC step
    (itself pinned to Newton + dense LU of the collocation system, test_oracle_sdc) within 10 tol."""
    n = 15
    cfg = Config(0, 2, n, 5, 0.05, 0.05, FE_CUBIC, sweep_tol=1e-12, max_sweeps=200)
    u0 = 0.8 * synth.random_field(n, 2, 9)
    u1, s1 = ora.step(ora.Problem(cfg), u0, 0.0)
    u2, s2 = ora.mlsdc_step(ora.Problem(cfg), u0, 0.0, coarse_sweeps=1)
    assert s1["converged"] and s2["converged"]
    assert np.abs(u1 - u2).max() < 1e-11
