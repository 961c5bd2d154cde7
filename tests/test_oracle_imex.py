"""Per-sweep pins of the oracle's IMEX explicit term and of its V-cycle schedule.

These close the two places round 1 left unpinned (Weak 1):

* The explicit difference dt_m [f^E(u_m^{k+1}) - f^E(u_m^k)] of the semi-implicit sweep
  (Eq. 4; weighted form P:68-76, Eq. 5).  It vanishes at every fixed point, so only a
  comparison after a FIXED number of sweeps, before convergence, can see it.  A periodic plane
  wave exp(i pi k.x) is an eigenvector of the compact pair (B_h, L_h) AND of the CD4 advection
  operator, so on one mode the whole PDE sweep reduces to the complex scalar IMEX-SDC recursion
  with lam_I = nu lam_L / lam_B and lam_E = the CD4 symbol -- an independent restatement of Eq. (4)
  per mode.  A sign flip of the explicit difference, or evaluating it at node m+1, changes the
  K-sweep iterate by O(dt |lam_E|) and fails these tests; the negative controls below show the
  mutated recursions are far outside the tolerance.

* The V-cycle schedule ("V-cycles"; components B:configs[1], R11-R14).  One
  oracle V(nu1, nu2) cycle is an affine map u -> M u + (I - M) A^{-1} b whose error propagator is
  composed here in numpy from the separately pinned pieces (dense node operator A, Jacobi
  I - omega D^{-1} A, full weighting R, prolongation P = 2^d R^T, rediscretised coarse operators,
  exact coarsest solve):
      M_l = J_l^nu2 (I - P (I - M_{l+1}) A_{l+1}^{-1} R A_l) J_l^nu1,    M_coarsest = 0.
  A V(1,1) cycle, swapped pre/post counts or a missing coarse correction give a different map;
  the negative control checks that the swapped schedule is detected.
"""
import math

import numpy as np
import pytest

import synth
from synth import BC_DIRICHLET, BC_PERIODIC, FE_ADVECTION, FE_FORCING, MODE_SDC, Config


# --------------------------------------------------------------------------------------------
# closed-form symbols on a single mode
# --------------------------------------------------------------------------------------------
def compact_symbols(ks, h):
    """Compact pair on exp(i pi k.x) (periodic) or prod sin(k pi x) (Dirichlet):
    c_a = cos(k_a pi h); 2D lam_L = (-20 + 8 c1 + 8 c2 + 4 c1 c2)/(6 h^2), lam_B = (8 + 2 c1 + 2 c2)/12."""
    c = [math.cos(k * math.pi * h) for k in ks]
    assert len(ks) == 2
    return (-20 + 8 * c[0] + 8 * c[1] + 4 * c[0] * c[1]) / (6 * h * h), (8 + 2 * c[0] + 2 * c[1]) / 12


def cd4_symbol(ks, a, h):
    """f^E = -a.grad u with CD4 differences (B:configs[5]) on exp(i theta), theta = pi k.x:
    (8 (e^{i phi} - e^{-i phi}) - (e^{2 i phi} - e^{-2 i phi}))/(12 h) = i (8 sin phi - sin 2 phi)/(6 h),
    phi = k_a pi h, so lam_E = -i sum_a a_a (8 sin phi_a - sin 2 phi_a)/(6 h)."""
    s = sum(aa * (8 * math.sin(k * math.pi * h) - math.sin(2 * k * math.pi * h)) / (6 * h) for k, aa in zip(ks, a))
    return -1j * s


def scalar_imex_sdc(lamI, lamE, dt, M, K, tables, u0=1.0 + 0j, g=None, variant="paper"):
    """K semi-implicit SDC sweeps (Eq. 4) on u' = lamI u + lamE u + g(t), exact implicit
    solves, spread initial iterate; returns the node values after K sweeps.

        u_{m+1}^{k+1} = u_m^{k+1} + dt_m [lamI (u_{m+1}^{k+1} - u_{m+1}^k)]
                        + dt_m [f^E(u_m^{k+1}) - f^E(u_m^k)] + dt sum_j s_{m,j} f(u_j^k)

    variant "flip" / "at_m1": deliberately wrong explicit difference (negative controls)."""
    tau, Q, S, dtau = tables
    fE = lambda x, j: lamE * x + (g[j] if g is not None else 0.0)
    u = np.full(M, u0, dtype=complex)
    for _ in range(K):
        un = np.empty(M, dtype=complex)
        un[0] = u0
        for m in range(M - 1):
            dtm = dt * dtau[m]
            if variant == "paper":
                expl = fE(un[m], m) - fE(u[m], m)
            elif variant == "flip":
                expl = fE(u[m], m) - fE(un[m], m)
            else:   # evaluated at node m+1 (old iterate only: an implicit-looking misreading)
                expl = fE(u[m + 1], m + 1) - fE(u[m], m)
            quad = sum(S[m, j] * (lamI * u[j] + fE(u[j], j)) for j in range(M))
            un[m + 1] = (un[m] - dtm * lamI * u[m + 1] + dtm * expl + dt * quad) / (1 - dtm * lamI)
        u = un
    return u


def plane_wave(n, ks):
    """cos(theta), sin(theta), theta = pi (k1 x + k2 y) on the periodic grid x_i = -1 + i h."""
    x = synth.grid_x_periodic(n)
    th = math.pi * (ks[0] * x[None, :] + ks[1] * x[:, None])
    return np.cos(th), np.sin(th)


def advection_cfg(n, M, dt, nu, a, K):
    return Config(0, 2, n, M, dt, nu, FE_ADVECTION, fe_a=(a[0], a[1], 0.0), fixed_sweeps=K,
                  inner_tol=1e-15, inner_cap=300, bc=BC_PERIODIC)


# --------------------------------------------------------------------------------------------
# IMEX explicit term, sweep by sweep
# --------------------------------------------------------------------------------------------
CASES = [((1, 2), 3, 0.02, 0.5, (4.0, -3.0)), ((2, 1), 5, 0.02, 0.2, (6.0, 2.5)), ((3, 1), 5, 0.05, 1.0, (-5.0, 4.0))]


@pytest.mark.parametrize("ks,M,dt,nu,a", CASES)
@pytest.mark.parametrize("K", [1, 2, 3, 4])
def test_imex_sweeps_match_scalar_recursion(ora, ks, M, dt, nu, a, K):
    """The oracle's K-sweep iterate on a periodic plane wave equals the scalar IMEX-SDC recursion
    (Eq. 4) with lam_I = nu lam_L/lam_B and lam_E = the CD4 symbol, at atol 1e-12."""
    n = 16
    h = 2.0 / n
    c, s = plane_wave(n, ks)
    cfg = advection_cfg(n, M, dt, nu, a, K)
    u, st = ora.step(ora.Problem(cfg, mode=MODE_SDC), c, 0.0)
    assert st["sweeps"] == K
    lL, lB = compact_symbols(ks, h)
    uh = scalar_imex_sdc(nu * lL / lB, cd4_symbol(ks, a, h), dt, M, K, ora.tables(M))[-1]
    np.testing.assert_allclose(u, uh.real * c - uh.imag * s, rtol=0, atol=1e-12)
    # negative controls: both misreadings of the explicit difference move the iterate far outside
    # the tolerance (so a mutated oracle could not pass this test)
    if K < 4 or M == 3:
        for variant in ("flip", "at_m1"):
            ub = scalar_imex_sdc(nu * lL / lB, cd4_symbol(ks, a, h), dt, M, K, ora.tables(M), variant=variant)[-1]
            assert np.abs(u - (ub.real * c - ub.imag * s)).max() > 1e-6, variant


def test_imex_every_node_matches(ora):
    """All nodes (not only the end value) after 2 sweeps, through oracle.sweep."""
    n, ks, M, dt, nu, a = 16, (1, 3), 5, 0.03, 0.3, (3.0, 5.0)
    h = 2.0 / n
    c, s = plane_wave(n, ks)
    cfg = advection_cfg(n, M, dt, nu, a, 2)
    prob = ora.Problem(cfg, mode=MODE_SDC)
    state = [c] * M
    for _ in range(2):
        state, _ = ora.sweep(prob, 0.0, state)
    lL, lB = compact_symbols(ks, h)
    uh = scalar_imex_sdc(nu * lL / lB, cd4_symbol(ks, a, h), dt, M, 2, ora.tables(M))
    for m in range(M):
        np.testing.assert_allclose(state[m], uh[m].real * c - uh[m].imag * s, rtol=0, atol=1e-12)


@pytest.mark.parametrize("K", [1, 2, 3])
def test_forcing_sweeps_match_scalar_recursion(ora, K):
    """Config-3 type forcing f^E = G cos t on Dirichlet mode (2,2) (G is that mode): the K-sweep
    iterate equals scalar_imex_sdc with lam_E = 0 and g_j = cos(t_j) (the explicit difference
    G cos t_m - G cos t_m vanishes identically, reading R20)."""
    n, M, dt, nu, amp = 15, 5, 0.01, 0.1, 0.7
    h = 1.0 / (n + 1)
    G = synth.forcing_field(n)
    t_n = 2 * dt
    cfg = Config(0, 2, n, M, dt, nu, FE_FORCING, fixed_sweeps=K, inner_tol=1e-15, inner_cap=300)
    u, st = ora.step(ora.Problem(cfg, G, mode=MODE_SDC), amp * G, t_n)
    lL, lB = compact_symbols((2, 2), h)
    tau = ora.tables(M)[0]
    g = np.array([math.cos(t_n + dt * t) for t in tau])
    uh = scalar_imex_sdc(nu * lL / lB, 0.0, dt, M, K, ora.tables(M), u0=amp, g=g)[-1]
    np.testing.assert_allclose(u, uh.real * G, rtol=0, atol=1e-12)
    # dropping the forcing's quadrature term fails
    un = scalar_imex_sdc(nu * lL / lB, 0.0, dt, M, K, ora.tables(M), u0=amp)[-1]
    assert np.abs(u - un.real * G).max() > 1e-6


def test_imex_order_per_sweep(ora):
    """With f^E != 0 every IMEX sweep also raises the order by one (Minion 2003): the error
    after K sweeps per step against the semi-discrete exact solution exp(T (lam_I + lam_E)) has
    observed order K +- 0.3 for K = 1..4 (M = 5, a single advected and diffused plane wave)."""
    n, ks, nu, a, T, M = 16, (1, 1), 0.05, (2.0, 1.0), 0.1, 5
    h = 2.0 / n
    c, s = plane_wave(n, ks)
    lL, lB = compact_symbols(ks, h)
    ex = np.exp(T * (nu * lL / lB + cd4_symbol(ks, a, h)))
    exact = ex.real * c - ex.imag * s
    for K in (1, 2, 3, 4):
        errs = []
        for nsteps in (4, 8, 16):
            dt = T / nsteps
            prob = ora.Problem(advection_cfg(n, M, dt, nu, a, K), mode=MODE_SDC)
            u = c.copy()
            for st in range(nsteps):
                u, _ = ora.step(prob, u, float(st) * dt)
            errs.append(np.abs(u - exact).max())
        orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
        assert all(abs(o - K) < 0.3 for o in orders), (K, orders, errs)


# --------------------------------------------------------------------------------------------
# V-cycle schedule against the composed dense iteration operator
# --------------------------------------------------------------------------------------------
_DENSE = {}


def dense_level(ora, dim, n, gamma):
    """Dense node operator A = S_l (pinned by its Fourier symbols, test_oracle_stencils) and dense
    full weighting R (pinned by its symbol and the adjoint identity, test_oracle_mg) of level n."""
    key = (dim, n, gamma)
    if key not in _DENSE:
        P = n ** dim
        I = np.eye(P)
        A = np.stack([ora.apply_S(I[i].reshape((n,) * dim), gamma).ravel() for i in range(P)], axis=1)
        R = None
        if n > 3:
            R = np.stack([ora.restrict(I[i].reshape((n,) * dim)).ravel() for i in range(P)], axis=1)
        _DENSE[key] = (A, R)
    return _DENSE[key]


def apply_propagator(ora, dim, n, gamma, nu1, nu2, e, omega=0.8):
    """M_l e for the error propagator of one V(nu1, nu2) cycle on level n (recursive; the coarsest
    level n = 3 is solved exactly, M = 0):
        M_l = J^nu2 (I - P (I - M_{l+1}) A_{l+1}^{-1} R A_l) J^nu1,  J = I - omega D^{-1} A,  P = 2^d R^T."""
    A, R = dense_level(ora, dim, n, gamma)
    if n == 3:
        return np.zeros_like(e)
    d = np.diag(A)
    for _ in range(nu1):
        e = e - omega * (A @ e) / d
    nc = (n - 1) // 2
    Ac, _ = dense_level(ora, dim, nc, gamma)
    v = np.linalg.solve(Ac, R @ (A @ e))
    v = v - apply_propagator(ora, dim, nc, gamma, nu1, nu2, v, omega)
    e = e - (2 ** dim) * (R.T @ v)
    for _ in range(nu2):
        e = e - omega * (A @ e) / d
    return e


@pytest.mark.parametrize("dim,n,gamma", [(2, 7, 0.004), (2, 15, 0.03), (3, 7, 0.002), (3, 15, 0.0007)])
@pytest.mark.parametrize("nu1,nu2", [(2, 2), (1, 0), (0, 2), (3, 1)])
def test_vcycle_equals_composed_operator(ora, dim, n, gamma, nu1, nu2):
    """One oracle V(nu1,nu2) cycle = x + M (u - x), x = A^{-1} b, M composed from the pinned pieces."""
    A, _ = dense_level(ora, dim, n, gamma)
    b = synth.random_field(n, dim, 11)
    u = synth.random_field(n, dim, 12)
    x = np.linalg.solve(A, b.ravel())
    expect = x + apply_propagator(ora, dim, n, gamma, nu1, nu2, u.ravel() - x)
    got = ora.vcycle(b, u, gamma, nu1=nu1, nu2=nu2).ravel()
    np.testing.assert_allclose(got, expect, rtol=1e-13, atol=1e-13 * np.abs(expect).max())
    # negative controls: the swapped schedule and V(1,1) are different maps
    for w1, w2 in {(nu2, nu1), (1, 1)} - {(nu1, nu2)}:
        wrong = x + apply_propagator(ora, dim, n, gamma, w1, w2, u.ravel() - x)
        assert np.abs(got - wrong).max() > 1e-6 * np.abs(expect).max(), (w1, w2)
