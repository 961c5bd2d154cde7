"""Pins of the oracle's periodic grid and WENO5 Burgers f^E (NEXT f3: P:94; reading R31).

References independent of the oracle: the linear-weight limit of WENO5 (the fixed 5-point upwind
formula (2, -13, 47, 27, -3)/60), its non-oscillatory behaviour on a step, fifth-order convergence
to the analytic -u(u_x + u_y), exact invariants (constants, conservation, translation and axis
symmetry), the closed-form Fourier symbols of the periodic compact pair, the adjointness of full
weighting and bilinear prolongation, dense linear algebra for the node systems, and a Fourier
pseudo-spectral solution of the same PDE for a whole time step.
"""
import math

import numpy as np
import pytest

import synth
from synth import FE_BURGERS, MODE_ISDC, MODE_SDC


def mesh(n):
    x = synth.grid_x_periodic(n)
    return np.meshgrid(x, x)        # X varies along axis 1 (x fastest), Y along axis 0


# ------------------------------------------------------------------------------------ WENO5
def test_weno5_constant_and_linear_limit(ora):
    assert abs(ora.weno5(0.7, 0.7, 0.7, 0.7, 0.7) - 0.7) <= 4e-16
    rng = np.random.default_rng(5)
    for _ in range(20):
        a, b = rng.uniform(-2, 2, 2)
        v = a + b * np.arange(5.0)            # equal smoothness indicators -> linear weights
        lin = (2 * v[0] - 13 * v[1] + 47 * v[2] + 27 * v[3] - 3 * v[4]) / 60
        assert abs(ora.weno5(*v) - lin) <= 1e-14 * (1 + abs(lin))


def test_weno5_step_is_non_oscillatory(ora):
    # the only smooth candidate stencil dominates: value within (eps/beta)^2 of the upwind side
    assert abs(ora.weno5(0, 0, 0, 1, 1)) < 1e-10
    assert abs(ora.weno5(1, 1, 1, 0, 0) - 1) < 1e-10
    assert abs(ora.weno5(0, 0, 1, 1, 1) - 1) < 1e-10   # jump behind the face: upwind value 1
    # smooth data: 5th-order face value of a cell-point sampled function (point values here)
    f = lambda x: math.sin(x)                          # noqa: E731
    errs = []
    for h in (0.1, 0.05, 0.025):
        xs = [(-2 + s) * h for s in range(5)]
        lin = (2 * f(xs[0]) - 13 * f(xs[1]) + 47 * f(xs[2]) + 27 * f(xs[3]) - 3 * f(xs[4])) / 60
        errs.append(abs(ora.weno5(*[f(x) for x in xs]) - lin))
    assert errs[-1] < 1e-9


@pytest.mark.parametrize("dim", [2, 3])
def test_burgers_fe_fifth_order(ora, dim):
    """f^E -> -u (u_x + u_y [+ u_z]) at 5th order on a smooth periodic field (rates ~5.2-5.6)."""
    errs = []
    for n in ((32, 64, 128) if dim == 2 else (16, 32, 64)):
        x = synth.grid_x_periodic(n)
        if dim == 2:
            X, Y = np.meshgrid(x, x)
            u = 0.5 + 0.25 * np.sin(np.pi * X) * np.cos(np.pi * Y)
            gsum = 0.25 * np.pi * (np.cos(np.pi * X) * np.cos(np.pi * Y) - np.sin(np.pi * X) * np.sin(np.pi * Y))
        else:
            Z, Y, X = np.meshgrid(x, x, x, indexing="ij")
            u = 0.5 + 0.25 * np.sin(np.pi * X) * np.cos(np.pi * Y) * np.cos(np.pi * Z)
            gsum = 0.25 * np.pi * (np.cos(np.pi * X) * np.cos(np.pi * Y) * np.cos(np.pi * Z)
                                   - np.sin(np.pi * X) * np.sin(np.pi * Y) * np.cos(np.pi * Z)
                                   - np.sin(np.pi * X) * np.cos(np.pi * Y) * np.sin(np.pi * Z))
        f = ora.fe_eval(FE_BURGERS, u, periodic=True)
        errs.append(np.abs(f + u * gsum).max())
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    assert rates[-1] > 4.6 and min(rates) > 4.0, (errs, rates)   # pre-asymptotic on 16^3


def test_burgers_fe_invariants(ora):
    n = 64
    assert np.array_equal(ora.fe_eval(FE_BURGERS, np.full((n, n), 0.3), periodic=True), np.zeros((n, n)))
    u = synth.burgers_initial(n, seed=3, sigma=0.2) - 0.4 * synth.burgers_initial(n, seed=4, sigma=0.15)
    f = ora.fe_eval(FE_BURGERS, u, periodic=True)
    # conservation: the flux differences telescope over the periodic grid
    assert abs(f.sum()) <= 1e-13 * np.abs(f).sum()
    # translation equivariance (exact: the same operations on the same values)
    for sx, sy in ((1, 0), (0, 3), (17, 40)):
        assert np.array_equal(ora.fe_eval(FE_BURGERS, np.roll(u, (sy, sx), (0, 1)), periodic=True),
                              np.roll(f, (sy, sx), (0, 1)))
    # x <-> y symmetry of u u_x + u u_y (exact: gx + gy == gy + gx)
    assert np.array_equal(ora.fe_eval(FE_BURGERS, u.T.copy(), periodic=True), f.T)
    # point reflection x -> -x, u -> -u maps the equation to itself: f'(x) = -f(-x) (to rounding)
    idx = (-np.arange(n)) % n
    ur = -u[np.ix_(idx, idx)]
    fr = ora.fe_eval(FE_BURGERS, ur, periodic=True)
    np.testing.assert_allclose(fr, -f[np.ix_(idx, idx)], rtol=0, atol=1e-12 * np.abs(f).max())


# ----------------------------------------------------------------------- periodic multigrid
def psymbols(ks, n):
    h = 2.0 / n
    c = [math.cos(k * math.pi * h) for k in ks]
    if len(ks) == 2:
        return (-20 + 8 * c[0] + 8 * c[1] + 4 * c[0] * c[1]) / (6 * h * h), (8 + 2 * c[0] + 2 * c[1]) / 12
    s = sum(c)
    pr = c[0] * c[1] + c[0] * c[2] + c[1] * c[2]
    return (-24 + 4 * s + 4 * pr) / (6 * h * h), (6 + 2 * s) / 12


@pytest.mark.parametrize("ks,n", [((1, 1), 16), ((3, 5), 32), ((16, 1), 32), ((0, 7), 64), ((1, 2, 3), 16), ((8, 0, 2), 16)])
def test_periodic_symbols(ora, ks, n):
    """cos(pi k x) products are eigenvectors of the periodic pair; h = 2/n (reading R31)."""
    x = synth.grid_x_periodic(n)
    c = [np.cos(k * np.pi * x) for k in ks]
    phi = np.multiply.outer(c[1], c[0]) if len(ks) == 2 else np.multiply.outer(np.multiply.outer(c[2], c[1]), c[0])
    lL, lB = psymbols(ks, n)
    np.testing.assert_allclose(ora.apply_L(phi, periodic=True), lL * phi, rtol=0, atol=1e-11 * max(1, abs(lL)))
    np.testing.assert_allclose(ora.apply_B(phi, periodic=True), lB * phi, rtol=0, atol=1e-14)
    for gamma in (0.0, 1e-4, 0.3):
        np.testing.assert_allclose(ora.apply_S(phi, gamma, periodic=True), (lB - gamma * lL) * phi, rtol=0,
                                   atol=1e-11 * (1 + gamma * abs(lL)))


@pytest.mark.parametrize("dim,n", [(2, 16), (2, 32), (3, 8)])
def test_periodic_transfers(ora, dim, n):
    """Full weighting is 2^-d times the transpose of bilinear prolongation; constants pass through."""
    rng = np.random.default_rng(7)
    d = rng.uniform(-1, 1, (n,) * dim)
    e = rng.uniform(-1, 1, (n // 2,) * dim)
    Rd = ora.restrict(d, periodic=True)
    Pe = ora.prolong_add(e, np.zeros_like(d), periodic=True)
    assert abs((2 ** dim) * np.vdot(Rd, e) - np.vdot(d, Pe)) <= 1e-12 * np.abs(d).sum()
    assert np.array_equal(ora.restrict(np.full(d.shape, 0.75), periodic=True), np.full(e.shape, 0.75))
    assert np.array_equal(ora.prolong_add(np.full(e.shape, 0.5), np.full(d.shape, 0.25), periodic=True),
                          np.full(d.shape, 0.75))
    # coarse points coincide with the even fine points (x_{2I} = X_I): injection there
    sl = (slice(0, None, 2),) * dim
    assert np.array_equal(Pe[sl], e)


def dense_S(ora, dim, n, gamma):
    P = n ** dim
    S = np.zeros((P, P))
    for c in range(P):
        v = np.zeros(P)
        v[c] = 1.0
        S[:, c] = ora.apply_S(v.reshape((n,) * dim), gamma, periodic=True).ravel()
    return S


@pytest.mark.parametrize("dim,gamma", [(2, 1.5e-4), (2, 5e-3), (2, 0.0), (3, 5e-3)])
def test_periodic_coarse_inverse(ora, dim, gamma):
    G = ora.coarse_inverse(dim, gamma, periodic=True)
    S = dense_S(ora, dim, 4, gamma)
    assert np.abs(G @ S - np.eye(S.shape[0])).max() < 1e-13


@pytest.mark.parametrize("dim,n,gamma", [(2, 16, 1.5e-4), (2, 32, 5e-3), (2, 16, 0.0), (3, 8, 5e-3)])
def test_periodic_vcycle_converges_to_dense_solve(ora, dim, n, gamma):
    S = dense_S(ora, dim, n, gamma)
    b = synth.random_field(n, dim, 3)
    x = np.linalg.solve(S, b.ravel()).reshape(b.shape)
    u = np.zeros_like(b)
    errs = []
    for _ in range(14 if dim == 2 else 24):
        u = ora.vcycle(b, u, gamma, periodic=True)
        errs.append(np.abs(u - x).max())
    assert errs[-1] < 1e-11 * np.abs(x).max()
    assert errs[4] / errs[3] < (0.15 if dim == 2 else 0.25), errs     # grid-independent V(2,2) factor


# ----------------------------------------------------------------------------- whole steps
def spectral_step(u0, nu, dt, substeps=200):
    """Fourier pseudo-spectral + classical RK4 for u_t = -(u^2/2)_x - (u^2/2)_y + nu Lap u on [-1,1)^2."""
    n = u0.shape[0]
    k = np.pi * np.fft.fftfreq(n, d=1.0 / n)           # wavenumbers of period 2
    KX, KY = np.meshgrid(k, k)

    def rhs(u):
        q = np.fft.fft2(0.5 * u * u)
        U = np.fft.fft2(u)
        return np.real(np.fft.ifft2(-1j * KX * q - 1j * KY * q - nu * (KX ** 2 + KY ** 2) * U))

    u = u0.copy()
    h = dt / substeps
    for _ in range(substeps):
        a = rhs(u)
        b = rhs(u + 0.5 * h * a)
        c = rhs(u + 0.5 * h * b)
        d = rhs(u + h * c)
        u = u + (h / 6) * (a + 2 * b + 2 * c + d)
    return u


@pytest.mark.parametrize("nu", [0.01, 1.0])
def test_burgers_step_matches_spectral(ora, nu):
    """One converged SDC step of the IMEX/WENO5/compact discretisation vs a spectral solution of
    the same PDE: the change u(dt) - u(0) agrees to the spatial error (relative 1e-3)."""
    n = 128
    u0 = synth.burgers_initial(n, sigma=0.25)
    cfg = synth.burgers_config(nu, 5, n=n, sweep_tol=1e-10, max_sweeps=60, dt=0.002)
    u1, st = ora.step(ora.Problem(cfg, mode=MODE_SDC), u0, 0.0)
    assert st["converged"]
    ref = spectral_step(u0, nu, cfg.dt)
    d_ora, d_ref = u1 - u0, ref - u0
    assert np.abs(d_ora - d_ref).max() <= 1e-3 * np.abs(d_ref).max(), np.abs(d_ora - d_ref).max() / np.abs(d_ref).max()


@pytest.mark.parametrize("nu,M", [(0.1, 3), (1.0, 5), (10.0, 3)])
def test_burgers_step_invariants(ora, nu, M):
    """Table 1b problem: mass conserved (1^T W = 1^T, 1^T A = 0, sum f^E = 0), maximum principle,
    and fixed-L ISDC spends exactly K~(M-1)L cycles."""
    cfg = synth.burgers_config(nu, M)
    u0 = synth.burgers_initial(cfg.n)
    for mode in (MODE_SDC, MODE_ISDC):
        u1, st = ora.step(ora.Problem(cfg, mode=mode), u0, 0.0)
        assert st["converged"]
        assert abs(u1.sum() - u0.sum()) <= 1e-12 * np.abs(u0).sum()
        assert u1.max() <= u0.max() and u1.min() >= -1e-6
        if mode == MODE_ISDC:
            assert st["vcycles"] == st["sweeps"] * (M - 1) * cfg.L
