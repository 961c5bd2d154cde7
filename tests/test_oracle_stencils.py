"""Pins of the oracle's compact (Mehrstellen) operators.

References independent of the oracle: the closed-form Fourier symbols of the stencils on discrete
sine modes (exact eigenvectors under zero Dirichlet data), the continuous Laplacian symbol
-pi^2|k|^2 (4th-order consistency), SPEC's printed stencil patterns, invariants.
"""
import math

import numpy as np
import pytest

import synth


def symbols(ks, n):
    h = 1.0 / (n + 1)
    c = [math.cos(k * math.pi * h) for k in ks]
    if len(ks) == 2:
        lL = (-20 + 8 * c[0] + 8 * c[1] + 4 * c[0] * c[1]) / (6 * h * h)
        lB = (8 + 2 * c[0] + 2 * c[1]) / 12
    else:
        s = sum(c)
        pr = c[0] * c[1] + c[0] * c[2] + c[1] * c[2]
        lL = (-24 + 4 * s + 4 * pr) / (6 * h * h)
        lB = (6 + 2 * s) / 12
    return lL, lB


CASES = [((1, 1), 15), ((3, 2), 31), ((7, 5), 31), ((31, 1), 63), ((1, 2, 3), 15), ((5, 1, 7), 15), ((2, 2, 2), 31)]


@pytest.mark.parametrize("ks,n", CASES)
def test_symbols(ora, ks, n):
    phi = synth.sine_mode(n, ks)
    lL, lB = symbols(ks, n)
    np.testing.assert_allclose(ora.apply_L(phi), lL * phi, rtol=0, atol=1e-12 * abs(lL))
    np.testing.assert_allclose(ora.apply_B(phi), lB * phi, rtol=0, atol=1e-14)
    for gamma in (0.0, 1e-4, 0.05, 3.0):
        np.testing.assert_allclose(ora.apply_S(phi, gamma), (lB - gamma * lL) * phi, rtol=0,
                                   atol=1e-12 * (1 + gamma * abs(lL)))


@pytest.mark.parametrize("ks", [(1, 2), (2, 3), (1, 2, 3), (2, 1, 1)])
def test_fourth_order(ks):
    """lambda_L/lambda_B = -pi^2|k|^2 + O(h^4): error ratio ~16 per halving."""
    exact = -math.pi ** 2 * sum(k * k for k in ks)
    errs = []
    for n in (15, 31, 63, 127):
        lL, lB = symbols(ks, n)
        errs.append(abs(lL / lB - exact))
    ratios = [errs[i] / errs[i + 1] for i in range(len(errs) - 1)]
    assert all(r > 14.5 for r in ratios), ratios


@pytest.mark.parametrize("ks,n", [((1, 2), 15), ((2, 1, 1), 15)])
def test_operators_converge_4th_order(ora, ks, n):
    """Grid operators: ||L phi - B(-pi^2|k|^2 phi)||_inf falls ~16x per halving."""
    errs = []
    for nn in (n, 2 * n + 1, 4 * n + 3):
        phi = synth.sine_mode(nn, ks)
        k2 = sum(k * k for k in ks)
        errs.append(np.abs(ora.apply_L(phi) - ora.apply_B(-math.pi ** 2 * k2 * phi)).max())
    assert errs[0] / errs[1] > 14.0 and errs[1] / errs[2] > 14.0, errs


def test_delta_patterns(ora):
    """a delta field reproduces the stencil patterns; 3D per SURVEY §8(c1)."""
    n = 7
    N2 = (n + 1) ** 2
    d = np.zeros((n, n)); d[3, 3] = 1.0
    B = ora.apply_B(d)[2:5, 2:5] * 12
    L = ora.apply_L(d)[2:5, 2:5] * 6 / N2
    np.testing.assert_allclose(B, [[0, 1, 0], [1, 8, 1], [0, 1, 0]], atol=1e-14)
    np.testing.assert_allclose(L, [[1, 4, 1], [4, -20, 4], [1, 4, 1]], atol=1e-12)
    d3 = np.zeros((n, n, n)); d3[3, 3, 3] = 1.0
    B3 = ora.apply_B(d3)[2:5, 2:5, 2:5] * 12
    L3 = ora.apply_L(d3)[2:5, 2:5, 2:5] * 6 / N2
    off = np.abs(np.indices((3, 3, 3)) - 1).sum(axis=0)   # 0 centre, 1 face, 2 edge, 3 corner
    np.testing.assert_allclose(B3, np.choose(off, [6, 1, 0, 0]), atol=1e-14)
    np.testing.assert_allclose(L3, np.choose(off, [-24, 2, 1, 0]), atol=1e-12)


@pytest.mark.parametrize("dim", [2, 3])
def test_constants_symmetry_contraction(ora, dim):
    n = 15
    one = np.ones((n,) * dim)
    inner = (slice(1, -1),) * dim
    np.testing.assert_allclose(ora.apply_B(one)[inner], 1.0, atol=1e-15)     # S:98 row sums 1
    np.testing.assert_allclose(ora.apply_L(one)[inner], 0.0, atol=1e-9)      # S:97 row sums 0
    u = synth.random_field(n, dim, 1)
    v = synth.random_field(n, dim, 2)
    for op in (ora.apply_B, ora.apply_L, lambda x: ora.apply_S(x, 0.37)):
        assert abs((op(u) * v).sum() - (u * op(v)).sum()) < 1e-10 * np.abs(op(u)).max() * u.size
    assert np.abs(ora.apply_B(u)).max() <= np.abs(u).max()


def test_cd4_advection(ora):
    """CD4 derivative (B:configs[5]): 4th-order in the interior; exact on cubics away from the
    boundary; zero ghost values (DESIGN R22) only change the two boundary-adjacent layers."""
    a = (1.0, 0.5, 0.25)
    errs = []
    for n in (31, 63, 127):
        x = synth.grid_x(n)
        X = x[None, :]; Y = x[:, None]
        u = np.sin(math.pi * X) * np.sin(2 * math.pi * Y) + 0 * X
        du = -(a[0] * math.pi * np.cos(math.pi * X) * np.sin(2 * math.pi * Y)
               + a[1] * 2 * math.pi * np.sin(math.pi * X) * np.cos(2 * math.pi * Y))
        f = ora.fe_eval(synth.FE_ADVECTION, u, a)
        errs.append(np.abs(f - du)[2:-2, 2:-2].max())
    assert errs[0] / errs[1] > 14 and errs[1] / errs[2] > 14, errs
    # exact for cubic polynomials (CD4 is exact up to degree 4) away from the boundary
    n = 15
    x = synth.grid_x(n)
    Z, Y, X = np.meshgrid(x, x, x, indexing="ij")
    u = X ** 3 - 2 * Y ** 2 * Z + Z ** 3
    du = -(a[0] * 3 * X ** 2 + a[1] * (-4 * Y * Z) + a[2] * (-2 * Y ** 2 + 3 * Z ** 2))
    f = ora.fe_eval(synth.FE_ADVECTION, u, a)
    np.testing.assert_allclose(f[2:-2, 2:-2, 2:-2], du[2:-2, 2:-2, 2:-2], atol=1e-11)


def test_fe_pointwise_kinds(ora):
    """Pointwise kinds: u - u^3 has fixed points {-1, 0, 1}; forcing is G*cos(t)."""
    u = np.array([[-1.0, 0.0], [1.0, 0.5]])
    f = ora.fe_eval(synth.FE_CUBIC, u)
    assert f[0, 0] == 0 and f[0, 1] == 0 and f[1, 0] == 0 and f[1, 1] == 0.375
    G = synth.forcing_field(7)
    np.testing.assert_array_equal(ora.fe_eval(synth.FE_FORCING, G * 0, G=G, ct=0.5), G * 0.5)
