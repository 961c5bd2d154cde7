"""Pins of the oracle's multigrid pieces (B:configs[1] components; R11-R14).

Independent references: closed-form symbols of full weighting on sine modes, the adjoint identity
P = 2^d R^T, exact bilinear interpolation, dense LU / matrix inverse (numpy) of the node systems on
tiny grids, and the contraction / fixed-point properties of a convergent V-cycle.
"""
import math

import numpy as np
import pytest

import synth


def dense_S(ora, dim, n, gamma):
    P = n ** dim
    A = np.zeros((P, P))
    for i in range(P):
        e = np.zeros(P); e[i] = 1.0
        A[:, i] = ora.apply_S(e.reshape((n,) * dim), gamma).ravel()
    return A


@pytest.mark.parametrize("ks,nf", [((1, 1), 15), ((3, 5), 31), ((2, 1, 3), 15)])
def test_restriction_symbol(ora, ks, nf):
    """FW of a fine sine mode = prod cos^2(k pi h_f / 2) times the coarse mode (same points)."""
    phi_f = synth.sine_mode(nf, ks)
    nc = (nf - 1) // 2
    hf = 1.0 / (nf + 1)
    fac = np.prod([math.cos(k * math.pi * hf / 2) ** 2 for k in ks])
    np.testing.assert_allclose(ora.restrict(phi_f), fac * synth.sine_mode(nc, ks), atol=1e-15)


@pytest.mark.parametrize("dim", [2, 3])
def test_prolongation_adjoint_and_interpolation(ora, dim):
    nc = 7
    nf = 2 * nc + 1
    e = synth.random_field(nc, dim, 3)
    d = synth.random_field(nf, dim, 4)
    Pe = ora.prolong_add(e, np.zeros((nf,) * dim))
    assert abs((Pe * d).sum() - 2 ** dim * (e * ora.restrict(d)).sum()) < 1e-12
    # coincident points are injected
    sl = (slice(1, None, 2),) * dim
    np.testing.assert_array_equal(Pe[sl], e)
    # multilinear functions are interpolated exactly away from the (zero) boundary
    xc = synth.grid_x(nc)
    xf = synth.grid_x(nf)
    if dim == 2:
        f = lambda y, x: 1 + 2 * x + 3 * y + 4 * x * y
        fc = f(xc[:, None], xc[None, :]); ff = f(xf[:, None], xf[None, :])
    else:
        f = lambda z, y, x: 1 + 2 * x + 3 * y - z + 4 * x * y * z
        fc = f(xc[:, None, None], xc[None, :, None], xc[None, None, :])
        ff = f(xf[:, None, None], xf[None, :, None], xf[None, None, :])
    Pf = ora.prolong_add(fc, np.zeros((nf,) * dim))
    inner = (slice(1, -1),) * dim
    np.testing.assert_allclose(Pf[inner], ff[inner], atol=1e-14)


@pytest.mark.parametrize("dim,gamma", [(2, 0.0), (2, 0.005), (2, 1.7), (3, 0.01), (3, 2.0)])
def test_coarse_inverse(ora, dim, gamma):
    G = ora.coarse_inverse(dim, gamma)
    A = dense_S(ora, dim, 3, gamma)
    np.testing.assert_allclose(G, np.linalg.inv(A), rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(G @ A, np.eye(A.shape[0]), atol=1e-13)
    # on n = 3 the V-cycle is the exact solve
    b = synth.random_field(3, dim, 5)
    u = ora.vcycle(b, np.zeros_like(b), gamma)
    np.testing.assert_allclose(u.ravel(), np.linalg.solve(A, b.ravel()), rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("dim,n,gamma", [(2, 7, 0.005), (2, 15, 0.2), (3, 7, 0.01), (3, 15, 0.0005)])
def test_jacobi_and_vcycle_vs_dense(ora, dim, n, gamma):
    A = dense_S(ora, dim, n, gamma)
    b = synth.random_field(n, dim, 6)
    u = synth.random_field(n, dim, 7)
    # weighted Jacobi: u + (omega/diag) (b - A u)
    ref = u.ravel() + 0.8 / np.diag(A) * (b.ravel() - A @ u.ravel())
    np.testing.assert_allclose(ora.jacobi(b, u, gamma).ravel(), ref, rtol=1e-13, atol=1e-13)
    # cycles converge to the dense LU solution
    x = np.linalg.solve(A, b.ravel())
    v = np.zeros_like(b)
    for _ in range(40):
        v = ora.vcycle(b, v, gamma)
        if ora.defect_norm(b, v, gamma) < 1e-14:
            break
    np.testing.assert_allclose(v.ravel(), x, rtol=0, atol=1e-12 * np.abs(x).max())
    # the exact solution is a fixed point; so is zero
    xs = x.reshape(b.shape)
    np.testing.assert_allclose(ora.vcycle(b, xs, gamma), xs, atol=1e-13 * np.abs(x).max())
    z = np.zeros_like(b)
    assert np.all(ora.vcycle(z, z, gamma) == 0)


@pytest.mark.parametrize("dim,n,gamma", [(2, 63, 0.005), (2, 127, 0.01 * 0.172673), (2, 255, 0.1 * 0.01 * 0.327),
                                         (3, 31, 0.005), (3, 63, 0.01 * 0.5)])
def test_vcycle_contraction(ora, dim, n, gamma):
    """V(2,2) defect contraction per cycle <= 0.2 and monotone while above the floor."""
    xs = synth.random_field(n, dim, 8)
    b = ora.apply_S(xs, gamma)
    u = np.zeros_like(b)
    d = [ora.defect_norm(b, u, gamma)]
    for _ in range(5):
        u = ora.vcycle(b, u, gamma)
        d.append(ora.defect_norm(b, u, gamma))
    rates = [d[i + 1] / d[i] for i in range(len(d) - 1) if d[i] > 1e-12 * d[0]]
    assert max(rates) < 0.2, rates
