"""Pins of the oracle's collocation tables (Eq. 2) against exact values and invariants.

Independent references: the golden values printed in SPEC.md (tests/golden/spec_tables.txt),
the closed-form Lobatto-5 nodes, and a 50-digit mpmath quadrature of the Lagrange basis.
"""
import os
from fractions import Fraction

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_tables.txt")


def _golden():
    out = {}
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        key, *vals = line.split()
        out[key] = [float(Fraction(v)) for v in vals]
    return out


def test_lobatto3_golden(ora):
    g = _golden()
    tau, Q, S, dtau = ora.tables(3)
    assert list(tau) == g["lobatto3_nodes"]
    assert list(S[0]) == g["lobatto3_S_row0"]                     # S:58, correctly rounded
    # sum of the rows integrates tau^2 over [0,1] exactly
    f = tau ** 2
    assert abs((S.sum(axis=0) * f).sum() - g["lobatto3_int_tau2"][0]) < 1e-16
    assert list(Q[-1]) == [1 / 6, 2 / 3, 1 / 6]                   # Simpson's rule


def test_lobatto5_closed_form(ora):
    tau, Q, S, dtau = ora.tables(5)
    assert tau[1] == (1 - np.sqrt(3 / 7)) / 2 or abs(tau[1] - 0.17267316464601143) < 1e-17
    assert tau[1] == 0.17267316464601143      # (1-sqrt(3/7))/2 correctly rounded
    assert tau[2] == 0.5 and tau[0] == 0.0 and tau[4] == 1.0
    np.testing.assert_allclose(Q[-1], [1 / 20, 49 / 180, 16 / 45, 49 / 180, 1 / 20], rtol=0, atol=2e-17)


@pytest.mark.parametrize("M", [3, 4, 5, 7])
def test_tables_mpmath_exact(ora, M):
    """Every table entry is the correctly rounded value of its 50-digit definition."""
    mp = pytest.importorskip("mpmath")
    mp.mp.dps = 50
    # Lobatto nodes: roots of P'_{M-1} on [-1,1], mapped to [0,1]
    # exact monomial coefficients of P_{M-1} (Bonnet recurrence in rationals), then P'
    p0, p1 = [Fraction(1)], [Fraction(0), Fraction(1)]
    for k in range(1, M - 1):
        p2 = [Fraction(0)] * (k + 2)
        for i, c in enumerate(p1):
            p2[i + 1] += Fraction(2 * k + 1, k + 1) * c
        for i, c in enumerate(p0):
            p2[i] -= Fraction(k, k + 1) * c
        p0, p1 = p1, p2
    dP = [i * c for i, c in enumerate(p1)][1:]
    roots = mp.polyroots([mp.mpf(c.numerator) / c.denominator for c in reversed(dP)],
                         maxsteps=500, extraprec=500) if len(dP) > 1 else []
    xs = [mp.mpf(-1)] + sorted(mp.re(r) for r in roots) + [mp.mpf(1)]
    t = [(x + 1) / 2 for x in xs]

    def lag(j, s):
        r = mp.mpf(1)
        for k in range(M):
            if k != j:
                r *= (s - t[k]) / (t[j] - t[k])
        return r

    tau, Q, S, dtau = ora.tables(M)
    assert [float(v) for v in t] == list(tau)
    for m in range(M):
        for j in range(M):
            assert float(mp.quad(lambda s: lag(j, s), [0, t[m]])) == Q[m, j], (m, j)
    for m in range(M - 1):
        assert float(t[m + 1] - t[m]) == dtau[m]
        for j in range(M):
            assert float(mp.quad(lambda s: lag(j, s), [t[m], t[m + 1]])) == S[m, j], (m, j)


@pytest.mark.parametrize("M", [3, 5, 7])
def test_table_invariants(ora, M):
    tau, Q, S, dtau = ora.tables(M)
    # row sums = subinterval lengths (exactness on constants)
    np.testing.assert_allclose(S.sum(axis=1), dtau, atol=1e-15)
    np.testing.assert_allclose(Q.sum(axis=1), tau, atol=1e-15)
    # exact on polynomials of degree <= M-1
    rng = np.random.default_rng(0)
    for _ in range(5):
        c = rng.uniform(-1, 1, M)
        p = np.polynomial.Polynomial(c)
        P = p.integ()
        for m in range(M - 1):
            assert abs((S[m] * p(tau)).sum() - (P(tau[m + 1]) - P(tau[m]))) < 1e-13
        for m in range(M):
            assert abs((Q[m] * p(tau)).sum() - (P(tau[m]) - P(0.0))) < 1e-13
    # time-reversal symmetry s_{m,j} = s_{M-m,M+1-j}, 1-based -> 0-based
    for m in range(M - 1):
        for j in range(M):
            assert abs(S[m, j] - S[M - 2 - m, M - 1 - j]) < 1e-16
    # Q rows are cumulative sums of S rows
    np.testing.assert_allclose(np.cumsum(S, axis=0), Q[1:], atol=1e-15)
    assert np.all(Q[0] == 0.0)
