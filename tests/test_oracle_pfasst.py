"""Pins of the oracle's PFASST with ISDC sweeps (NEXT f4b; reading R33).

Independent references:
* the fixed point: a converged PFASST block of P slices equals P consecutive collocation steps --
  per sine mode the end value of slice p is R(z)^(p+1) u0 with R(z) = [(I - zQ)^{-1} 1]_M (the
  diagonal Pade closed forms of tests/test_oracle_sdc.py) -- whatever P, the predictor and the
  number of coarse sweeps;
* with forcing and with the nonlinear Allen-Cahn term: a converged block equals the converged
  single-level ISDC steps (pinned separately) run one after another;
* special cases that reduce to the pinned MLSDC (R32): one slice without predictor is the MLSDC
  step bit for bit; slice 0 of any block never receives a transferred value, so without the
  predictor its residual history and end value are the MLSDC step's bit for bit;
* the forward transfer: with the transfer cut (every slice starting from the spread u0), the block
  converges to P copies of the FIRST step -- the negative control showing that step 1 of R33 is what
  carries the initial values forward;
* behaviour: the iterations of a block are far fewer than the serial sweeps of the same
  P steps (the time-parallel potential).
"""
import math

import numpy as np
import pytest

import synth
from synth import Config, FE_CUBIC, FE_FORCING, FE_NONE


def sym(ks, n):
    h = 1.0 / (n + 1)
    c = [math.cos(k * math.pi * h) for k in ks]
    if len(ks) == 2:
        return (-20 + 8 * c[0] + 8 * c[1] + 4 * c[0] * c[1]) / (6 * h * h), (8 + 2 * c[0] + 2 * c[1]) / 12
    s = sum(c); pr = c[0] * c[1] + c[0] * c[2] + c[1] * c[2]
    return (-24 + 4 * s + 4 * pr) / (6 * h * h), (6 + 2 * s) / 12


@pytest.mark.parametrize("ks,M,nu,P,pred,cs", [((1, 2), 3, 1.0, 4, True, 1), ((2, 1), 5, 10.0, 3, False, 2),
                                                ((1, 1, 2), 3, 1.0, 2, True, 1), ((1, 3), 5, 1.0, 5, True, 1)])
def test_converged_block_is_p_collocation_steps(ora, ks, M, nu, P, pred, cs):
    n = 15
    dim = len(ks)
    cfg = Config(0, dim, n, M, 0.02, nu, FE_NONE, sweep_tol=1e-13, max_sweeps=300)
    u0 = synth.sine_mode(n, ks)
    ue, st = ora.pfasst_block(ora.Problem(cfg), u0, P, coarse_sweeps=cs, predictor=pred)
    assert st["converged"] and st["coarse_vcycles"] > 0
    lL, lB = sym(ks, n)
    z = cfg.dt * nu * lL / lB
    tau, Q, S, dtau = ora.tables(M)
    R = np.linalg.solve(np.eye(M) - z * Q, np.ones(M))[-1]
    for p in range(P):
        np.testing.assert_allclose(ue[p], R ** (p + 1) * u0, atol=2e-12)


@pytest.mark.parametrize("fe,dim", [(FE_FORCING, 2), (FE_CUBIC, 2), (FE_CUBIC, 3)])
def test_converged_block_equals_serial_isdc_steps(ora, fe, dim):
    n = 15 if dim == 2 else 7
    P = 3
    cfg = Config(0, dim, n, 3, 0.01, 0.5, fe, sweep_tol=1e-13, max_sweeps=300)
    u0 = synth.initial_condition(2 if dim == 2 else 4, 1, n) * (0.5 if fe == FE_CUBIC else 1.0)
    G = None
    if fe == FE_FORCING:
        x = synth.grid_x(n)
        G = np.outer(np.sin(2 * np.pi * x), np.sin(2 * np.pi * x))
    prob = ora.Problem(cfg, G)
    ue, st = ora.pfasst_block(prob, u0, P, step0=2)
    assert st["converged"]
    u = u0.copy()
    for p in range(P):
        u, s1 = ora.step(prob, u, float(2 + p) * cfg.dt)
        assert s1["converged"]
        np.testing.assert_allclose(ue[p], u, atol=1e-11 * max(1.0, np.abs(u).max()))


@pytest.mark.parametrize("fixed", [4, 0])
def test_one_slice_without_predictor_is_mlsdc(ora, fixed):
    n = 31
    cfg = Config(0, 2, n, 5, 0.005, 3.0, FE_FORCING, fixed_sweeps=fixed, sweep_tol=1e-10)
    u0 = synth.initial_condition(2, 0, n)
    x = synth.grid_x(n)
    G = np.outer(np.sin(2 * np.pi * x), np.sin(2 * np.pi * x))
    prob = ora.Problem(cfg, G)
    ue, st = ora.pfasst_block(prob, u0, 1, step0=3, coarse_sweeps=2, predictor=False)
    um, sm = ora.mlsdc_step(prob, u0, 3 * cfg.dt, coarse_sweeps=2)
    assert np.array_equal(ue[0], um)
    assert np.array_equal(st["res_hist"][:, 0], sm["res_hist"])
    assert st["iterations"] == sm["sweeps"] and st["coarse_vcycles"] == sm["coarse_vcycles"]


def test_slice0_without_predictor_is_mlsdc(ora):
    n, K = 31, 5
    cfg = Config(0, 2, n, 3, 0.01, 1.0, FE_CUBIC, fixed_sweeps=K)
    u0 = 0.5 * synth.initial_condition(2, 0, n)
    prob = ora.Problem(cfg)
    ue, st = ora.pfasst_block(prob, u0, 3, predictor=False)
    um, sm = ora.mlsdc_step(prob, u0, 0.0)
    assert np.array_equal(ue[0], um)
    assert np.array_equal(st["res_hist"][:, 0], sm["res_hist"])
    # the later slices differ (they receive transferred values)
    assert not np.array_equal(ue[1], ue[0])


def test_forward_transfer_negative_control(ora):
    """Cutting the forward transfer (R33 step 1) leaves every slice on the FIRST step's problem: the
    slices then converge to copies of step 1, not to steps 1..P.  Emulated with the slice phases
    (oracle.PfasstSlice) in the R33 order but without set_u0 / coarse node-0 transfers."""
    n, P = 15, 3
    cfg = Config(0, 2, n, 3, 0.02, 1.0, FE_NONE, sweep_tol=1e-13, max_sweeps=300)
    u0 = synth.sine_mode(n, (1, 1))
    prob = ora.Problem(cfg)
    sl = [ora.PfasstSlice(prob, u0, 0) for p in range(P)]   # all on t = 0 (f^E = 0: t is irrelevant)
    for _ in range(60):
        res = max(s.fine() for s in sl)
        if res < 1e-13:
            break
        for s in sl:
            s.restrict(); s.coarse(None); s.interpolate()
    ends = [s.end() for s in sl]
    assert np.array_equal(ends[0], ends[2])
    ue, st = ora.pfasst_block(prob, u0, P, predictor=False)
    np.testing.assert_allclose(ue[0], ends[0], atol=1e-13)
    assert np.abs(ue[2] - ends[2]).max() > 1e-3 * np.abs(ends[2]).max()


def test_slice_phases_recompose_the_block(ora):
    """The exported slice phases (PfasstSlice: A fine, B restrict, C coarse, D interpolate) driven in
    the R33 order reproduce ora_pfasst_block bit for bit (with the predictor)."""
    n, P = 15, 3
    cfg = Config(0, 2, n, 5, 0.01, 1.0, FE_CUBIC, fixed_sweeps=4)
    u0 = 0.5 * synth.initial_condition(2, 1, n)
    prob = ora.Problem(cfg)
    ue, st = ora.pfasst_block(prob, u0, P, step0=1, coarse_sweeps=1, predictor=True)
    sl = [ora.PfasstSlice(prob, u0, 1 + p) for p in range(P)]
    for s in sl:
        s.predict_restrict()
    for stage in range(P):
        for p in range(P - 1, stage - 1, -1):
            s = sl[p]
            s.coarse(sl[p - 1].U[-1].copy() if stage >= 1 else None)
    for s in sl:
        s.interpolate()
    hist = []
    for k in range(4):
        ends = [s.end() for s in sl]
        for p in range(1, P):
            sl[p].set_u0(ends[p - 1])
        hist.append([s.fine() for s in sl])
        if k == 3:
            break
        for s in sl:
            s.restrict()
        for p in range(P):
            sl[p].coarse(sl[p - 1].U[-1].copy() if p >= 1 else None)
        for s in sl:
            s.interpolate()
    assert np.array_equal(np.array(hist), st["res_hist"])
    for p in range(P):
        assert np.array_equal(sl[p].end(), ue[p])


def test_block_iterations_below_serial_sweeps(ora):
    """PFASST performs one sweep per level and iteration on every slice at once; a block
    of P = 4 slices converges in far fewer iterations than the 4 serial MLSDC steps' fine sweeps."""
    n, P = 15, 4
    cfg = Config(0, 2, n, 3, 0.02, 1.0, FE_NONE, sweep_tol=1e-12, max_sweeps=300)
    u0 = synth.sine_mode(n, (1, 2))
    prob = ora.Problem(cfg)
    ue, st = ora.pfasst_block(prob, u0, P)
    u, serial = u0.copy(), 0
    for s in range(P):
        u, sm = ora.mlsdc_step(prob, u, s * cfg.dt)
        serial += sm["sweeps"]
    assert st["converged"] and st["iterations"] < 0.5 * serial
    np.testing.assert_allclose(ue[-1], u, atol=1e-11)
