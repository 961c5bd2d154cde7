"""ctypes wrapper of the CPU oracle (oracle/isdc_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs, never by the product package ``paper_1401_7824_b200``.  It shares no code
with the CUDA path; see DESIGN.md §5 ("oracle").  Every function cites the paper passage it follows
in isdc_oracle.c.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "isdc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC", "-Wall"]


def _hash() -> str:
    import hashlib
    with open(_SRC, "rb") as f:
        return hashlib.sha256(f.read() + " ".join(CFLAGS).encode()).hexdigest()


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no FMA contraction, no fast-math); rebuilt whenever the
    source or the flags differ from the stamp of the last build."""
    stamp = _LIB + ".sha256"
    h = _hash()
    fresh = os.path.exists(_LIB) and os.path.exists(stamp) and open(stamp).read().strip() == h
    if force or not fresh:
        tmp = _LIB + ".tmp"
        subprocess.run(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lquadmath", "-lm"], check=True)
        os.replace(tmp, _LIB)
        with open(stamp, "w") as f:
            f.write(h + "\n")
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_LIB)
        _declare(_lib)
    return _lib


class OraProblem(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("n", C.c_int), ("M", C.c_int),
        ("dt", C.c_double), ("nu", C.c_double),
        ("fe", C.c_int), ("fe_a", C.c_double * 3), ("G", C.c_void_p),
        ("mode", C.c_int), ("L", C.c_int), ("inner_tol", C.c_double), ("inner_cap", C.c_int),
        ("sweep_tol", C.c_double), ("max_sweeps", C.c_int), ("fixed_sweeps", C.c_int),
        ("nu1", C.c_int), ("nu2", C.c_int), ("omega", C.c_double), ("guess", C.c_int),
        ("res_kind", C.c_int), ("w_tol", C.c_double), ("w_cap", C.c_int), ("bc", C.c_int),
    ]


_dp = C.POINTER(C.c_double)


def _declare(L):
    L.ora_tables.argtypes = [C.c_int, _dp, _dp, _dp, _dp]
    L.ora_apply_B.argtypes = [C.c_int, C.c_int, _dp, _dp]
    L.ora_apply_L.argtypes = [C.c_int, C.c_int, _dp, _dp]
    L.ora_apply_S.argtypes = [C.c_int, C.c_int, C.c_double, _dp, _dp]
    L.ora_level_coefs.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, _dp]
    L.ora_jacobi.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _dp, _dp]
    L.ora_defect_norm.argtypes = [C.c_int, C.c_int, C.c_double, _dp, _dp]
    L.ora_defect_norm.restype = C.c_double
    L.ora_restrict.argtypes = [C.c_int, C.c_int, _dp, _dp]
    L.ora_prolong_add.argtypes = [C.c_int, C.c_int, _dp, _dp]
    L.ora_coarse_inverse.argtypes = [C.c_int, C.c_double, C.c_double, _dp]
    L.ora_vcycle.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_double, _dp, _dp]
    L.ora_fe_eval.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_double, _dp, _dp]
    PP = C.POINTER(_dp)
    L.ora_rhs.argtypes = [C.POINTER(OraProblem), C.c_double, C.c_int, PP, PP, _dp]
    L.ora_residual.argtypes = [C.POINTER(OraProblem), C.c_double, PP, _dp]
    L.ora_residual.restype = C.c_double
    L.ora_sweep_state.argtypes = [C.POINTER(OraProblem), C.c_double, PP, PP, C.POINTER(C.c_int)]
    L.ora_step.argtypes = [C.POINTER(OraProblem), _dp, C.c_double, C.POINTER(C.c_int),
                           C.POINTER(C.c_long), _dp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                           C.POINTER(C.c_int)]
    L.ora_num_threads.restype = C.c_int
    L.ora_set_num_threads.argtypes = [C.c_int]
    L.ora_last_wcycles.restype = C.c_long
    L.ora_set_bc.argtypes = [C.c_int]
    L.ora_inject.argtypes = [C.c_int, C.c_int, _dp, _dp]
    L.ora_prolong4_add.argtypes = [C.c_int, C.c_int, _dp, _dp]
    L.ora_mlsdc_correction.argtypes = [C.POINTER(OraProblem), C.c_int, C.c_double, PP, C.c_void_p, C.c_int]
    L.ora_mlsdc_correction.restype = C.c_long
    L.ora_mlsdc_step.argtypes = [C.POINTER(OraProblem), C.c_int, _dp, C.c_double, C.POINTER(C.c_int),
                                 C.POINTER(C.c_long), C.POINTER(C.c_long), _dp, C.POINTER(C.c_int)]
    L.ora_pf_fine.argtypes = [C.POINTER(OraProblem), C.c_double, PP, PP, PP, C.POINTER(C.c_long)]
    L.ora_pf_fine.restype = C.c_double
    L.ora_pf_restrict.argtypes = [C.POINTER(OraProblem), C.c_double, PP, PP, PP, PP, PP]
    L.ora_pf_coarse.argtypes = [C.POINTER(OraProblem), C.c_int, C.c_double, C.c_void_p, PP, PP]
    L.ora_pf_coarse.restype = C.c_long
    L.ora_pf_interpolate.argtypes = [C.POINTER(OraProblem), PP, PP, PP]
    L.ora_pf_residual.argtypes = [C.POINTER(OraProblem), C.c_double, PP, PP]
    L.ora_pf_residual.restype = C.c_double
    L.ora_pfasst_block.argtypes = [C.POINTER(OraProblem), C.c_int, C.c_int, C.c_int, _dp, C.c_int,
                                   C.POINTER(C.c_int), C.POINTER(C.c_long), C.POINTER(C.c_long), _dp,
                                   C.POINTER(C.c_int), _dp]
    L.ora_weno5.argtypes = [C.c_double] * 5
    L.ora_weno5.restype = C.c_double


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def num_threads() -> int:
    return lib().ora_num_threads()


def set_num_threads(t: int) -> None:
    """OpenMP threads of the oracle's grid loops (timing only; results are thread-count independent)."""
    lib().ora_set_num_threads(int(t))


# ---------------------------------------------------------------------------------------------
# tables and operators
# ---------------------------------------------------------------------------------------------
def tables(M: int):
    """(tau[M], Q[M,M], S[M-1,M], dtau[M-1]) for Gauss-Lobatto nodes (Eq. 2)."""
    tau, Q = np.zeros(M), np.zeros((M, M))
    S, dtau = np.zeros((M - 1, M)), np.zeros(M - 1)
    if lib().ora_tables(M, _p(tau), _p(Q), _p(S), _p(dtau)):
        raise ValueError(M)
    return tau, Q, S, dtau


def _bc(periodic):
    """Select the grid kind of the next oracle call (isdc_oracle.c header: Dirichlet / periodic)."""
    lib().ora_set_bc(1 if periodic else 0)
    return lib()


def weno5(v0, v1, v2, v3, v4):
    """WENO5-JS face value from five cell values (isdc_oracle.c weno5, reading R31)."""
    return lib().ora_weno5(float(v0), float(v1), float(v2), float(v3), float(v4))


def apply_B(u, periodic=False):
    u = _c(u); out = np.empty_like(u)
    _bc(periodic).ora_apply_B(u.ndim, u.shape[0], _p(u), _p(out)); return out


def apply_L(u, periodic=False):
    u = _c(u); out = np.empty_like(u)
    _bc(periodic).ora_apply_L(u.ndim, u.shape[0], _p(u), _p(out)); return out


def apply_S(u, gamma, periodic=False):
    u = _c(u); out = np.empty_like(u)
    _bc(periodic).ora_apply_S(u.ndim, u.shape[0], gamma, _p(u), _p(out)); return out


def level_coefs(dim, n, gamma, omega=0.8, periodic=False):
    c = np.zeros(4)
    _bc(periodic).ora_level_coefs(dim, n, gamma, omega, _p(c)); return c


def jacobi(b, u, gamma, sweeps=1, omega=0.8, periodic=False):
    b = _c(b); u = _c(u).copy()
    _bc(periodic).ora_jacobi(u.ndim, u.shape[0], gamma, omega, sweeps, _p(b), _p(u)); return u


def defect_norm(b, u, gamma, periodic=False):
    b = _c(b); u = _c(u)
    return _bc(periodic).ora_defect_norm(u.ndim, u.shape[0], gamma, _p(b), _p(u))


def restrict(d, periodic=False):
    d = _c(d); nc = d.shape[0] // 2 if periodic else (d.shape[0] - 1) // 2
    out = np.zeros((nc,) * d.ndim)
    _bc(periodic).ora_restrict(d.ndim, d.shape[0], _p(d), _p(out)); return out


def prolong_add(ec, uf, periodic=False):
    ec = _c(ec); uf = _c(uf).copy()
    _bc(periodic).ora_prolong_add(ec.ndim, ec.shape[0], _p(ec), _p(uf)); return uf


def coarse_inverse(dim, gamma, omega=0.8, periodic=False):
    P = (4 if periodic else 3) ** dim
    G = np.zeros((P, P))
    if _bc(periodic).ora_coarse_inverse(dim, gamma, omega, _p(G)):
        raise ValueError("singular")
    return G


def vcycle(b, u, gamma, nu1=2, nu2=2, omega=0.8, cycles=1, periodic=False):
    b = _c(b); u = _c(u).copy()
    for _ in range(cycles):
        _bc(periodic).ora_vcycle(u.ndim, u.shape[0], gamma, nu1, nu2, omega, _p(b), _p(u))
    return u


def fe_eval(fe, u, a=(0.0, 0.0, 0.0), G=None, ct=1.0, periodic=False):
    u = _c(u); out = np.empty_like(u)
    av = np.array(a, dtype=np.float64)
    Gp = _p(_c(G)) if G is not None else None
    _bc(periodic).ora_fe_eval(fe, u.ndim, u.shape[0], _p(av), Gp, ct, _p(u), _p(out)); return out


# ---------------------------------------------------------------------------------------------
# problem-level entry points
# ---------------------------------------------------------------------------------------------
class Problem:
    """Mirror of synth.Config plus run-time choices; holds the ctypes struct and keeps G alive."""

    def __init__(self, cfg, G=None, mode=0, guess=0, res_kind=0, w_tol=1e-6, w_cap=50):
        self.cfg = cfg
        self.G = None if G is None else _c(G)
        self.s = OraProblem()
        s = self.s
        s.dim, s.n, s.M = cfg.dim, cfg.n, cfg.M
        s.dt, s.nu, s.fe = cfg.dt, cfg.nu, cfg.fe
        for i in range(3):
            s.fe_a[i] = cfg.fe_a[i]
        s.G = self.G.ctypes.data if self.G is not None else None
        s.mode, s.L, s.inner_tol, s.inner_cap = mode, cfg.L, cfg.inner_tol, cfg.inner_cap
        s.sweep_tol, s.max_sweeps, s.fixed_sweeps = cfg.sweep_tol, cfg.max_sweeps, cfg.fixed_sweeps
        s.nu1, s.nu2, s.omega, s.guess = cfg.nu1, cfg.nu2, cfg.omega, guess
        s.res_kind, s.w_tol, s.w_cap = res_kind, w_tol, w_cap
        s.bc = getattr(cfg, "bc", 0)


def _ptrs(fields):
    arr = (_dp * len(fields))()
    for i, f in enumerate(fields):
        arr[i] = _p(f)
    return arr


def rhs(prob: Problem, t_n, m, uold, unew):
    """b of Eq. (5) for substep m (0-based) from node fields uold[M], unew[M]."""
    uold = [_c(x) for x in uold]; unew = [_c(x) for x in unew]
    b = np.empty_like(uold[0])
    lib().ora_rhs(C.byref(prob.s), t_n, m, _ptrs(uold), _ptrs(unew), _p(b))
    return b


def residual(prob: Problem, t_n, u):
    """(max_m ||r~_m||, per_node[M-1]) of the node fields u[M] (weighted residual, DESIGN R15)."""
    u = [_c(x) for x in u]
    per = np.zeros(prob.cfg.M - 1)
    r = lib().ora_residual(C.byref(prob.s), t_n, _ptrs(u), _p(per))
    return r, per


def sweep(prob: Problem, t_n, uold):
    """One sweep from node fields uold[M]; returns (unew[M], cycles[M-1])."""
    uold = [_c(x) for x in uold]
    unew = [uold[0]] + [np.empty_like(uold[0]) for _ in range(prob.cfg.M - 1)]
    cyc = (C.c_int * (prob.cfg.M - 1))()
    lib().ora_sweep_state(C.byref(prob.s), t_n, _ptrs(uold), _ptrs(unew), cyc)
    return unew, list(cyc)


def step(prob: Problem, u0, t_n):
    """One time step; returns (u_M, stats dict)."""
    cfg = prob.cfg
    u = _c(u0).copy()
    kmax = cfg.fixed_sweeps if cfg.fixed_sweeps > 0 else cfg.max_sweeps
    hist = np.zeros(kmax)
    ncyc = (C.c_int * (kmax * (cfg.M - 1)))()
    sw, vc, caps, conv = C.c_int(0), C.c_long(0), C.c_int(0), C.c_int(0)
    t0 = time.perf_counter()
    rc = lib().ora_step(C.byref(prob.s), _p(u), t_n, C.byref(sw), C.byref(vc), _p(hist), ncyc,
                        C.byref(caps), C.byref(conv))
    el = time.perf_counter() - t0
    if rc:
        raise RuntimeError("ora_step failed")
    k = sw.value
    return u, dict(sweeps=k, vcycles=vc.value, res_hist=hist[:k].copy(), wcycles=lib().ora_last_wcycles(),
                   node_cycles=np.array(ncyc[: k * (cfg.M - 1)]).reshape(k, cfg.M - 1),
                   cap_hits=caps.value, converged=bool(conv.value), seconds=el)


def run(prob: Problem, u0, steps=None):
    """``steps`` time steps from t = 0 (t_n = float(n)*dt, DESIGN R28)."""
    cfg = prob.cfg
    steps = cfg.steps if steps is None else steps
    u = _c(u0).copy()
    stats = []
    for s in range(steps):
        u, st = step(prob, u, float(s) * cfg.dt)
        stats.append(st)
    return u, stats


# ---------------------------------------------------------------------------------------------
# MLSDC with ISDC sweeps (NEXT f4; isdc_oracle.c ora_mlsdc_step, reading R32)
# ---------------------------------------------------------------------------------------------
def inject(uf):
    """Injection coarse I <- fine 2I+1 (Dirichlet)."""
    uf = _c(uf); nc = (uf.shape[0] - 1) // 2
    out = np.zeros((nc,) * uf.ndim)
    _bc(False).ora_inject(uf.ndim, uf.shape[0], _p(uf), _p(out)); return out


def prolong4_add(ec, uf):
    """u += P4 e: 4th-order (cubic Lagrange) interpolation of a coarse correction (Dirichlet)."""
    ec = _c(ec); uf = _c(uf).copy()
    _bc(False).ora_prolong4_add(ec.ndim, ec.shape[0], _p(ec), _p(uf)); return uf


def mlsdc_correction(prob: Problem, t_n, u, coarse_sweeps=1, fas=True):
    """Steps 2-5 of an MLSDC iteration on node fields u[M]; returns (corrected u, coarse V-cycles)."""
    u = [_c(x).copy() for x in u]
    cv = lib().ora_mlsdc_correction(C.byref(prob.s), int(coarse_sweeps), t_n, _ptrs(u), None, 0 if fas else 1)
    return u, cv


def mlsdc_step(prob: Problem, u0, t_n, coarse_sweeps=1):
    """One two-level MLSDC time step with ISDC sweeps; returns (u_M, stats dict)."""
    cfg = prob.cfg
    u = _c(u0).copy()
    kmax = cfg.fixed_sweeps if cfg.fixed_sweeps > 0 else cfg.max_sweeps
    hist = np.zeros(kmax)
    sw, vc, cvc, conv = C.c_int(0), C.c_long(0), C.c_long(0), C.c_int(0)
    t0 = time.perf_counter()
    rc = lib().ora_mlsdc_step(C.byref(prob.s), int(coarse_sweeps), _p(u), t_n, C.byref(sw), C.byref(vc),
                              C.byref(cvc), _p(hist), C.byref(conv))
    if rc:
        raise ValueError(f"ora_mlsdc_step: unsupported problem ({rc})")
    k = sw.value
    return u, dict(sweeps=k, vcycles=vc.value, coarse_vcycles=cvc.value, res_hist=hist[:k].copy(),
                   converged=bool(conv.value), seconds=time.perf_counter() - t0)


# ---------------------------------------------------------------------------------------------
# PFASST with ISDC sweeps (NEXT f4b; isdc_oracle.c ora_pfasst_block, reading R33)
# ---------------------------------------------------------------------------------------------
def pfasst_block(prob: Problem, u0, nslices, step0=0, coarse_sweeps=1, predictor=True):
    """One PFASST block of `nslices` time slices (steps step0 .. step0+nslices-1) from u0, serial
    emulation in the order of R33.  Returns (fine end value of every slice [nslices, ...], stats)."""
    cfg = prob.cfg
    u = _c(u0).copy()
    kmax = cfg.fixed_sweeps if cfg.fixed_sweeps > 0 else cfg.max_sweeps
    hist = np.zeros(kmax * nslices)
    uend = np.zeros((nslices,) + u.shape)
    it, vc, cvc, conv = C.c_int(0), C.c_long(0), C.c_long(0), C.c_int(0)
    t0 = time.perf_counter()
    rc = lib().ora_pfasst_block(C.byref(prob.s), int(nslices), int(coarse_sweeps), 1 if predictor else 0, _p(u),
                                int(step0), C.byref(it), C.byref(vc), C.byref(cvc), _p(hist), C.byref(conv),
                                _p(uend))
    if rc:
        raise ValueError(f"ora_pfasst_block: unsupported problem ({rc})")
    k = it.value
    return uend, dict(iterations=k, vcycles=vc.value, coarse_vcycles=cvc.value,
                      res_hist=hist[: k * nslices].reshape(k, nslices).copy(), converged=bool(conv.value),
                      seconds=time.perf_counter() - t0)


class PfasstSlice:
    """One PFASST time slice on the oracle (phases A-D of isdc_oracle.c, R33): the same per-slice
    operations the CUDA slice handle performs; used by the multi-process tests of the product's
    PFASST driver (tests/test_pfasst_driver.py)."""

    def __init__(self, prob: Problem, u0, step_index, coarse_sweeps=1):
        self.prob, self.cfg = prob, prob.cfg
        self.coarse_sweeps = coarse_sweeps
        M, n, d = self.cfg.M, self.cfg.n, self.cfg.dim
        nc = (n - 1) // 2
        self.t_n = float(step_index) * self.cfg.dt
        u0 = _c(u0)
        self.u0 = u0.copy()
        self.uold = [self.u0] + [u0.copy() for _ in range(M - 1)]
        self.unew = [self.u0] + [np.zeros_like(u0) for _ in range(M - 1)]
        self.rh = [np.zeros_like(u0) for _ in range(M)]
        self.Ub = [np.zeros((nc,) * d) for _ in range(M)]
        self.U = [np.zeros((nc,) * d) for _ in range(M)]
        self.fas = [np.zeros((nc,) * d) for _ in range(M)]
        self.vcycles = 0
        self.coarse_vcycles = 0
        self.fine_shape, self.coarse_shape, self.wants_torch = (n,) * d, (nc,) * d, False

    def set_u0(self, u0):
        self.u0[...] = u0

    def predict_restrict(self):
        """Predictor: the fine residual fields of the current (spread) state, then phase B."""
        lib().ora_pf_residual(C.byref(self.prob.s), self.t_n, _ptrs(self.uold), _ptrs(self.rh))
        self.restrict()

    def fine(self):
        vc = C.c_long(0)
        r = lib().ora_pf_fine(C.byref(self.prob.s), self.t_n, _ptrs(self.uold), _ptrs(self.unew), _ptrs(self.rh),
                              C.byref(vc))
        self.vcycles += vc.value
        self.uold, self.unew = self.unew, self.uold
        return float(r)

    def restrict(self):
        lib().ora_pf_restrict(C.byref(self.prob.s), self.t_n, _ptrs(self.uold), _ptrs(self.rh), _ptrs(self.Ub),
                              _ptrs(self.U), _ptrs(self.fas))

    def coarse(self, U0=None):
        U0c = None if U0 is None else _c(U0)
        self.coarse_vcycles += lib().ora_pf_coarse(C.byref(self.prob.s), int(self.coarse_sweeps), self.t_n,
                                                   None if U0c is None else U0c.ctypes.data, _ptrs(self.U),
                                                   _ptrs(self.fas))
        return self.U[-1].copy()

    def interpolate(self):
        lib().ora_pf_interpolate(C.byref(self.prob.s), _ptrs(self.U), _ptrs(self.Ub), _ptrs(self.uold))
        return self.uold[-1].copy()

    def end(self):
        return self.uold[-1].copy()
