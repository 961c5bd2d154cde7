"""Thin ctypes binding of libisdc.so (include/isdc.h): argument marshalling only.

Every step of the ISDC hot path runs in the CUDA library; PyTorch supplies device memory
(the workspace and the caller's fields) and the stream.  There is no CPU fallback: if the
library or a CUDA device is missing, construction raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libisdc.so")

FE_NONE, FE_CUBIC, FE_FORCING, FE_ADVECTION, FE_BURGERS = 0, 1, 2, 3, 4
BC_DIRICHLET, BC_PERIODIC = 0, 1
MODE_ISDC, MODE_SDC, MODE_ISDC_CAPPED = 0, 1, 2
STATUS = {0: "ok", 1: "invalid argument", 2: "unsupported", 3: "cuda error", 4: "non-finite value",
          5: "bad workspace"}


class IsdcError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__(f"isdc status {status} ({STATUS.get(status, '?')}): {msg}")
        self.status = status


class _Grid(C.Structure):
    _fields_ = [("dim", C.c_int), ("n", C.c_int), ("coarsest_n", C.c_int), ("bc", C.c_int)]


class _Mg(C.Structure):
    _fields_ = [("nu1", C.c_int), ("nu2", C.c_int), ("omega", C.c_double)]


class _Solve(C.Structure):
    _fields_ = [("mode", C.c_int), ("L", C.c_int), ("inner_tol", C.c_double), ("inner_cap", C.c_int),
                ("sweep_tol", C.c_double), ("max_sweeps", C.c_int), ("fixed_sweeps", C.c_int),
                ("guess", C.c_int)]


class _Problem(C.Structure):
    _fields_ = [("grid", _Grid), ("M", C.c_int), ("nodes", C.c_int), ("dt", C.c_double), ("nu", C.c_double),
                ("fe", C.c_int), ("fe_params", C.c_double * 3), ("fe_field_dev", C.c_void_p),
                ("mg", _Mg), ("solve", _Solve), ("residual_kind", C.c_int), ("w_tol", C.c_double),
                ("w_cap", C.c_int), ("mlsdc_levels", C.c_int), ("coarse_sweeps", C.c_int)]


class _Stats(C.Structure):
    _fields_ = [("sweeps", C.c_int), ("vcycles", C.c_long), ("cap_hits", C.c_int), ("converged", C.c_int),
                ("final_residual", C.c_double), ("wcycles", C.c_long), ("coarse_vcycles", C.c_long)]


_lib = None
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_vp = C.c_void_p


def lib():
    """Load libisdc.so (built in-tree by ``paper_1401_7824_b200.build``); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_1401_7824_b200.build` "
                              "(no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER(_Problem)
        L.isdc_workspace_bytes.argtypes = [P, C.POINTER(C.c_size_t)]
        L.isdc_create.argtypes = [P, _vp, C.c_size_t, _vp, C.POINTER(_vp)]
        L.isdc_set_initial.argtypes = [_vp, _vp, C.c_int]
        L.isdc_set_initial_host.argtypes = [_vp, _dp, C.c_int]
        L.isdc_set_state.argtypes = [_vp, C.POINTER(_vp), C.c_int]
        L.isdc_sweep.argtypes = [_vp, _dp, _dp, _ip]
        L.isdc_step.argtypes = [_vp, C.POINTER(_Stats), _dp, _ip]
        L.isdc_run.argtypes = [_vp, C.c_int, C.POINTER(_Stats)]
        L.mg_vcycle.argtypes = [_vp, C.c_int, _vp, _vp, _dp, _dp]
        L.residual_norm.argtypes = [_vp, _dp, _dp]
        L.isdc_get_solution.argtypes = [_vp, C.c_int, _vp]
        L.isdc_get_solution_host.argtypes = [_vp, C.c_int, _dp]
        L.isdc_get_tables.argtypes = [_vp, _dp, _dp, _dp, _dp]
        L.isdc_rhs.argtypes = [_vp, C.c_int, C.POINTER(_vp), _vp, _vp]
        L.isdc_kernel_launches.argtypes = [_vp]
        L.isdc_kernel_launches.restype = C.c_long
        L.isdc_destroy.argtypes = [_vp]
        L.isdc_pfasst_set_u0.argtypes = [_vp, _vp]
        L.isdc_pfasst_restrict.argtypes = [_vp]
        L.isdc_pfasst_coarse.argtypes = [_vp, _vp, _vp, C.POINTER(C.c_long)]
        L.isdc_pfasst_interpolate.argtypes = [_vp, _vp]
        L.isdc_last_error.argtypes = [_vp]
        L.isdc_last_error.restype = C.c_char_p
        L.isdc_profile_enable.argtypes = [_vp, C.c_int]
        L.isdc_profile_reset.argtypes = [_vp]
        L.isdc_profile_get.argtypes = [_vp, C.c_int, _dp, C.POINTER(C.c_long), _dp]
        L.isdc_build_tables.argtypes = [C.c_int, _dp, _dp, _dp, _dp]
        L.isdc_coarse_inverse.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, _dp]
        _lib = L
    return _lib


EXPORTED = ["isdc_workspace_bytes", "isdc_create", "isdc_set_initial", "isdc_set_initial_host", "isdc_sweep",
            "isdc_step", "isdc_run", "mg_vcycle", "residual_norm", "isdc_get_solution",
            "isdc_get_solution_host", "isdc_set_state", "isdc_get_tables", "isdc_rhs", "isdc_kernel_launches",
            "isdc_destroy", "isdc_last_error", "isdc_status_string", "isdc_profile_enable", "isdc_profile_reset",
            "isdc_profile_get"]

PROFILE_CLASS_IDS = {"fine_smoother": 0, "fine_defect_restrict": 1, "fine_prolong_correct": 2, "rhs": 3,
                     "residual": 4, "coarse_levels": 5}
PROFILE_CLASSES = {0: "fine_smoother", 1: "fine_defect_restrict", 2: "fine_prolong_correct", 3: "rhs", 4: "residual",
                   5: "coarse_levels"}


def _np_ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


class ISDC:
    """One ISDC problem instance bound to a CUDA stream (see include/isdc.h)."""

    def __init__(self, dim: int, n: int, M: int, dt: float, nu: float, fe: int = FE_NONE,
                 fe_a=(0.0, 0.0, 0.0), G: Optional[torch.Tensor] = None, mode: int = MODE_ISDC, L: int = 2,
                 inner_tol: float = 1e-12, inner_cap: int = 50, sweep_tol: float = 1e-10, max_sweeps: int = 200,
                 fixed_sweeps: int = 0, nu1: int = 2, nu2: int = 2, omega: float = 0.8, guess: int = 0,
                 residual_kind: int = 0, w_tol: float = 1e-6, w_cap: int = 50, bc: int = BC_DIRICHLET,
                 mlsdc_levels: int = 0, coarse_sweeps: int = 1,
                 device: Optional[torch.device] = None, stream: Optional[torch.cuda.Stream] = None):
        if not torch.cuda.is_available():
            raise RuntimeError("ISDC needs a CUDA device (no CPU fallback)")
        self.L = lib()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        p = _Problem()
        p.grid.dim, p.grid.n, p.grid.coarsest_n, p.grid.bc = dim, n, 0, bc
        p.M, p.nodes, p.dt, p.nu, p.fe = M, 0, dt, nu, fe
        for i in range(3):
            p.fe_params[i] = fe_a[i]
        self._G = None
        if fe == FE_FORCING:
            if G is None:
                raise ValueError("forcing needs G")
            self._G = torch.as_tensor(G, dtype=torch.float64).to(self.device).contiguous()
            p.fe_field_dev = self._G.data_ptr()
        p.mg.nu1, p.mg.nu2, p.mg.omega = nu1, nu2, omega
        s = p.solve
        s.mode, s.L, s.inner_tol, s.inner_cap = mode, L, inner_tol, inner_cap
        s.sweep_tol, s.max_sweeps, s.fixed_sweeps, s.guess = sweep_tol, max_sweeps, fixed_sweeps, guess
        p.residual_kind, p.w_tol, p.w_cap = residual_kind, w_tol, w_cap
        p.mlsdc_levels, p.coarse_sweeps = mlsdc_levels, coarse_sweeps
        self.p = p
        self.dim, self.n, self.M = dim, n, M
        self.kmax = fixed_sweeps if fixed_sweeps > 0 else max_sweeps
        nb = C.c_size_t(0)
        self._check(self.L.isdc_workspace_bytes(C.byref(p), C.byref(nb)))
        self.workspace_bytes = nb.value
        self.ws = torch.empty(max(nb.value, 1), dtype=torch.uint8, device=self.device)
        h = _vp()
        self._check(self.L.isdc_create(C.byref(p), self.ws.data_ptr(), nb.value, self.stream.cuda_stream, C.byref(h)))
        self.h = h
        self._G = None  # copied at create

    @classmethod
    def from_config(cls, cfg, G=None, mode=MODE_ISDC, **kw):
        return cls(cfg.dim, cfg.n, cfg.M, cfg.dt, cfg.nu, cfg.fe, cfg.fe_a, G, mode=mode, L=cfg.L,
                   inner_tol=cfg.inner_tol, inner_cap=cfg.inner_cap, sweep_tol=cfg.sweep_tol,
                   max_sweeps=cfg.max_sweeps, fixed_sweeps=cfg.fixed_sweeps, nu1=cfg.nu1, nu2=cfg.nu2,
                   omega=cfg.omega, bc=getattr(cfg, "bc", BC_DIRICHLET), **kw)

    # ------------------------------------------------------------------ plumbing
    def _check(self, st):
        if st != 0:
            msg = ""
            if getattr(self, "h", None) is not None:
                msg = self.L.isdc_last_error(self.h).decode()
            raise IsdcError(st, msg)

    def _check_shape(self, t):
        if tuple(t.shape) != (self.n,) * self.dim:
            raise ValueError(f"field shape {tuple(t.shape)} != {(self.n,) * self.dim}")

    def _field(self, x) -> torch.Tensor:
        """A dense device field for the library.  A copy made here lives on torch's current stream:
        the handle's stream waits for it and the tensor is recorded on that stream, so neither the
        copy nor the caching allocator can race the library's stream-ordered reads."""
        t = torch.as_tensor(x, dtype=torch.float64).to(self.device).contiguous()
        self._check_shape(t)
        cur = torch.cuda.current_stream(self.device)
        if cur.cuda_stream != self.stream.cuda_stream:
            self.stream.wait_stream(cur)
            t.record_stream(self.stream)
        return t

    def empty_field(self) -> torch.Tensor:
        return torch.empty((self.n,) * self.dim, dtype=torch.float64, device=self.device)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.L.isdc_destroy(self.h)
                self.h = None
        except Exception:
            pass

    # ------------------------------------------------------------------ API
    def set_initial(self, u0, step_index: int = 0):
        """u0: device tensor, or a host numpy array / CPU tensor (copied H2D by the library)."""
        if isinstance(u0, np.ndarray) or (isinstance(u0, torch.Tensor) and not u0.is_cuda):
            a = np.ascontiguousarray(u0 if isinstance(u0, np.ndarray) else u0.numpy(), dtype=np.float64)
            self._check_shape(a)
            self._host_u0 = a
            self._check(self.L.isdc_set_initial_host(self.h, _np_ptr(a), step_index))
        else:
            t = self._field(u0)
            self._check(self.L.isdc_set_initial(self.h, t.data_ptr(), step_index))

    def set_state(self, fields: Sequence, step_index: int = 0):
        ts = [self._field(f) for f in fields]
        arr = (_vp * self.M)(*[t.data_ptr() for t in ts])
        self._check(self.L.isdc_set_state(self.h, arr, step_index))

    def sweep(self):
        per = np.zeros(self.M - 1)
        mx = C.c_double(0)
        cyc = (C.c_int * (self.M - 1))()
        self._check(self.L.isdc_sweep(self.h, _np_ptr(per), C.byref(mx), cyc))
        return per, mx.value, list(cyc)

    def step(self):
        st = _Stats()
        hist = np.zeros(self.kmax)
        ncyc = (C.c_int * (self.kmax * (self.M - 1)))()
        self._check(self.L.isdc_step(self.h, C.byref(st), _np_ptr(hist), ncyc))
        k = st.sweeps
        return dict(sweeps=k, vcycles=st.vcycles, cap_hits=st.cap_hits, converged=bool(st.converged),
                    final_residual=st.final_residual, res_hist=hist[:k].copy(), wcycles=st.wcycles,
                    coarse_vcycles=st.coarse_vcycles,
                    node_cycles=np.array(ncyc[: k * (self.M - 1)]).reshape(k, self.M - 1))

    def run(self, nsteps: int):
        sts = (_Stats * max(nsteps, 1))()
        self._check(self.L.isdc_run(self.h, nsteps, sts))
        return [dict(sweeps=s.sweeps, vcycles=s.vcycles, cap_hits=s.cap_hits, converged=bool(s.converged),
                     final_residual=s.final_residual) for s in list(sts)[:nsteps]]

    def vcycle(self, m: int, b, u: torch.Tensor):
        """One V-cycle in place on the device tensor u; returns (defect_before, defect_after)."""
        bt = self._field(b)
        if not (u.is_cuda and u.dtype == torch.float64 and u.is_contiguous()):
            raise ValueError("u must be a contiguous float64 CUDA tensor (updated in place)")
        self._check_shape(u)   # mg_vcycle writes n^d doubles into u
        d0, d1 = C.c_double(0), C.c_double(0)
        self._check(self.L.mg_vcycle(self.h, m, bt.data_ptr(), u.data_ptr(), C.byref(d0), C.byref(d1)))
        return d0.value, d1.value

    def residual(self):
        per = np.zeros(self.M - 1)
        mx = C.c_double(0)
        self._check(self.L.residual_norm(self.h, _np_ptr(per), C.byref(mx)))
        return mx.value, per

    def solution(self, node: int = -1, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        node = node % self.M
        out = self.empty_field() if out is None else out
        if not (out.is_cuda and out.dtype == torch.float64 and out.is_contiguous()):
            raise ValueError("out must be a contiguous float64 CUDA tensor")
        self._check_shape(out)
        self._check(self.L.isdc_get_solution(self.h, node, out.data_ptr()))
        return out

    def solution_host(self, node: int = -1, out: Optional[np.ndarray] = None) -> np.ndarray:
        node = node % self.M
        out = np.empty((self.n,) * self.dim) if out is None else out
        if out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous float64 array")
        self._check_shape(out)
        self._check(self.L.isdc_get_solution_host(self.h, node, _np_ptr(out)))
        return out

    def tables(self):
        M = self.M
        tau, Q, S, dtau = np.zeros(M), np.zeros((M, M)), np.zeros((M - 1, M)), np.zeros(M - 1)
        self._check(self.L.isdc_get_tables(self.h, _np_ptr(tau), _np_ptr(Q), _np_ptr(S), _np_ptr(dtau)))
        return tau, Q, S, dtau

    def rhs(self, m: int, uold: Sequence, unew_m, step_index: int = 0) -> torch.Tensor:
        """b of Eq. (5) for substep m; note it overwrites the handle's iterate state."""
        ts = [self._field(f) for f in uold]
        un = self._field(unew_m)
        out = self.empty_field()
        arr = (_vp * self.M)(*[t.data_ptr() for t in ts])
        self.set_initial(un, step_index)
        self._check(self.L.isdc_rhs(self.h, m, arr, un.data_ptr(), out.data_ptr()))
        return out

    # ------------------------------------------------------------------ PFASST slice (R33)
    def coarse_n(self) -> int:
        return (self.n - 1) // 2

    def pfasst_set_u0(self, u0):
        """Forward transfer (R33 step 1): node 0 of the fine iterate <- u0 (dense device field)."""
        t = self._field(u0)
        self._check(self.L.isdc_pfasst_set_u0(self.h, t.data_ptr()))

    def pfasst_restrict(self):
        """Phase B: injection + FAS from the current fine iterate (the spread state in the predictor)."""
        self._check(self.L.isdc_pfasst_restrict(self.h))

    def pfasst_coarse(self, U0=None, out: Optional[torch.Tensor] = None):
        """Phase C: coarse node 0 <- U0 (dense n_c^d, None keeps it), coarse sweeps; returns (coarse
        end value, coarse V-cycles)."""
        nc = self.coarse_n()
        ptr = None
        if U0 is not None:
            t = torch.as_tensor(U0, dtype=torch.float64).to(self.device).contiguous()
            if tuple(t.shape) != (nc,) * self.dim:
                raise ValueError(f"coarse field shape {tuple(t.shape)} != {(nc,) * self.dim}")
            cur = torch.cuda.current_stream(self.device)
            if cur.cuda_stream != self.stream.cuda_stream:
                self.stream.wait_stream(cur)
                t.record_stream(self.stream)
            ptr, self._U0_keep = t.data_ptr(), t
        out = torch.empty((nc,) * self.dim, dtype=torch.float64, device=self.device) if out is None else out
        cv = C.c_long(0)
        self._check(self.L.isdc_pfasst_coarse(self.h, ptr, out.data_ptr(), C.byref(cv)))
        return out, cv.value

    def pfasst_interpolate(self, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Phase D: u_j += P4(U_j - Ubar_j); returns the fine end value u_M (dense device field)."""
        out = self.empty_field() if out is None else out
        self._check_shape(out)
        self._check(self.L.isdc_pfasst_interpolate(self.h, out.data_ptr()))
        return out

    def profile(self, level: int = 1):
        """0 off, 1 the fine-level kernel classes, 2 every class, 16 + c class c only (bench's timed region)."""
        self._check(self.L.isdc_profile_enable(self.h, int(level)))

    def profile_reset(self):
        self._check(self.L.isdc_profile_reset(self.h))

    def profile_get(self):
        """{class: (total_ms, launches, algorithmic_bytes)} accumulated since the last reset."""
        out = {}
        for cls, name in PROFILE_CLASSES.items():
            ms, n, by = C.c_double(0), C.c_long(0), C.c_double(0)
            self._check(self.L.isdc_profile_get(self.h, cls, C.byref(ms), C.byref(n), C.byref(by)))
            out[name] = (ms.value, n.value, by.value)
        return out

    @property
    def launches(self) -> int:
        return int(self.L.isdc_kernel_launches(self.h))
