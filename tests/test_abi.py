"""CPU-side checks of the C-ABI library: it builds, loads, exports every symbol include/isdc.h
declares, validates arguments without a GPU, and its host-built tables equal the oracle's bits."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_1401_7824_b200 import build
    build.build()
    import paper_1401_7824_b200 as pk
    return pk.lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "isdc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_]+\s*\*?\s*([a-z_]+)\s*\(", src, flags=re.M)))


def test_exports_every_declared_symbol(L):
    syms = declared_symbols()
    assert len(syms) >= 18, syms
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_workspace_and_validation_without_gpu(L):
    from paper_1401_7824_b200.isdc import _Problem
    p = _Problem()
    p.grid.dim, p.grid.n, p.grid.coarsest_n, p.grid.bc = 2, 63, 3, 0
    p.M, p.dt, p.nu = 3, 0.01, 1.0
    p.mg.nu1 = p.mg.nu2 = 2
    p.mg.omega = 0.8
    p.solve.L, p.solve.max_sweeps = 2, 200
    nb = C.c_size_t(0)
    assert L.isdc_workspace_bytes(C.byref(p), C.byref(nb)) == 0
    # 2 iterate sets (2M-1 fields) + 4 scratch, each 63*64 doubles, plus the coarse levels
    assert nb.value >= (2 * 3 - 1 + 4) * 63 * 64 * 8
    for field, bad, code in [("n", 62, 1), ("n", 0, 1), ("dim", 4, 1), ("M", 9, 2), ("M", 1, 2)]:
        q = _Problem.from_buffer_copy(p)
        if field in ("n", "dim"):
            setattr(q.grid, field, bad)
        else:
            setattr(q, field, bad)
        assert L.isdc_workspace_bytes(C.byref(q), C.byref(nb)) == code, (field, bad)
    q = _Problem.from_buffer_copy(p)
    q.dt = 0.0
    assert L.isdc_workspace_bytes(C.byref(q), C.byref(nb)) == 1
    q = _Problem.from_buffer_copy(p)
    q.nodes = 2
    assert L.isdc_workspace_bytes(C.byref(q), C.byref(nb)) == 2
    q = _Problem.from_buffer_copy(p)
    q.fe = 2  # forcing without a field
    assert L.isdc_workspace_bytes(C.byref(q), C.byref(nb)) == 1
    # periodic grids (NEXT f3): n = 2^p points, coarsest 4; WENO5 Burgers only on periodic grids
    q = _Problem.from_buffer_copy(p)
    q.fe = 4
    assert L.isdc_workspace_bytes(C.byref(q), C.byref(nb)) == 2
    q.grid.bc, q.grid.n, q.grid.coarsest_n = 1, 128, 0
    assert L.isdc_workspace_bytes(C.byref(q), C.byref(nb)) == 0
    assert nb.value >= (2 * 3 - 1 + 4) * 128 * 128 * 8
    for n, cn, code in [(127, 0, 1), (96, 0, 1), (128, 3, 1), (128, 4, 0), (4, 0, 0)]:
        q.grid.n, q.grid.coarsest_n = n, cn
        assert L.isdc_workspace_bytes(C.byref(q), C.byref(nb)) == code, (n, cn)
    q.grid.bc = 2
    assert L.isdc_workspace_bytes(C.byref(q), C.byref(nb)) == 1
    # two-level MLSDC (NEXT f4): Dirichlet, n >= 7, ISDC mode, weighted residual; the coarse handle's
    # workspace and the transfer fields are part of the caller's workspace
    one = C.c_size_t(0)
    assert L.isdc_workspace_bytes(C.byref(p), C.byref(one)) == 0
    q = _Problem.from_buffer_copy(p)
    q.mlsdc_levels, q.coarse_sweeps = 2, 1
    assert L.isdc_workspace_bytes(C.byref(q), C.byref(nb)) == 0
    assert nb.value > one.value + (3 - 1) * 63 * 64 * 8
    for field, bad, code in [("coarse_sweeps", -1, 1), ("mlsdc_levels", 3, 1)]:
        r = _Problem.from_buffer_copy(q)
        setattr(r, field, bad)
        assert L.isdc_workspace_bytes(C.byref(r), C.byref(nb)) == code, field
    r = _Problem.from_buffer_copy(q)
    r.solve.mode = 1
    assert L.isdc_workspace_bytes(C.byref(r), C.byref(nb)) == 2
    r = _Problem.from_buffer_copy(q)
    r.grid.n = 3
    assert L.isdc_workspace_bytes(C.byref(r), C.byref(nb)) == 2
    r = _Problem.from_buffer_copy(q)
    r.residual_kind = 1
    assert L.isdc_workspace_bytes(C.byref(r), C.byref(nb)) == 2
    # create refuses a missing / too-small workspace before touching the device
    h = C.c_void_p()
    assert L.isdc_create(C.byref(p), None, 0, None, C.byref(h)) == 5


@pytest.mark.parametrize("M", range(2, 9))
def test_library_tables_equal_oracle_bits(L, ora, M):
    dp = C.POINTER(C.c_double)
    tau, Q, S, dtau = np.zeros(M), np.zeros(M * M), np.zeros((M - 1) * M), np.zeros(M - 1)
    assert L.isdc_build_tables(M, *[a.ctypes.data_as(dp) for a in (tau, Q, S, dtau)]) == 0
    ot, oQ, oS, od = ora.tables(M)
    assert np.array_equal(tau, ot) and np.array_equal(Q, oQ.ravel())
    assert np.array_equal(S, oS.ravel()) and np.array_equal(dtau, od)


@pytest.mark.parametrize("dim,periodic", [(2, False), (3, False), (2, True), (3, True)])
def test_library_coarse_inverse_equals_oracle_bits(L, ora, dim, periodic):
    dp = C.POINTER(C.c_double)
    n = 4 if periodic else 3
    P = n ** dim
    for g in [0.0, 1e-5, 3e-3, 0.0172, 0.5]:
        c = ora.level_coefs(dim, n, g, periodic=periodic)
        Gi = np.zeros(P * P)
        assert L.isdc_coarse_inverse(dim, n, int(periodic), c[0], c[1], c[2], Gi.ctypes.data_as(dp)) == 0
        assert np.array_equal(Gi, ora.coarse_inverse(dim, g, periodic=periodic).ravel())
