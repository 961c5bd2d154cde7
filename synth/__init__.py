"""Seeded synthetic inputs for the ISDC hot path (shared by the oracle tests and the CUDA path).

This module holds NONE of the method's arithmetic: it only draws random numbers and samples the
initial data / forcing field of the five BASELINE.json configs.  Both the CPU
oracle (``oracle/``) and the CUDA library receive the same float64 bits from here.

Recipes (readings in DESIGN.md §3):

====  ==========================================================================================
cfg   draws (numpy ``default_rng(seed)``, PCG64; integers first, then amplitudes)
====  ==========================================================================================
1     kl = integers(1, 9, (8, 2));   a = standard_normal(8)          u0 = Σ a sin(kπx) sin(lπy)
2     kl = integers(1, 33, (32, 2)); a = 0.1*standard_normal(32)
3     kl = integers(1, 65, (64, 2)); a = 0.1*standard_normal(64);   G = sin(2πx) sin(2πy)
4     kln = integers(1, 9, (16, 3)); a = standard_normal(16)        u0 = Σ a sin sin sin
5     c = uniform(0.3, 0.7, 3);      u0 = exp(-|x-c|^2 / 0.01)       (Gaussian blob)
B     (NEXT f3, viscous Burgers P:106-112, periodic [-1,1)^2): seed 0: u0 = exp(-|x|^2/sigma^2),
      sigma = 0.1 (x read as the vector (x, y)); seed s > 0: c = uniform(-0.5, 0.5, 2),
      A = uniform(0.5, 1.5); u0 = A exp(-|x-c|^2/sigma^2)
====  ==========================================================================================

Grid: n interior points per direction, N = n + 1 = 2^p, x_i = i / N for i = 1..n (h = 1/N).
Periodic grids (Burgers): n = 2^p points x_i = -1 + i h, i = 0..n-1, h = 2/n.
Arrays are C-contiguous, shape (n, n) or (n, n, n), x fastest (index [z, y, x]).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

FE_NONE, FE_CUBIC, FE_FORCING, FE_ADVECTION, FE_BURGERS = 0, 1, 2, 3, 4
MODE_ISDC, MODE_SDC, MODE_ISDC_CAPPED = 0, 1, 2
BC_DIRICHLET, BC_PERIODIC = 0, 1


@dataclasses.dataclass
class Config:
    """One BASELINE.json config (numbered 1..5 in file order)."""

    cid: int
    dim: int
    n: int
    M: int
    dt: float
    nu: float
    fe: int
    fe_a: tuple = (0.0, 0.0, 0.0)
    steps: int = 1
    sweep_tol: float = 1e-10
    max_sweeps: int = 200
    fixed_sweeps: int = 0
    modes: tuple = (MODE_ISDC,)
    L: int = 2
    inner_tol: float = 1e-12
    inner_cap: int = 50
    nu1: int = 2
    nu2: int = 2
    omega: float = 0.8
    bc: int = BC_DIRICHLET


# SURVEY.md §8 per-config table; stop rules per the DESIGN.md readings (c2 items 19, 25, 26).
CONFIGS = {
    1: Config(1, 2, 63, 3, 0.01, 1.0, FE_NONE, steps=1, fixed_sweeps=8,
              modes=(MODE_ISDC, MODE_SDC)),
    2: Config(2, 2, 1023, 5, 0.005, 1e-3, FE_CUBIC, steps=10),
    3: Config(3, 2, 4095, 5, 0.01, 0.1, FE_FORCING, steps=1, modes=(MODE_ISDC, MODE_SDC)),
    4: Config(4, 3, 255, 3, 0.01, 1.0, FE_NONE, steps=1),
    5: Config(5, 3, 511, 5, 0.002, 0.01, FE_ADVECTION, fe_a=(1.0, 0.5, 0.25), steps=5),
}


def grid_x(n: int) -> np.ndarray:
    """Interior coordinates x_i = i/N, i = 1..n (exact in binary since N = n+1 is a power of 2)."""
    N = n + 1
    if N & (N - 1):
        raise ValueError(f"n+1 must be a power of two, got n={n}")
    return np.arange(1, n + 1, dtype=np.float64) / float(N)


def _sine_modes(n: int, dim: int, nmodes: int, kmax: int, amp: float, seed: int):
    rng = np.random.default_rng(seed)
    ks = rng.integers(1, kmax + 1, size=(nmodes, dim))
    a = amp * rng.standard_normal(nmodes)
    x = grid_x(n)
    u = np.zeros((n,) * dim, dtype=np.float64)
    for p in range(nmodes):
        s = [np.sin(float(ks[p, ax]) * math.pi * x) for ax in range(dim)]
        if dim == 2:
            u += a[p] * np.multiply.outer(s[1], s[0])
        else:
            u += a[p] * np.multiply.outer(np.multiply.outer(s[2], s[1]), s[0])
    return u, ks, a


def initial_condition(cid: int, seed: int = 0, n: Optional[int] = None) -> np.ndarray:
    """u0 for config ``cid`` with the given seed; ``n`` overrides the grid size (reduced parity cases)."""
    cfg = CONFIGS[cid]
    n = cfg.n if n is None else n
    if cid == 1:
        return _sine_modes(n, 2, 8, 8, 1.0, seed)[0]
    if cid == 2:
        return _sine_modes(n, 2, 32, 32, 0.1, seed)[0]
    if cid == 3:
        return _sine_modes(n, 2, 64, 64, 0.1, seed)[0]
    if cid == 4:
        return _sine_modes(n, 3, 16, 8, 1.0, seed)[0]
    if cid == 5:
        rng = np.random.default_rng(seed)
        c = rng.uniform(0.3, 0.7, 3)
        x = grid_x(n)
        gx = np.exp(-((x - c[0]) ** 2) / 0.01)
        gy = np.exp(-((x - c[1]) ** 2) / 0.01)
        gz = np.exp(-((x - c[2]) ** 2) / 0.01)
        return np.multiply.outer(np.multiply.outer(gz, gy), gx)
    raise ValueError(cid)


def forcing_field(n: int, dim: int = 2) -> np.ndarray:
    """G(x) = sin(2πx) sin(2πy) [sin(2πz)] sampled on the interior (config 3's forcing profile)."""
    s = np.sin(2.0 * math.pi * grid_x(n))
    if dim == 2:
        return np.multiply.outer(s, s)
    return np.multiply.outer(np.multiply.outer(s, s), s)


def sine_mode(n: int, ks) -> np.ndarray:
    """A single discrete sine mode Π_a sin(k_a π x_a) (used by the pins)."""
    x = grid_x(n)
    s = [np.sin(float(k) * math.pi * x) for k in ks]
    if len(ks) == 2:
        return np.multiply.outer(s[1], s[0])
    return np.multiply.outer(np.multiply.outer(s[2], s[1]), s[0])


def random_field(n: int, dim: int, seed: int) -> np.ndarray:
    """Uniform(-1,1) field, for operator-level parity cases."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, size=(n,) * dim)


def problem_inputs(cid: int, seed: int = 0, n: Optional[int] = None):
    """(cfg, u0, G-or-None) for config ``cid``; reduced grids keep every other parameter."""
    cfg = CONFIGS[cid]
    nn = cfg.n if n is None else n
    cfg = dataclasses.replace(cfg, n=nn)
    u0 = initial_condition(cid, seed, nn)
    G = forcing_field(nn, cfg.dim) if cfg.fe == FE_FORCING else None
    return cfg, u0, G


# ------------------------------------------------------------------ viscous Burgers (NEXT f3)
def grid_x_periodic(n: int) -> np.ndarray:
    """Periodic coordinates x_i = -1 + i h, h = 2/n, i = 0..n-1 (exact: n is a power of two)."""
    if n < 4 or n & (n - 1):
        raise ValueError(f"periodic n must be a power of two >= 4, got n={n}")
    return -1.0 + np.arange(n, dtype=np.float64) * (2.0 / float(n))


def burgers_config(nu: float, M: int, n: int = 128, dt: float = 0.001, **kw) -> Config:
    """Table 1b problem: 2D viscous Burgers on [-1,1)^2, periodic, IMEX
    with WENO5 advection; h = 1/64 (n = 128, reading R30), dt = 0.001, one step, L = 2,
    residual tolerance 5e-8."""
    base = dict(steps=1, sweep_tol=5e-8, max_sweeps=100, bc=BC_PERIODIC)
    base.update(kw)
    return Config(0, 2, n, M, dt, float(nu), FE_BURGERS, **base)


def burgers_initial(n: int, seed: int = 0, sigma: float = 0.1, dim: int = 2) -> np.ndarray:
    """u0 = A exp(-|x - c|^2 / sigma^2) on the periodic grid (seed 0: A = 1, c = 0)."""
    x = grid_x_periodic(n)
    if seed == 0:
        c, A = np.zeros(dim), 1.0
    else:
        rng = np.random.default_rng(seed)
        c = rng.uniform(-0.5, 0.5, dim)
        A = rng.uniform(0.5, 1.5)
    g = [np.exp(-((x - c[a]) ** 2) / (sigma * sigma)) for a in range(dim)]
    if dim == 2:
        return A * np.multiply.outer(g[1], g[0])
    return A * np.multiply.outer(np.multiply.outer(g[2], g[1]), g[0])
