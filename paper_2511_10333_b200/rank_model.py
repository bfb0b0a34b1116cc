"""Entropy-to-rank model (CQM), host side.

The Marchenko–Pastur g-table and its inversions are init-time / per-window
scalar work, so they stay in NumPy on the host.  Rank decisions must be
*identical* to the reference's, so every floating-point expression below is
evaluated in the same order and with the same NumPy primitives as
pkg/src/edgc/rank_model.py (line numbers cited per function); the layout of
the module is our own.
"""

from __future__ import annotations

import math
import threading
from dataclasses import dataclass

import numpy as np

__all__ = ["GRID_POINTS", "DEFAULT_TRIALS", "MpSupport", "mp_support", "mp_cdf", "sample_eigenvalues", "GTable",
           "build_g_table", "g_table", "estimate_g", "invert_g", "rank_from_sigma", "rank_from_entropy"]

GRID_POINTS = 1024
DEFAULT_TRIALS = 64


@dataclass(frozen=True)
class MpSupport:
    a: float
    b: float
    m: int
    n: int


def mp_support(m: int, n: int) -> MpSupport:
    """[a, b] = [(sqrt n - sqrt m)^2, (sqrt n + sqrt m)^2], m <= n (rank_model.py:37-45)."""
    if not 1 <= m <= n:
        raise ValueError(f"need 1 <= m <= n, got ({m}, {n}); transpose the matrix before modeling")
    rn, rm = math.sqrt(n), math.sqrt(m)
    return MpSupport(a=(rn - rm) ** 2, b=(rn + rm) ** 2, m=m, n=n)


def _cdf_interior(x: np.ndarray, a: float, b: float, m: int) -> np.ndarray:
    # closed form of rank_model.py:68-75, operation order preserved
    root = np.sqrt((x - a) * (b - x))
    arc_sin = (a + b) * np.arcsin(np.clip(np.sqrt((x - a) / (b - a)), 0.0, 1.0))
    arc_tan = 0.0
    if a > 0.0:
        arc_tan = -2.0 * math.sqrt(a * b) * np.arctan(np.sqrt(b * (x - a) / (a * (b - x))))
    return np.clip((arc_tan + arc_sin + root) / (2.0 * math.pi * m), 0.0, 1.0)


def mp_cdf(lam, m: int, n: int):
    """MP CDF of the eigenvalues of A A^T (rank_model.py:48-76); 0 below a, 1 above b."""
    sup = mp_support(m, n)
    arr = np.asarray(lam, dtype=np.float64)
    is_scalar = arr.ndim == 0
    arr = np.atleast_1d(arr)
    out = np.empty_like(arr)
    lo, hi = arr <= sup.a, arr >= sup.b
    mid = ~(lo | hi)
    out[lo] = 0.0
    out[hi] = 1.0
    if mid.any():
        out[mid] = _cdf_interior(arr[mid], sup.a, sup.b, m)
    return float(out[0]) if is_scalar else out


def _grid(m: int, n: int):
    sup = mp_support(m, n)
    lam = np.linspace(sup.a, sup.b, GRID_POINTS)
    return lam, np.asarray(mp_cdf(lam, m, n))


def sample_eigenvalues(m: int, n: int, seed: int = 0) -> np.ndarray:
    """m inverse-transform eigenvalue draws (rank_model.py:86-94)."""
    lam, cdf = _grid(m, n)
    return np.interp(np.random.default_rng(seed).uniform(size=m), cdf, lam)


@dataclass(frozen=True)
class GTable:
    """g_sq[r] ~ E||A - A_r||_F^2 for unit-variance m x n A; g_values = sqrt(g_sq)."""

    m: int
    n: int
    trials: int
    rng_seed: int
    g_sq: np.ndarray
    g_values: np.ndarray

    def g(self, r: int) -> float:
        if not 0 <= r <= self.m:
            raise ValueError(f"rank {r} outside [0, {self.m}]")
        return float(self.g_values[r])


def build_g_table(m: int, n: int, trials: int = DEFAULT_TRIALS, seed: int = 0) -> GTable:
    """Monte-Carlo table (rank_model.py:118-129): sort trials' eigenvalues, tail sums, mean."""
    if trials < 1:
        raise ValueError(f"trials must be positive, got {trials}")
    lam_grid, cdf = _grid(m, n)
    draws = np.interp(np.random.default_rng(seed).uniform(size=(trials, m)), cdf, lam_grid)
    draws.sort(axis=1)
    prefix = np.cumsum(draws, axis=1)            # prefix[:, k-1] = sum of the k smallest
    sq = np.zeros(m + 1)
    sq[:m] = prefix[:, ::-1].mean(axis=0)         # r -> sum of the m - r smallest
    return GTable(m=m, n=n, trials=trials, rng_seed=seed, g_sq=sq, g_values=np.sqrt(sq))


class _TableCache:
    def __init__(self):
        self._tables: dict = {}
        self._lock = threading.Lock()

    def get(self, key):
        with self._lock:
            tab = self._tables.get(key)
            if tab is None:
                tab = build_g_table(*key)
                self._tables[key] = tab
        return tab


_CACHE = _TableCache()


def g_table(m: int, n: int, trials: int = DEFAULT_TRIALS, seed: int = 0) -> GTable:
    """Cached, serialised construction (rank_model.py:136-144)."""
    return _CACHE.get((m, n, trials, seed))


def estimate_g(r: int, m: int, n: int, trials: int = DEFAULT_TRIALS, seed: int = 0) -> float:
    return g_table(m, n, trials, seed).g(r)


def invert_g(target_error: float, table: GTable) -> int:
    """Smallest r with g(r) <= target (rank_model.py:152-161); 0 and m saturate."""
    if target_error < 0.0:
        raise ValueError(f"target error must be non-negative, got {target_error}")
    pos = np.searchsorted(-table.g_values, -target_error, side="left")
    return min(int(pos), table.m)


def rank_from_sigma(r0: int, sigma0: float, sigma1: float, table: GTable) -> int:
    """Constant-error rank under a scale change: g^{-1}((s0/s1) g(r0)) (rank_model.py:164-172)."""
    if sigma0 <= 0.0 or sigma1 <= 0.0:
        raise ValueError(f"standard deviations must be positive, got {sigma0}, {sigma1}")
    return invert_g((sigma0 / sigma1) * table.g(r0), table)


def rank_from_entropy(r0: int, h0: float, h1: float, table: GTable) -> int:
    """Constant-error rank across an entropy change: g^{-1}(e^{h0-h1} g(r0)) (rank_model.py:175-190)."""
    if not (math.isfinite(h0) and math.isfinite(h1)):
        raise ValueError(f"entropies must be finite, got {h0}, {h1}")
    try:
        scale = math.exp(h0 - h1)
    except OverflowError:
        scale = math.inf
    target = scale * table.g(r0)
    return invert_g(target, table) if math.isfinite(target) else 0
