"""ORACLE — test infrastructure, not product (see oracle/__init__.py).

CPU restatement of the EDGC reference's data-parallel hot path, in float64
NumPy exactly as the reference computes it.  Each function cites the
reference lines it restates (paths relative to /root/reference/pkg/src/edgc)
or, for third-party arithmetic, the NumPy 2.3.5 source it restates.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

__all__ = [
    "TAG_SYNTH", "TAG_SUBSAMPLE", "TAG_BASIS", "COLUMN_TOL", "GAUSS_CONST",
    "pcg64_words", "subsample_seed", "sample_count", "choice_branch", "choice_indices",
    "pcg64_u32", "subsample", "gaussian_entropy", "fd_histogram", "histogram_entropy",
    "OracleState", "basis_column", "orthonormalize", "compress", "decompress", "set_rank",
    "state_seeds", "dp_step", "synth_matrix", "GPT2_2P5B_LAYER", "GPT2_12P1B_LAYER",
]

# seeds.py:14-16
TAG_SYNTH = 1
TAG_SUBSAMPLE = 2
TAG_BASIS = 3
# compressor.py:23
COLUMN_TOL = 1e-12
# entropy.py:24
GAUSS_CONST = 0.5 * math.log(2.0 * math.pi * math.e)

# per-layer weight-gradient shapes (QKV, proj, fc1, fc2)
GPT2_2P5B_LAYER = ((1920, 5760), (1920, 1920), (1920, 7680), (7680, 1920))
GPT2_12P1B_LAYER = ((3584, 10752), (3584, 3584), (3584, 14336), (14336, 3584))

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _npchoice():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "_build", "liboracle_npchoice.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        lib = ctypes.CDLL(path)
        lib.oracle_choice.restype = ctypes.c_int64
        lib.oracle_choice.argtypes = [ctypes.c_uint64] * 4 + [ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
        lib.oracle_pcg64_u32.restype = None
        lib.oracle_pcg64_u32.argtypes = [ctypes.c_uint64] * 4 + [ctypes.c_int64, ctypes.c_void_p]
        _LIB = lib
    return _LIB


def pcg64_words(seed):
    """(state_hi, state_lo, inc_hi, inc_lo) of np.random.default_rng(seed)'s PCG64."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    mask = (1 << 64) - 1
    s, i = int(st["state"]), int(st["inc"])
    return (s >> 64) & mask, s & mask, (i >> 64) & mask, i & mask


def subsample_seed(run_seed: int, iteration: int, layer: int) -> int:
    """entropy.py:170-174 with seeds.py:26-28: per-(iteration, layer) sampler seed."""
    return int(np.random.default_rng([run_seed, TAG_SUBSAMPLE, iteration, layer]).integers(2**31))


def sample_count(n_elems: int, beta: float) -> int:
    """entropy.py:75."""
    return min(n_elems, math.ceil(beta * n_elems))


def choice_branch(n_elems: int, count: int) -> str:
    return "tail" if (n_elems > 10000 and count > n_elems // 20) else "floyd"


def choice_indices(seed: int, n_elems: int, count: int) -> np.ndarray:
    """entropy.py:78 index sequence (npchoice.c restates NumPy's Generator.choice)."""
    out = np.empty(count, dtype=np.int64)
    if count:
        rc = _npchoice().oracle_choice(*pcg64_words(seed), n_elems, count, out.ctypes.data)
        if rc < 0:
            raise ValueError(f"oracle_choice rejected N={n_elems} count={count}")
    return out


def pcg64_u32(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint32)
    _npchoice().oracle_pcg64_u32(*pcg64_words(seed), n, out.ctypes.data)
    return out


def subsample(matrix, beta: float, seed: int) -> np.ndarray:
    """entropy.py:67-79: ceil(beta*N) row-major entries without replacement."""
    flat = np.asarray(matrix, dtype=np.float64).ravel()
    count = sample_count(flat.size, beta)
    if count == flat.size:
        return flat.copy()
    return flat[choice_indices(seed, flat.size, count)]


def gaussian_entropy(samples) -> float:
    """entropy.py:82-90; std(ddof=1) restated from numpy/_core/_methods.py:_var (two-pass)."""
    x = np.asarray(samples, dtype=np.float64).ravel()
    n = x.size
    if n < 2:
        raise ValueError("need at least 2 samples")
    mean = np.add.reduce(x) / n
    dev = x - mean
    var = np.add.reduce(dev * dev) / (n - 1)
    sigma = math.sqrt(float(var))
    if sigma == 0.0:
        raise ValueError("degenerate: zero variance")
    return math.log(sigma) + GAUSS_CONST


def _lerp(a: float, b: float, t: float) -> float:
    """numpy/lib/_function_base_impl.py:4657-4678 (_lerp), scalar form."""
    diff = b - a
    out = a + diff * t
    if t >= 0.5:
        out = b - diff * (1 - t)
    return out


def _percentile_linear(sorted_x: np.ndarray, q: float) -> float:
    """numpy/lib/_function_base_impl.py:126-128 ((n-1)*q), 4753-4785 (_get_indexes)."""
    n = sorted_x.size
    virtual = (n - 1) * q
    if virtual >= n - 1:
        return float(sorted_x[-1])
    lo = math.floor(virtual)
    gamma = virtual - lo
    return _lerp(float(sorted_x[lo]), float(sorted_x[lo + 1]), gamma)


def fd_histogram(samples):
    """np.histogram(x, bins="fd") restated step by step (NumPy 2.3.5).

    numpy/lib/_histograms_impl.py:200-227 (_hist_bin_fd), 298-326 (outer edges),
    392-443 (n_equal_bins, linspace edges, too-many-bins check),
    818-873 (uniform-bin index rule + bincount);
    numpy/_core/function_base.py:139-172 (linspace).
    Returns (counts int64[nb], edges float64[nb+1]).
    """
    x = np.asarray(samples, dtype=np.float64).ravel()
    s = np.sort(x)
    first, last = float(s[0]), float(s[-1])
    if first == last:
        first, last = first - 0.5, last + 0.5
    iqr = _percentile_linear(s, 0.75) - _percentile_linear(s, 0.25)
    width = 2.0 * iqr * x.size ** (-1.0 / 3.0)
    delta = last - first
    nb = int(math.ceil(delta / width)) if width else 1
    step = delta / nb
    if step == 0.0:
        edges = (np.arange(nb + 1, dtype=np.float64) / nb) * delta
    else:
        edges = np.arange(nb + 1, dtype=np.float64) * step
    edges += first
    edges[-1] = last
    if np.any(edges[:-1] >= edges[1:]):
        raise ValueError(f"Too many bins for data range. Cannot create {nb} finite-sized bins.")
    idx = (((x - first) / delta) * nb).astype(np.intp)
    idx[idx == nb] -= 1
    idx[x < edges[idx]] -= 1
    bump = (x >= edges[idx + 1]) & (idx != nb - 1)
    idx[bump] += 1
    return np.bincount(idx, minlength=nb).astype(np.int64), edges


def histogram_entropy(samples) -> float:
    """entropy.py:93-107 with the FD rule."""
    x = np.asarray(samples, dtype=np.float64).ravel()
    if x.size < 2:
        raise ValueError("need at least 2 samples")
    if float(x.max()) == float(x.min()):
        raise ValueError("degenerate: zero range")
    counts, edges = fd_histogram(x)
    widths = np.diff(edges)
    p = counts / counts.sum()
    nz = p > 0
    return float(-(p[nz] * np.log(p[nz] / widths[nz])).sum())


# ---------------------------------------------------------------- compressor


def basis_column(rng_seed: int, j: int, n: int) -> np.ndarray:
    """compressor.py:63-66: fixed fresh column j = rng(seed, TAG_BASIS, j).standard_normal(n)."""
    return np.random.default_rng([rng_seed, TAG_BASIS, j]).standard_normal(n)


class OracleState:
    """compressor.py:45-61: residual zeros(m, n) and seeded warm-start basis."""

    def __init__(self, m: int, n: int, rank: int, rng_seed: int = 0):
        if not 1 <= rank <= min(m, n):
            raise ValueError("rank out of range")
        self.m, self.n, self.rank, self.rng_seed = m, n, rank, rng_seed
        self.residual = np.zeros((m, n))
        self.q_warm = np.stack([basis_column(rng_seed, j, n) for j in range(rank)], axis=1)


def orthonormalize(p: np.ndarray) -> np.ndarray:
    """compressor.py:74-91: in-place MGS, tolerance fixed before the sweep."""
    tol = COLUMN_TOL * np.linalg.norm(p)
    dead = np.zeros(p.shape[1], dtype=bool)
    for j in range(p.shape[1]):
        v = p[:, j]
        for i in range(j):
            v -= (p[:, i] @ v) * p[:, i]
        nrm = np.linalg.norm(v)
        if nrm > tol:
            v /= nrm
        else:
            v[:] = 0.0
            dead[j] = True
    return dead


def compress(matrix, st: OracleState):
    """compressor.py:94-123.  Returns (p, q, dead)."""
    a = np.asarray(matrix, dtype=np.float64)
    if a.shape != (st.m, st.n):
        raise ValueError("shape mismatch")
    work = a + st.residual
    if not np.isfinite(work).all():
        raise ValueError("non-finite entries in gradient or residual")
    p = work @ st.q_warm
    dead = orthonormalize(p)
    q = work.T @ p
    st.residual = work - p @ q.T
    for j in np.flatnonzero(dead):
        q[:, j] = basis_column(st.rng_seed, int(j), st.n)
    st.q_warm = q
    return p, q, dead


def decompress(p: np.ndarray, q: np.ndarray) -> np.ndarray:
    """compressor.py:126-133 (the GradientMatrix wrapper only validates)."""
    return p @ q.T


def set_rank(st: OracleState, r_new: int) -> None:
    """compressor.py:136-151."""
    if not 1 <= r_new <= min(st.m, st.n):
        raise ValueError("rank out of range")
    if r_new < st.rank:
        st.q_warm = st.q_warm[:, :r_new].copy()
    elif r_new > st.rank:
        extra = np.stack([basis_column(st.rng_seed, j, st.n) for j in range(st.rank, r_new)], axis=1)
        st.q_warm = np.concatenate([st.q_warm, extra], axis=1)
    st.rank = r_new


# ------------------------------------------------------------------- DP step


def state_seeds(seed: int, workers: int, layers: int) -> dict:
    """grad_source.py:440-447: per-(worker, layer) basis seeds."""
    kids = np.random.SeedSequence([seed, TAG_BASIS]).spawn(workers * layers)
    return {(w, k): int(kids[w * layers + k].generate_state(1)[0])
            for w in range(workers) for k in range(layers)}


def dp_step(grads, states):
    """grad_source.py:389-408: per-worker compress->decompress, worker-order sum, /W.

    grads[w][k] are worker w's layer-k gradients, states[w][k] their OracleStates.
    """
    workers = len(grads)
    sums = None
    for w in range(workers):
        recon = []
        for k, g in enumerate(grads[w]):
            p, q, _ = compress(g, states[w][k])
            recon.append(decompress(p, q))
        if sums is None:
            sums = [np.zeros_like(r) for r in recon]
        for k, r in enumerate(recon):
            sums[k] += r
    return [s / workers for s in sums]


def synth_matrix(seed: int, t: int, k: int, w: int, m: int, n: int, sigma: float) -> np.ndarray:
    """fp32-representable synthetic gradient: TAG_SYNTH stream scaled in fp32."""
    z = np.random.default_rng([seed, TAG_SYNTH, t, k, w]).standard_normal((m, n), dtype=np.float32)
    return z * np.float32(sigma)
