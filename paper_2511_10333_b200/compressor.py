"""Rank-r power-iteration compression with error feedback, on the device.

Mirrors pkg/src/edgc/compressor.py (names, argument meaning, errors) with the
arithmetic in libedgc_b200.so.  Device semantics:

* Storage is fp32; reductions are fp64.  The orthonormalisation is Cholesky-
  QR run twice on the fp64 P, which equals the reference's modified
  Gram-Schmidt (compressor.py:74-91) up to rounding, including its
  dead-column rule: a column whose projected norm is <= tol * ||P||_F is
  zeroed and its warm-start slot re-seeded with the fixed fresh column
  (compressor.py:113-114).  ``DEVICE_COLUMN_TOL`` is the fp32-storage
  counterpart of the reference's 1e-12.
* The error-feedback residual is kept as (w, p_res, q_res) with
  residual = w - p_res q_res^T (w = last step's work matrix); ``residual``
  materialises it on demand.  Same arithmetic as compressor.py:106-112.
* ``compress`` checks the work matrix for non-finite entries before touching
  any state, as compressor.py:106-108 does.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .matrix_core import GradientMatrix, as_device_array, as_device_matrix
from .seeds import TAG_BASIS, rng

__all__ = ["LowRankFactors", "CompressorState", "compress", "decompress", "set_rank", "compressed_element_count",
           "basis_columns", "DEVICE_COLUMN_TOL"]

_COLUMN_TOL = 1e-12          # the reference's fp64 value (compressor.py:23)
DEVICE_COLUMN_TOL = 1e-5     # fp32 storage: noise columns sit near 1e-7 relative


@dataclass
class LowRankFactors:
    p: torch.Tensor   # m x r, orthonormal or zero columns
    q: torch.Tensor   # n x r
    layer_id: int = 0
    stage_id: int = 0
    iteration: int = 0

    @property
    def rank(self) -> int:
        return self.p.shape[1]

    @property
    def element_count(self) -> int:
        return self.p.numel() + self.q.numel()


def basis_columns(rng_seed: int, n: int, start: int, stop: int) -> np.ndarray:
    """Fresh warm-start columns j in [start, stop): rng(seed, TAG_BASIS, j).standard_normal(n) (compressor.py:63-66)."""
    cols = [rng(rng_seed, TAG_BASIS, j).standard_normal(n) for j in range(start, stop)]
    return np.stack(cols, axis=1).astype(np.float32) if cols else np.zeros((n, 0), np.float32)


def _check_rank(r: int, m: int, n: int) -> None:
    if not 1 <= r <= min(m, n):
        raise ValueError(f"rank {r} outside [1, {min(m, n)}] for shape {(m, n)}")


class CompressorState:
    """Error-feedback state plus warm-start basis for one (matrix, worker); single owner."""

    def __init__(self, m: int, n: int, rank: int, rng_seed: int = 0):
        if m < 1 or n < 1:
            raise ValueError(f"matrix dimensions must be positive, got {(m, n)}")
        _check_rank(rank, m, n)
        dev = torch.device("cuda", torch.cuda.current_device()) if _lib.lib() else None
        self.m, self.n, self.rank, self.rng_seed = m, n, rank, rng_seed
        self.device = dev
        self._w = torch.zeros((m, n), dtype=torch.float32, device=dev)
        self._cap = 0
        self._basis = torch.empty((n, 0), dtype=torch.float32, device=dev)
        self._q_warm = torch.empty((n, 0), dtype=torch.float32, device=dev)
        self._precond = torch.empty((0, 0), dtype=torch.float64, device=dev)
        self._grow(rank)
        self._q_warm[:, :rank].copy_(self._basis[:, :rank])
        # residual factor pair of the last compress (None: residual == w)
        self._p_res: torch.Tensor | None = None
        self._q_res: torch.Tensor | None = None

    def _grow(self, cap: int) -> None:
        if cap <= self._cap:
            return
        fresh = torch.from_numpy(basis_columns(self.rng_seed, self.n, self._cap, cap)).to(self.device)
        basis = torch.empty((self.n, cap), dtype=torch.float32, device=self.device)
        qw = torch.empty((self.n, cap), dtype=torch.float32, device=self.device)
        basis[:, :self._cap] = self._basis
        basis[:, self._cap:] = fresh
        qw[:, :self._cap] = self._q_warm
        qw[:, self._cap:] = fresh
        pre = torch.eye(cap, dtype=torch.float64, device=self.device)
        pre[:self._cap, :self._cap] = self._precond
        self._basis, self._q_warm, self._precond, self._cap = basis, qw, pre, cap

    @property
    def q_warm(self) -> torch.Tensor:
        return self._q_warm[:, :self.rank]

    @property
    def residual(self) -> torch.Tensor:
        """residual = work - p q^T of the last step (compressor.py:112), materialised on the device."""
        if self._p_res is None:
            return self._w.clone()
        out = torch.empty_like(self._w)
        L = _lib.lib()
        _lib.check(L.edgc_residual(_lib.ptr(self._w), _lib.ptr(self._p_res), _lib.ptr(self._q_res),
                                   self._p_res.shape[1], self.m, self.n, _lib.ptr(out), _lib.stream_ptr()),
                   "edgc_residual")
        return out

    def _residual_pair(self):
        if self._p_res is None:
            return None, None, 0
        return self._p_res, self._q_res, self._p_res.shape[1]


def compress(matrix, state: CompressorState) -> LowRankFactors:
    """One error-feedback power-iteration step (compressor.py:94-123)."""
    g = as_device_matrix(matrix)
    if tuple(g.shape) != (state.m, state.n):
        raise ValueError(f"state is bound to shape {(state.m, state.n)}, got {tuple(g.shape)}")
    L = _lib.lib()
    stream = _lib.stream_ptr()
    p_res, q_res, r_res = state._residual_pair()
    flag = torch.zeros(1, dtype=torch.int32, device=state.device)
    _lib.check(L.edgc_check_work_finite(_lib.ptr(g), g.stride(0), _lib.ptr(state._w), _lib.ptr(p_res),
                                        _lib.ptr(q_res), r_res, state.m, state.n, _lib.ptr(flag), stream),
               "edgc_check_work_finite")
    if flag.item():
        raise ValueError("non-finite entries in gradient or residual")
    r = state.rank
    p = torch.empty((state.m, r), dtype=torch.float32, device=state.device)
    q = torch.empty((state.n, r), dtype=torch.float32, device=state.device)
    desc = _lib.CompressDesc(_lib.ptr(g), _lib.ptr(state._w), _lib.ptr(p_res), _lib.ptr(q_res),
                             _lib.ptr(state._q_warm), _lib.ptr(state._basis), _lib.ptr(p), _lib.ptr(q),
                             _lib.ptr(state._precond), state.m, state.n, g.stride(0), r, r_res, state._cap,
                             state._cap)
    arr = (_lib.CompressDesc * 1)(desc)
    need = L.edgc_compress_workspace_bytes(arr, 1)
    if need < 0:
        _lib.check(_lib.EDGC_EINVAL, "edgc_compress layout")
    ws = _lib.WORKSPACE.get(need, state.device)
    status = torch.zeros(1, dtype=torch.int32, device=state.device)
    _lib.check(L.edgc_compress(arr, 1, DEVICE_COLUMN_TOL, _lib.ptr(status), _lib.ptr(ws), ws.numel(), stream),
               "edgc_compress")
    # the state keeps private copies of the pair: the reference's residual is an array of its own
    # (compressor.py:112), so in-place edits of the returned factors must not reach the next step
    state._p_res, state._q_res = p, q
    meta = matrix if isinstance(matrix, GradientMatrix) else None
    return LowRankFactors(p=p.clone(), q=q.clone(), layer_id=meta.layer_id if meta else 0,
                          stage_id=meta.stage_id if meta else 0, iteration=meta.iteration if meta else 0)


def reconstruct_into(out: torch.Tensor, p: torch.Tensor, q: torch.Tensor) -> torch.Tensor:
    """out <- p q^T through the device reconstruction kernel."""
    L = _lib.lib()
    m, r = p.shape
    n = q.shape[0]
    desc = _lib.ReconDesc(_lib.ptr(p), _lib.ptr(q), _lib.ptr(out), m, n, out.stride(0), 0, 0, r, 1, 1.0, 0)
    arr = (_lib.ReconDesc * 1)(desc)
    ws = _lib.WORKSPACE.get(L.edgc_reconstruct_workspace_bytes(arr, 1), out.device)
    _lib.check(L.edgc_reconstruct(arr, 1, _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "edgc_reconstruct")
    return out


def decompress(factors: LowRankFactors) -> GradientMatrix:
    """P Q^T as a validated GradientMatrix (compressor.py:126-133)."""
    p = as_device_array(factors.p)
    q = as_device_array(factors.q)
    if p.dim() != 2 or q.dim() != 2 or p.shape[1] != q.shape[1]:
        raise ValueError(f"factor shapes {tuple(p.shape)} and {tuple(q.shape)} do not pair")
    out = torch.empty((p.shape[0], q.shape[0]), dtype=torch.float32, device=p.device)
    if p.shape[1] == 0:
        out.zero_()
    else:
        reconstruct_into(out, p, q)
    return GradientMatrix(out, layer_id=factors.layer_id, stage_id=factors.stage_id, iteration=factors.iteration)


def set_rank(state: CompressorState, r_new: int) -> None:
    """Shrink (keep leading columns) or grow (append fixed fresh columns); residual untouched (compressor.py:136-151)."""
    _check_rank(r_new, state.m, state.n)
    r_old = state.rank
    if r_new == r_old:
        return
    if r_new > r_old:
        state._grow(r_new)
        state._q_warm[:, r_old:r_new].copy_(state._basis[:, r_old:r_new])
        # fresh warm-start columns restart unpreconditioned
        state._precond[:, r_old:r_new] = 0.0
        state._precond[r_old:r_new, r_old:r_new] = torch.eye(r_new - r_old, dtype=torch.float64,
                                                             device=state.device)
    state.rank = r_new


def compressed_element_count(m: int, n: int, r: int) -> int:
    """Wire elements of one rank-r pair: r (m + n)."""
    if m < 1 or n < 1:
        raise ValueError(f"matrix dimensions must be positive, got {(m, n)}")
    if r < 0:
        raise ValueError(f"rank must be non-negative, got {r}")
    return r * (m + n)
