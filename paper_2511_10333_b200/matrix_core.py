"""Device gradient matrices.

``GradientMatrix`` keeps the reference's identity fields and construction-time
invariants (2-D, positive dims, all finite; pkg/src/edgc/matrix_core.py:17-46)
but holds a CUDA fp32 tensor: the reference's float64 arrays are rounded to
fp32 on upload (the device path's storage precision).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import DegenerateInputError

__all__ = ["GradientMatrix", "as_device_matrix", "as_device_array", "frobenius_norm", "singular_values",
           "optimal_rank_r_error", "pearson_correlation"]


def _device() -> torch.device:
    _lib.lib()  # raises without a CUDA device / library
    return torch.device("cuda", torch.cuda.current_device())


def as_device_array(x, dtype=torch.float32) -> torch.Tensor:
    """Any array-like -> contiguous CUDA tensor of `dtype` (no copy if already so)."""
    dev = _device()
    if isinstance(x, GradientMatrix):
        x = x.data
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x)))
    if t.device != dev or t.dtype != dtype:
        t = t.to(device=dev, dtype=dtype, non_blocking=False)
    return t.contiguous()


def as_device_matrix(matrix) -> torch.Tensor:
    """The reference's ``_entries`` (matrix_core.py:49-56) on the device: 2-D fp32 CUDA tensor."""
    t = as_device_array(matrix)
    if t.dim() != 2:
        raise ValueError(f"expected a 2-D matrix, got shape {tuple(t.shape)}")
    return t


def any_nonfinite(t: torch.Tensor) -> bool:
    """Device finiteness check through the CUDA library (synchronises)."""
    L = _lib.lib()
    flag = torch.zeros(1, dtype=torch.int32, device=t.device)
    dtype = 0 if t.dtype == torch.float32 else 1
    src = t if t.dtype in (torch.float32, torch.float64) else t.to(torch.float64)
    _lib.check(L.edgc_check_finite(dtype, _lib.ptr(src), src.numel(), _lib.ptr(flag), _lib.stream_ptr()),
               "check_finite")
    return bool(flag.item())


@dataclass
class GradientMatrix:
    data: torch.Tensor
    layer_id: int = 0
    stage_id: int = 0
    iteration: int = 0

    def __post_init__(self) -> None:
        t = as_device_array(self.data)
        if t.dim() != 2:
            raise ValueError(f"gradient matrix must be 2-D, got shape {tuple(t.shape)}")
        if t.shape[0] < 1 or t.shape[1] < 1:
            raise ValueError(f"matrix dimensions must be positive, got {tuple(t.shape)}")
        if any_nonfinite(t):
            raise ValueError("gradient matrix contains non-finite entries")
        self.data = t

    @classmethod
    def trusted(cls, data: torch.Tensor, layer_id: int = 0, stage_id: int = 0, iteration: int = 0):
        """Wrap a 2-D fp32 CUDA tensor whose finiteness the caller already checked (no sync)."""
        obj = cls.__new__(cls)
        obj.data, obj.layer_id, obj.stage_id, obj.iteration = data, layer_id, stage_id, iteration
        return obj

    @property
    def m(self) -> int:
        return self.data.shape[0]

    @property
    def n(self) -> int:
        return self.data.shape[1]


# ---- spectral helpers (analysis / test oracles in the reference; not on the hot path)

def frobenius_norm(matrix) -> float:
    return float(torch.linalg.matrix_norm(as_device_matrix(matrix).double(), "fro"))


def singular_values(matrix) -> torch.Tensor:
    return torch.linalg.svdvals(as_device_matrix(matrix).double())


def optimal_rank_r_error(matrix, r: int) -> float:
    """sqrt(sum of squared singular values past index r): the Eckart–Young floor."""
    a = as_device_matrix(matrix)
    k = min(a.shape)
    if not 0 <= r <= k:
        raise ValueError(f"rank {r} outside [0, {k}] for shape {tuple(a.shape)}")
    s = singular_values(a)
    return float(torch.sqrt(torch.sum(s[r:] ** 2)))


def pearson_correlation(matrix_a, matrix_b) -> float:
    x = as_device_matrix(matrix_a).double().ravel()
    y = as_device_matrix(matrix_b).double().ravel()
    if x.numel() != y.numel():
        raise ValueError(f"element counts differ: {x.numel()} vs {y.numel()}")
    sx, sy = float(x.std(unbiased=False)), float(y.std(unbiased=False))
    if sx == 0.0 or sy == 0.0:
        raise DegenerateInputError("zero-variance input to correlation")
    rho = float(torch.dot(x - x.mean(), y - y.mean())) / (x.numel() * sx * sy)
    return min(1.0, max(-1.0, rho))
