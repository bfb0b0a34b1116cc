"""``edgc`` import alias over paper_2511_10333_b200, for running the reference's own unit tests
(/root/reference/pkg/tests: test_compressor, test_entropy, test_rank_model, test_controller)
against this package unchanged -- the drop-in check.

Every public name is this package's (the device path; nothing here computes).  The one
adaptation is the array type at the boundary: the reference hands back NumPy float64 arrays,
the device package fp32 CUDA tensors, and the reference's tests do NumPy arithmetic on the
results.  So results are copied back to float64 NumPy where a test reads them:
``compress`` -> LowRankFactors of NumPy arrays, ``decompress`` / ``GradientMatrix`` -> ``.data``
as NumPy, ``CompressorState.residual`` / ``.q_warm`` -> NumPy, ``subsample_entries`` -> NumPy.
Inputs of any kind go straight to the device API (rounded to fp32 there, as documented).
"""

from __future__ import annotations

import sys
from dataclasses import dataclass

import numpy as np
import torch

import paper_2511_10333_b200 as _impl
from paper_2511_10333_b200 import *  # noqa: F401,F403
from paper_2511_10333_b200 import compressor as _compressor
from paper_2511_10333_b200 import controller, entropy, errors, matrix_core, rank_model, seeds  # noqa: F401

for _name in ("entropy", "controller", "rank_model", "matrix_core", "errors", "seeds", "compressor"):
    sys.modules[f"edgc.{_name}"] = getattr(_impl, _name)

__version__ = getattr(_impl, "__version__", "b200")


def _np(x):
    if isinstance(x, torch.Tensor):
        return x.detach().to(torch.float64).cpu().numpy()
    return np.asarray(x)


class GradientMatrix(_impl.GradientMatrix):
    """The device GradientMatrix (validation on the device), with ``.data`` read back as NumPy."""

    def __post_init__(self) -> None:
        super().__post_init__()
        self._dev = self.data
        self.data = _np(self._dev)


@dataclass
class LowRankFactors:
    p: np.ndarray
    q: np.ndarray
    layer_id: int = 0
    stage_id: int = 0
    iteration: int = 0

    @property
    def rank(self) -> int:
        return self.p.shape[1]

    @property
    def element_count(self) -> int:
        return self.p.size + self.q.size


class CompressorState(_impl.CompressorState):
    @property
    def residual(self):
        return _np(_impl.CompressorState.residual.fget(self))

    @property
    def q_warm(self):
        return _np(_impl.CompressorState.q_warm.fget(self))


def compress(matrix, state):
    if isinstance(matrix, GradientMatrix):
        matrix = _impl.GradientMatrix.trusted(matrix._dev, matrix.layer_id, matrix.stage_id, matrix.iteration)
    f = _impl.compress(matrix, state)
    return LowRankFactors(_np(f.p), _np(f.q), f.layer_id, f.stage_id, f.iteration)


def decompress(factors):
    g = _impl.decompress(_compressor.LowRankFactors(p=_impl.matrix_core.as_device_array(factors.p),
                                                    q=_impl.matrix_core.as_device_array(factors.q),
                                                    layer_id=factors.layer_id, stage_id=factors.stage_id,
                                                    iteration=factors.iteration))
    return GradientMatrix(g.data, layer_id=g.layer_id, stage_id=g.stage_id, iteration=g.iteration)


def subsample_entries(matrix, beta, seed):
    return _np(_impl.subsample_entries(matrix, beta, seed))
