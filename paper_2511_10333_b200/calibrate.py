"""Compressor-cost calibration from GPU timings.

The reference measures its CPU compressor with ``time.perf_counter`` around
``compress`` / ``decompress`` at a sweep of ranks (cli.py:164-184,
``_measure_compressor``) and fits affine costs that feed the Eq. 2 rank bounds
(cli.py:187-225 ``cmd_calibrate`` -> ``comm_model.json``; controller.py:111-163).
With the B200 kernels those costs change by orders of magnitude, so r_max
changes materially; this module produces the same ``CommModel`` from CUDA-event
timings of the device compressor.

* ``measure_compressor_gpu(m, n, ranks, repeats, seed)`` -> ``[(r, t_compress_s,
  t_decompress_s)]`` medians, the reference's sweep format (same input: the
  seeded TAG_NOISE standard-normal matrix, in fp32).
* ``fit_comm_model(sweep, m, n, bandwidth, element_size)`` -> ``CommModel``: the
  reference's ``measure`` branch (degree-1 polyfit of both costs, MAPE of the
  compress fit, eta = element_size (m + n) / bandwidth).
* ``model_to_dict`` -> the ``comm_model.json`` layout (cli.py:228-236).
"""

from __future__ import annotations

import json

import numpy as np

from .controller import CommModel
from .errors import CalibrationError

__all__ = ["measure_compressor_gpu", "fit_comm_model", "calibrate_gpu", "model_to_dict", "write_comm_model"]


def measure_compressor_gpu(m: int, n: int, ranks, repeats: int = 50, seed: int = 0, device=None):
    """Median device seconds of one compress and one decompress of an m x n matrix per rank."""
    import torch

    from . import seeds
    from .engine import BucketEngine
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    matrix = seeds.rng(seed, seeds.TAG_NOISE, 0).standard_normal((m, n)).astype(np.float32)
    g = torch.from_numpy(matrix).to(dev)
    sweep = []
    for r in ranks:
        r = int(r)
        if not 1 <= r <= min(m, n):
            raise CalibrationError(f"rank {r} outside [1, {min(m, n)}]")
        eng = BucketEngine([(m, n)], rank=r, seed=seed, device=dev)
        eng.grads[0].copy_(g)
        eng.step()                                  # warm the state before timing (cli.py:176)
        stream = torch.cuda.current_stream(dev)
        t_c, t_d = [], []
        for _ in range(int(repeats)):
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
            eng.compress()
            e1.record(stream)
            eng.reconstruct()
            e2.record(stream)
            eng.advance()
            e2.synchronize()
            t_c.append(e0.elapsed_time(e1) / 1e3)
            t_d.append(e1.elapsed_time(e2) / 1e3)
        eng.check_status()
        sweep.append((r, float(np.median(t_c)), float(np.median(t_d))))
        del eng
    return sweep


def fit_comm_model(sweep, m: int, n: int, bandwidth: float, element_size: int = 4) -> CommModel:
    """The reference's ``calibrate`` fit of a measured sweep (cli.py:206-223)."""
    if len(sweep) < 2 or len({int(s[0]) for s in sweep}) < 2:
        raise CalibrationError("need measurements at two distinct ranks")
    ranks = np.array([s[0] for s in sweep], dtype=float)
    fit_c = np.polyfit(ranks, [s[1] for s in sweep], 1)
    fit_d = np.polyfit(ranks, [s[2] for s in sweep], 1)
    pred = np.polyval(fit_c, ranks)
    meas = np.array([s[1] for s in sweep])
    mape = float(np.mean(np.abs(pred - meas) / meas))
    eta = int(element_size) * (int(m) + int(n)) / float(bandwidth)
    return CommModel(eta=eta, bandwidth=float(bandwidth), element_size=int(element_size),
                     compress_cost=(max(0.0, float(fit_c[1])), max(0.0, float(fit_c[0]))),
                     decompress_cost=(max(0.0, float(fit_d[1])), max(0.0, float(fit_d[0]))), mape=mape)


def calibrate_gpu(m: int, n: int, ranks, *, bandwidth: float, element_size: int = 4, repeats: int = 50,
                  seed: int = 0, device=None):
    """Measure on the device and fit: (CommModel, sweep)."""
    sweep = measure_compressor_gpu(m, n, ranks, repeats=repeats, seed=seed, device=device)
    return fit_comm_model(sweep, m, n, bandwidth, element_size), sweep


def model_to_dict(model: CommModel) -> dict:
    return {"eta": model.eta, "bandwidth": model.bandwidth, "element_size": model.element_size,
            "compress_cost": list(model.compress_cost), "decompress_cost": list(model.decompress_cost),
            "mape": model.mape}


def write_comm_model(path: str, model: CommModel) -> None:
    with open(path, "w") as fh:
        json.dump(model_to_dict(model), fh, indent=2, sort_keys=True)
        fh.write("\n")
