"""Compressor-cost calibration (cli.py:164-225): the fit on the host (CPU) and the
GPU measurement sweep (gpu)."""

import numpy as np
import pytest

from paper_2511_10333_b200.calibrate import fit_comm_model, model_to_dict
from paper_2511_10333_b200.controller import compute_rank_bounds
from paper_2511_10333_b200.errors import CalibrationError


def test_fit_matches_reference_formula():
    sweep = [(4, 1.1e-4, 3.0e-5), (8, 1.3e-4, 3.9e-5), (16, 1.8e-4, 6.1e-5), (32, 2.9e-4, 1.05e-4)]
    m, n, bw = 1024, 4096, 2.5e10
    model = fit_comm_model(sweep, m, n, bw, 4)
    ranks = np.array([s[0] for s in sweep], dtype=float)
    fc = np.polyfit(ranks, [s[1] for s in sweep], 1)
    fd = np.polyfit(ranks, [s[2] for s in sweep], 1)
    assert model.eta == 4 * (m + n) / bw
    assert model.compress_cost == (max(0.0, fc[1]), max(0.0, fc[0]))
    assert model.decompress_cost == (max(0.0, fd[1]), max(0.0, fd[0]))
    pred = np.polyval(fc, ranks)
    meas = np.array([s[1] for s in sweep])
    assert model.mape == float(np.mean(np.abs(pred - meas) / meas))
    d = model_to_dict(model)
    assert set(d) == {"eta", "bandwidth", "element_size", "compress_cost", "decompress_cost", "mape"}


def test_fit_needs_two_ranks():
    with pytest.raises(CalibrationError):
        fit_comm_model([(4, 1e-4, 1e-5), (4, 1.1e-4, 1e-5)], 64, 64, 1e9)


@pytest.mark.gpu
def test_gpu_sweep_feeds_rank_bounds():
    from paper_2511_10333_b200.calibrate import calibrate_gpu
    model, sweep = calibrate_gpu(512, 1536, [2, 4, 8, 16], bandwidth=1e9, repeats=5)
    assert [s[0] for s in sweep] == [2, 4, 8, 16]
    assert all(t_c > 0 and t_d > 0 for _, t_c, t_d in sweep)
    bounds = compute_rank_bounds(model, 4.0 * 512 * 1536, [(512, 1536)])
    assert 1 <= bounds.r_min <= bounds.r_max <= 512


@pytest.mark.gpu
def test_gpu_compression_not_worth_it_at_high_bandwidth():
    """At NVLink-class bandwidth a small matrix is cheaper to send raw: the reference's rule
    raises CompressionInfeasibleError from the calibrated costs (controller.py:111-163)."""
    from paper_2511_10333_b200.calibrate import calibrate_gpu
    from paper_2511_10333_b200.errors import CompressionInfeasibleError
    model, _ = calibrate_gpu(512, 1536, [2, 4, 8, 16], bandwidth=5e11, repeats=5)
    with pytest.raises(CompressionInfeasibleError):
        compute_rank_bounds(model, 4.0 * 512 * 1536, [(512, 1536)])
