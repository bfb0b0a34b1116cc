"""GPU: Gaussian plug-in and FD-histogram entropy (entropy.py:82-107) vs the golden fixtures.

Histogram counts and edges: bit-exact.  Entropies: |dH| <= 1e-12 nats (fp64
reduction order is the only difference).
"""

import math

import numpy as np
import pytest
import torch

import oracle
from tests.golden.specs import HIST_SETS, hist_samples
from tests.helpers import load_json, load_npz, to_np

pytestmark = pytest.mark.gpu

HIST = load_json("hist.json")["sets"]
NPZ = load_npz("hist.npz")


@pytest.mark.parametrize("i", range(len(HIST_SETS)))
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_fd_histogram_bit_exact(i, dtype):
    from paper_2511_10333_b200.entropy import histogram_fd
    from paper_2511_10333_b200.errors import DegenerateInputError
    rec = HIST[i]
    x = hist_samples(HIST_SETS[i])
    dev = torch.from_numpy(x if dtype == "f64" else x.astype(np.float32)).cuda()
    if rec["h_hist"] is None:
        with pytest.raises(DegenerateInputError):
            histogram_fd(dev)
        return
    counts, edges, h = histogram_fd(dev)
    assert np.array_equal(to_np(counts), NPZ[f"counts_{i}"])
    assert np.array_equal(to_np(edges), NPZ[f"edges_{i}"])
    assert abs(h - rec["h_hist"]) <= 1e-12


@pytest.mark.parametrize("i", range(len(HIST_SETS)))
def test_gaussian_entropy_matches_reference(i):
    from paper_2511_10333_b200.entropy import entropy_gaussian_plugin
    from paper_2511_10333_b200.errors import DegenerateInputError
    rec = HIST[i]
    x = hist_samples(HIST_SETS[i])
    if rec["h_gauss"] is None:
        with pytest.raises(DegenerateInputError):
            entropy_gaussian_plugin(x)
        return
    assert abs(entropy_gaussian_plugin(x) - rec["h_gauss"]) <= 1e-12
    assert abs(entropy_gaussian_plugin(torch.from_numpy(x.astype(np.float32)).cuda()) - rec["h_gauss"]) <= 1e-12


def test_histogram_fixed_int_bins_matches_numpy():
    from paper_2511_10333_b200.entropy import histogram_fd
    x = np.random.default_rng(3).standard_normal(100_001).astype(np.float32).astype(np.float64)
    for bins in (1, 7, 64, 1000):
        c_ref, e_ref = np.histogram(x, bins=bins)
        c, e, _ = histogram_fd(x, bins=bins)
        assert np.array_equal(to_np(c), c_ref)
        assert np.array_equal(to_np(e), e_ref)


def test_gaussian_analytic_and_invariances():
    from paper_2511_10333_b200.entropy import GAUSSIAN_ENTROPY_CONST, entropy_gaussian_plugin
    x = np.random.default_rng(10).standard_normal(10**5)
    assert entropy_gaussian_plugin(x) == pytest.approx(GAUSSIAN_ENTROPY_CONST, abs=0.02)
    y = np.random.default_rng(12).standard_normal(4096)
    base = entropy_gaussian_plugin(y)
    for c in (0.5, 3.0, 10.0):
        assert entropy_gaussian_plugin(c * y) == pytest.approx(base + math.log(c), abs=1e-9)
    assert entropy_gaussian_plugin(y + 10.5) == pytest.approx(base, abs=1e-9)
    with pytest.raises(ValueError):
        entropy_gaussian_plugin(np.array([1.0]))


def test_histogram_analytic():
    from paper_2511_10333_b200.entropy import GAUSSIAN_ENTROPY_CONST, entropy_histogram
    x = np.random.default_rng(20).standard_normal(10**6)
    assert entropy_histogram(x) == pytest.approx(GAUSSIAN_ENTROPY_CONST, abs=0.05)
    u = np.random.default_rng(22).uniform(0.0, 2.0, 10**6)
    assert entropy_histogram(u) == pytest.approx(math.log(2.0), abs=0.05)
    assert entropy_histogram(u) == pytest.approx(oracle.histogram_entropy(u), abs=1e-12)


def test_layer_batch_gaussian_equals_oracle():
    """EntropyTracker's batched path: plan + fused gather + estimator over many layers at once."""
    from paper_2511_10333_b200.entropy import SamplerConfig, layer_entropies
    shapes = [(64, 96), (128, 128), (257, 33), (1024, 4096)]
    mats = [np.random.default_rng([4, k]).standard_normal(s, dtype=np.float32) * np.float32(1e-2)
            for k, s in enumerate(shapes)]
    cfg = SamplerConfig(alpha=1.0, beta=0.25, rng_seed=9)
    got = layer_entropies([torch.from_numpy(m).cuda() for m in mats], 30, cfg)
    for k, (m, h) in enumerate(zip(mats, got)):
        ref = oracle.gaussian_entropy(oracle.subsample(m, 0.25, oracle.subsample_seed(9, 30, k)))
        assert abs(h - ref) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("df,nbins", [(2.4, 16144), (2.2, 36578), (2.0, 123587), (1.5, 301971)])
def test_fd_histogram_many_bins_global_path(df, nbins):
    """Heavy tails: 16144 bins (just inside the 16K shared-memory bins), 36578
    (global-atomic counting), 123587 and 301971 (global path after the 64K-bin
    capacity retry)."""
    from paper_2511_10333_b200.entropy import histogram_fd
    import torch
    x = np.random.default_rng(5).standard_t(df, 1_000_000).astype(np.float32)
    c_ref, e_ref = np.histogram(x.astype(np.float64), bins="fd")
    assert c_ref.size == nbins
    c, e, _ = histogram_fd(torch.from_numpy(x).cuda())
    assert np.array_equal(c.cpu().numpy(), c_ref)
    assert np.array_equal(e.cpu().numpy(), e_ref)


@pytest.mark.parametrize("bad", [float("nan"), float("inf"), float("-inf")])
def test_histogram_rejects_non_finite_samples(bad):
    """np.histogram(bins='fd') raises ValueError when the autodetected range is not finite
    (numpy/lib/_histograms_impl.py:_get_outer_edges); the device histogram does too."""
    from paper_2511_10333_b200 import entropy as E
    x = torch.randn(100_003, device="cuda")
    x[12_345] = bad
    with pytest.raises(ValueError):
        E.histogram_fd(x)
    with pytest.raises(ValueError):
        E.histogram_fd(x, bins=64)
