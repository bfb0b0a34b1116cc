"""GPU: NumPy-exact sampled indices (entropy.py:67-79) through the CUDA C-ABI.

Bit-exact against the golden checksums made by NumPy 2.3.5 itself and against
the C restatement (oracle/npchoice.c) on extra seeds.
"""

import math

import numpy as np
import pytest
import torch

import oracle
from tests.helpers import load_json, sha, to_np

pytestmark = pytest.mark.gpu

CASES = load_json("choice.json")["cases"]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"N{c['N']}-b{c['beta']}-s{c['seed']}-{c['branch']}")
def test_sample_indices_bit_exact_vs_numpy_golden(case):
    from paper_2511_10333_b200.entropy import sample_indices
    idx = to_np(sample_indices(case["N"], case["beta"], case["seed"])).astype(np.int64)
    assert idx.size == case["count"]
    assert idx[:16].tolist() == case["head"]
    assert idx[-16:].tolist() == case["tail"]
    assert sha(idx) == case["sha256"]


def test_batched_plans_match_oracle_on_many_seeds():
    """Both branches, several seeds per shape, all planned in ONE batched device call."""
    from paper_2511_10333_b200.entropy import sample_count, sample_plans
    specs = []
    for n_elems in (12_345, 65_536, 1_000_000, 3_686_400):
        for beta in (0.05, 0.051, 0.25, 0.5, 0.9):
            for seed in (0, 7, 2**31 - 1):
                specs.append((n_elems, sample_count(n_elems, beta), seed))
    plans = sample_plans(specs)
    for (n_elems, count, seed), p in zip(specs, plans):
        ref = oracle.choice_indices(seed, n_elems, count)
        assert np.array_equal(to_np(p).astype(np.int64), ref), (n_elems, count, seed)


def test_subsample_entries_values_and_order():
    from paper_2511_10333_b200.entropy import subsample_entries
    rng = np.random.default_rng(5)
    m = rng.standard_normal((300, 200)).astype(np.float32)
    got = to_np(subsample_entries(m, 0.25, seed=77))
    ref = oracle.subsample(m.astype(np.float64), 0.25, 77)
    assert got.dtype == np.float64
    assert np.array_equal(got, ref)
    full = to_np(subsample_entries(m, 1.0, seed=0))
    assert np.array_equal(full, m.astype(np.float64).ravel())


def test_subsample_count_and_without_replacement():
    from paper_2511_10333_b200.entropy import subsample_entries
    m = np.arange(100.0, dtype=np.float32).reshape(10, 10)
    out = to_np(subsample_entries(m, 0.5, seed=3))
    assert out.size == 50 and len(set(out.tolist())) == 50
    m = np.random.default_rng(0).standard_normal((64, 64)).astype(np.float32)
    for beta in (0.1, 0.25, 0.333, 0.5, 0.999):
        assert subsample_entries(m, beta, seed=1).numel() == math.ceil(beta * 4096)


def test_bad_beta_raises():
    from paper_2511_10333_b200.entropy import subsample_entries
    with pytest.raises(ValueError):
        subsample_entries(np.zeros((4, 4), np.float32), 0.0, 1)
    with pytest.raises(ValueError):
        subsample_entries(np.zeros((4, 4), np.float32), 1.5, 1)


def test_native_library_is_loaded():
    import paper_2511_10333_b200._lib as L
    L.lib()
    assert L._lib is not None and torch.cuda.is_available()


@pytest.mark.parametrize("indices", [True, False])
def test_membership_bitmaps_match_oracle_sets(indices):
    """Membership bitmaps (full plans and EDGC_PLAN_BITMAP_ONLY plans) equal the oracle's
    sampled sets; bitmap-only plans still return one sampled element (the Gaussian shift).
    Includes a matrix spanning many 16K-position buckets and Floyd / tail branches."""
    from paper_2511_10333_b200.entropy import sample_count, sample_plans
    specs = [(n, sample_count(n, b), s) for n, b, s in [
        (14_745_600, 0.25, 3), (3_686_400, 0.25, 11), (1_000_000, 0.05, 2), (20_000, 0.999, 5),
        (9_999, 0.5, 1), (65_537, 0.051, 4), (100, 0.3, 9)]]
    plans, bms, status = sample_plans(specs, bitmaps=True, indices=indices)
    assert int(status.max()) == 0
    for (n, c, seed), p, bm in zip(specs, plans, bms):
        ref = oracle.choice_indices(seed, n, c)
        words = to_np(bm).astype(np.uint32)
        bits = np.unpackbits(words.view(np.uint8), bitorder="little")[:n]
        want = np.zeros(n, dtype=np.uint8)
        want[ref] = 1
        assert np.array_equal(bits, want), (n, c, seed)
        got = to_np(p).astype(np.int64)
        if indices:
            assert np.array_equal(got, ref)
        else:
            # bitmap-only: one sampled element (the Gaussian shift) -- Floyd plans give NumPy's first
            # sample, tail-shuffle plans (set-mode resolve) step 0's output, NumPy's last sample
            tail = n > 10000 and c > n // 20
            assert got.size == 1 and got[0] == (ref[-1] if tail else ref[0])


def test_set_resolve_beyond_2p25_positions():
    """GPT2-12.1B's largest matrices (3584 x 14336 = 51.4M elements > 2^25) take the order-free set
    resolve when the plans are bitmap-only: the bitmap equals NumPy's sampled set."""
    from paper_2511_10333_b200.entropy import sample_count, sample_plans
    n = 3584 * 14336
    c = sample_count(n, 0.25)
    plans, bms, status = sample_plans([(n, c, 41)], bitmaps=True, indices=False, ahead=True)
    assert int(status.max()) == 0
    ref = np.random.default_rng(41).choice(n, size=c, replace=False, shuffle=False)
    words = to_np(bms[0]).astype(np.uint32)
    bits = np.unpackbits(words.view(np.uint8), bitorder="little")[:n]
    want = np.zeros(n, dtype=np.uint8)
    want[ref] = 1
    assert np.array_equal(bits, want)
    assert int(to_np(plans[0])[0]) == int(ref[-1])
