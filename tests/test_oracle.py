"""CPU: the oracle restatement against the golden fixtures made from the live reference.

This pins the checker before any device result is compared with it.
"""

import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from tests.golden.specs import (
    COMPRESS_CASES, HIST_SETS, RANK_CASES, compress_inputs, hist_samples,
)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


CHOICE = _load("choice.json")["cases"]


@pytest.mark.parametrize("case", [c for c in CHOICE if c["N"] <= 4_194_304],
                         ids=lambda c: f"N{c['N']}-b{c['beta']}-s{c['seed']}")
def test_oracle_choice_matches_numpy_golden(case):
    if case["branch"] == "copy":
        idx = np.arange(case["N"], dtype=np.int64)
    else:
        assert oracle.choice_branch(case["N"], case["count"]) == case["branch"]
        idx = oracle.choice_indices(case["seed"], case["N"], case["count"])
    assert idx.size == case["count"]
    assert idx[:16].tolist() == case["head"]
    assert _sha(idx) == case["sha256"]


def test_oracle_choice_branches_covered():
    branches = {c["branch"] for c in CHOICE}
    assert branches == {"copy", "tail", "floyd"}
    # the count == N // 20 boundary goes to Floyd
    assert any(c["count"] == c["N"] // 20 and c["branch"] == "floyd" and c["N"] > 10000 for c in CHOICE)


HIST = _load("hist.json")["sets"]
HIST_NPZ = np.load(os.path.join(GOLD, "hist.npz"))


@pytest.mark.parametrize("i", range(len(HIST_SETS)))
def test_oracle_fd_histogram_bit_exact(i):
    rec = HIST[i]
    x = hist_samples(HIST_SETS[i])
    counts, edges = oracle.fd_histogram(x)
    assert np.array_equal(counts, HIST_NPZ[f"counts_{i}"])
    assert np.array_equal(edges, HIST_NPZ[f"edges_{i}"])
    if rec["h_hist"] is None:
        with pytest.raises(ValueError):
            oracle.histogram_entropy(x)
    else:
        assert oracle.histogram_entropy(x) == pytest.approx(rec["h_hist"], abs=1e-12)
    if rec["h_gauss"] is None:
        with pytest.raises(ValueError):
            oracle.gaussian_entropy(x)
    else:
        assert oracle.gaussian_entropy(x) == pytest.approx(rec["h_gauss"], abs=1e-12)


COMP = _load("compress.json")["cases"]
COMP_NPZ = np.load(os.path.join(GOLD, "compress.npz"))


@pytest.mark.parametrize("ci", range(len(COMPRESS_CASES)))
def test_oracle_compress_matches_reference(ci):
    case = COMPRESS_CASES[ci]
    st = oracle.OracleState(case["m"], case["n"], case["rank"], case["seed"])
    assert np.array_equal(st.q_warm, COMP_NPZ[f"c{ci}_q0"])
    for t in range(case["steps"]):
        if t in case.get("set_rank_at", {}):
            oracle.set_rank(st, case["set_rank_at"][t])
        p, q, _ = oracle.compress(compress_inputs(case, t), st)
        np.testing.assert_allclose(p, COMP_NPZ[f"c{ci}_t{t}_p"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(q, COMP_NPZ[f"c{ci}_t{t}_q"], rtol=0, atol=1e-12)
        if f"c{ci}_t{t}_res" in COMP_NPZ:
            np.testing.assert_allclose(st.residual, COMP_NPZ[f"c{ci}_t{t}_res"], rtol=0, atol=1e-12)
            np.testing.assert_allclose(oracle.decompress(p, q), COMP_NPZ[f"c{ci}_t{t}_out"], rtol=0, atol=1e-12)


def test_oracle_seeds_match_reference():
    gold = _load("seeds.json")
    for rec in gold["subsample"]:
        assert oracle.subsample_seed(rec["seed"], rec["t"], rec["k"]) == rec["sub_seed"]
    dp = oracle.state_seeds(0, 8, 208)
    assert {f"{w},{k}": v for (w, k), v in dp.items()} == gold["state_seeds_0_8_208"]


def test_oracle_dp_step_single_worker_equals_compress_decompress():
    rng = np.random.default_rng(0)
    g = rng.standard_normal((16, 24)).astype(np.float32).astype(np.float64)
    a = [[oracle.OracleState(16, 24, 4, 7)]]
    b = oracle.OracleState(16, 24, 4, 7)
    avg = oracle.dp_step([[g]], a)[0]
    p, q, _ = oracle.compress(g, b)
    assert np.array_equal(avg, oracle.decompress(p, q))


def test_rank_golden_shapes():
    ranks = _load("ranks.json")["cases"]
    assert [c["tau"] for c in ranks] == [c["tau"] for c in RANK_CASES]
    assert ranks[0]["trace"][0] is None and ranks[0]["trace"][1] == 128
