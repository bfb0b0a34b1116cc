"""CPU: host-side logic (rank model, controller, tracker windowing, seeds) and the C-ABI surface.

No device work here: the CUDA library is only loaded and its exported symbols
checked against include/edgc_b200.h.
"""

import ctypes
import math
import os
import re

import numpy as np
import pytest

from tests.golden.specs import RANK_CASES
from tests.helpers import load_json, sha

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    from paper_2511_10333_b200 import _build, _lib
    _build.build()
    lib = _lib.load_library()
    header = open(os.path.join(ROOT, "include", "edgc_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int64_t|int|void|const char \*)\s*(edgc_\w+)\s*\(", header, re.M))
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
    for name in declared:
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr)
    assert lib.edgc_abi_version() == 1


def test_workspace_queries_need_no_device():
    from paper_2511_10333_b200 import _lib
    lib = _lib.load_library()
    plans = (_lib.PlanDesc * 2)(_lib.PlanDesc(1, 2, 3, 5, 4_194_304, 1_048_576, None),
                                _lib.PlanDesc(1, 2, 3, 5, 11_059_200, 552_960, None))
    assert lib.edgc_sample_plan_workspace_bytes(plans, 2) > 4 * (1_048_576 + 552_960)
    bad = (_lib.PlanDesc * 1)(_lib.PlanDesc(1, 2, 3, 5, 10, 10, None))
    assert lib.edgc_sample_plan_workspace_bytes(bad, 1) == -1
    d = (_lib.CompressDesc * 1)(_lib.CompressDesc(1, 1, 0, 0, 1, 1, 1, 1, 0, 1920, 7680, 7680, 4, 0, 4, 4))
    assert lib.edgc_compress_workspace_bytes(d, 1) > 1920 * 4 * 8


def test_g_table_identical_to_reference():
    from paper_2511_10333_b200 import rank_model
    for rec in load_json("ranks.json")["cases"]:
        m, n = rec["shape"]
        tab = rank_model.build_g_table(min(m, n), max(m, n), rec["trials"], rec["table_seed"])
        assert sha(tab.g_values) == rec["g_sha256"]
        assert tab.g(rec["r_max"]) == rec["g_at_rmax"]


@pytest.mark.parametrize("ci", range(len(RANK_CASES)))
def test_controller_trace_from_golden_window_entropies(ci):
    """Feed the reference's window entropies to our controller: identical decisions."""
    import paper_2511_10333_b200 as e
    from paper_2511_10333_b200 import controller as C
    rec = load_json("ranks.json")["cases"][ci]
    m, n = rec["shape"]
    table = e.g_table(min(m, n), max(m, n), rec["trials"], rec["table_seed"])
    ctl = e.RankControllerState(bounds=e.RankBounds(rec["r_min"], rec["r_max"]), window=rec["window"],
                                step_limit=rec["step_limit"], warmup_floor=rec["warmup_floor"],
                                total_iterations=rec["iterations"])
    model = e.CommModel(eta=4.0 * (m + n) / 1e9, bandwidth=1e9)
    trace = []
    for w in rec["windows"]:
        if ctl.phase == C.PHASE_WARMUP:
            e.warmup_step(ctl, w["mean"], (w["index"] + 1) * ctl.window, table)
            trace.append(ctl.r_prev if ctl.phase == C.PHASE_ACTIVE else None)
        else:
            trace.append(e.adjust_rank_window(ctl, w["mean"], table, model)[0])
    assert trace == rec["trace"]


def test_rank_law_and_bounds():
    from paper_2511_10333_b200 import controller as C
    from paper_2511_10333_b200 import rank_model as R
    tab = R.g_table(64, 128, 16, 0)
    assert R.invert_g(0.0, tab) == 64
    assert R.invert_g(tab.g(0) * 2, tab) == 0
    for r0 in (5, 20, 40):
        assert R.rank_from_entropy(r0, 0.3, 0.3, tab) == R.invert_g(tab.g(r0), tab)
        assert R.rank_from_entropy(r0, 0.1, 0.3, tab) == R.rank_from_sigma(r0, math.exp(0.1), math.exp(0.3), tab)
    assert R.rank_from_entropy(10, 800.0, 0.0, tab) == 0
    b = C.RankBounds(4, 20)
    assert C.clamp_rank_step(40, 10, 8, b) == 18
    assert C.clamp_rank_step(1, 10, 8, b) == 4
    assert C.clamp_rank_step(12, 10, 8, b) == 12
    model = C.CommModel(eta=1e-3, bandwidth=1e9)
    bounds = C.compute_rank_bounds(model, 4 * 1024 * 4096, [(1024, 4096)])
    assert bounds.r_max == min(1024, int(4 * 1024 * 4096 / (4 * (1024 + 4096))))
    with pytest.raises(Exception):
        C.calibrate_comm_model([(1, 1.0)])
    fit = C.calibrate_comm_model([(1, 2.0), (2, 4.0), (4, 8.0)])
    assert fit.eta == pytest.approx(2.0) and fit.mape == pytest.approx(0.0)


def test_sampling_gate_and_windows():
    from paper_2511_10333_b200 import entropy as E
    assert [t for t in range(21) if E.should_sample_iteration(t, 0.1)] == [0, 10, 20]
    assert not E.should_sample_iteration(6, 0.25)
    with pytest.raises(ValueError):
        E.should_sample_iteration(0, 0.0)
    with pytest.raises(ValueError):
        E.SamplerConfig(alpha=0.1, beta=1.5)
    w = E.close_window([1.0, 3.0])
    assert w.mean_entropy == 2.0 and w.samples_used == 2
    with pytest.raises(E.DegenerateInputError):
        E.close_window([])
    with pytest.raises(ValueError):
        E.EntropyTracker(E.SamplerConfig(alpha=0.1, beta=1.0), window=5)
    s = np.array([1.0, 2.0, 4.0])
    assert np.allclose(E.relative_change_rate(1.05 * s, s), 0.05, atol=1e-12)


def test_tracker_windowing_without_sampling():
    """Iterations the gate skips never touch the device: window logic alone runs on CPU."""
    from paper_2511_10333_b200 import entropy as E
    tr = E.EntropyTracker(E.SamplerConfig(alpha=0.1, beta=0.25), window=10)
    tr._pending = [1.0]
    assert tr.observe(5, []) is None       # not a sampled iteration
    closed = tr.observe(11, [])             # window 0 closes, 11 is not sampled
    assert closed.window_index == 0 and closed.mean_entropy == 1.0
    with pytest.raises(ValueError):
        tr.observe(3, [])


def test_seeds_match_reference_golden():
    from paper_2511_10333_b200 import seeds
    gold = load_json("seeds.json")
    for rec in gold["subsample"]:
        assert seeds.subsample_seed(rec["seed"], rec["t"], rec["k"]) == rec["sub_seed"]
        assert seeds.subsample_seeds(rec["seed"], rec["t"], rec["k"] + 1)[rec["k"]] == rec["sub_seed"]
    got = {f"{w},{k}": v for (w, k), v in seeds.state_seeds(0, 8, 208).items()}
    assert got == gold["state_seeds_0_8_208"]


def test_batched_seed_derivation_matches_numpy():
    """pcg64_words_many / subsample_seeds (restated SeedSequence + PCG64 seeding) equal
    NumPy's default_rng word for word: single-word, multi-word (>= 2^32) and list entropy."""
    from paper_2511_10333_b200.seeds import pcg64_words, pcg64_words_many, subsample_seed, subsample_seeds
    r = np.random.default_rng(11)
    seeds = [0, 1, 2**31 - 1, 2**32 - 1, 2**32, 2**63 + 5, 2**64, 2**100 + 7] + [int(x) for x in r.integers(0, 2**31, 40)]
    lists = [[0, 2, 0, 0], [7, 2, 10, 207], [2**40, 2, 3, 1], [5], [1, 2, 3, 4, 5, 6, 7], []]
    assert pcg64_words_many(seeds) == [pcg64_words(s) for s in seeds]
    assert pcg64_words_many(lists) == [pcg64_words(l) for l in lists]
    for run_seed, it in [(0, 0), (0, 10), (12345, 3), (2**33 + 1, 7)]:
        assert subsample_seeds(run_seed, it, 30) == [subsample_seed(run_seed, it, k) for k in range(30)]


@pytest.mark.parametrize("name", ["gpt2_2p5b", "gpt2_12p1b", "gpt2_2p5b_layer", "dp_small", "dp_check"])
def test_dp_setup_bounds_match_reference_golden(name):
    """train_toy's EDGC setup (grad_source.py:311-327 -> controller.py:111-163) on the GPT-2 bucket
    sets: our edgc_setup gives the live reference's r_min / r_max (tests/golden/dp.json)."""
    from paper_2511_10333_b200.dp import edgc_setup
    from tests.golden.specs import DP_BOUND_SETS
    rec = load_json("dp.json")["bounds"][name]
    _, bounds, table = edgc_setup(DP_BOUND_SETS[name])
    assert (bounds.r_min, bounds.r_max, table.m) == (rec["r_min"], rec["r_max"], rec["table_m"])


def test_dp_driver_history_from_oracle_entropies():
    """The DP scenario's window entropies, computed by the oracle (NumPy choice + std), equal the
    reference's (dp.json), and our controller turns them into the reference's rank history."""
    import oracle
    from paper_2511_10333_b200 import controller as C
    from paper_2511_10333_b200.dp import edgc_setup
    from tests.golden.specs import DP_SCENARIO, dp_scenario_grads
    gold = load_json("dp.json")["driver"]
    sc = DP_SCENARIO
    model, bounds, table = edgc_setup([tuple(s) for s in sc["shapes"]])
    assert [bounds.r_min, bounds.r_max] == gold["bounds"]
    period = max(1, round(1 / sc["alpha"]))
    per_win = {}
    for t in range(0, sc["iters"], period):
        gs = dp_scenario_grads(t, 0)
        h = [oracle.gaussian_entropy(oracle.subsample(g.astype(np.float64), sc["beta"], oracle.subsample_seed(0, t, k)))
             for k, g in enumerate(gs)]
        per_win.setdefault(t // sc["window"], []).append(float(np.mean(h)))
    means = [float(np.mean(v)) for _, v in sorted(per_win.items())]
    assert np.allclose(means, gold["window_entropies"], rtol=0, atol=1e-12)
    ctl = C.RankControllerState(bounds=bounds, window=sc["window"], total_iterations=sc["iters"])
    hist = []
    for i, h in enumerate(gold["window_entropies"]):
        if ctl.phase == C.PHASE_WARMUP:
            C.warmup_step(ctl, h, (i + 1) * ctl.window, table)
            hist.append(ctl.r_prev if ctl.phase == C.PHASE_ACTIVE else None)
        else:
            hist.append(C.adjust_rank_window(ctl, h, table, model)[0])
    assert hist == gold["history"]
