"""GPU: config 3 — window rank schedule over 200 decaying-entropy iterations.

The device EntropyTracker (sampled indices + Gaussian plug-in on the GPU) feeds
the host controller; the rank trace must be IDENTICAL to the reference's
(golden ranks.json, made by the live reference on the same fp32 inputs) and
the window entropies within 1e-9 nats.
"""

import pytest
import torch

from tests.golden.specs import RANK_CASES, rank_case_matrix
from tests.helpers import load_json

pytestmark = pytest.mark.gpu

GOLD = load_json("ranks.json")["cases"]


def run_case(case):
    import paper_2511_10333_b200 as e
    from paper_2511_10333_b200 import controller as ctl_mod
    from paper_2511_10333_b200.entropy import sampling_period
    m, n = case["shape"]
    table = e.g_table(min(m, n), max(m, n), case["trials"], case["table_seed"])
    bounds = e.RankBounds(r_min=case["r_min"], r_max=case["r_max"])
    model = e.CommModel(eta=4.0 * (m + n) / 1e9, bandwidth=1e9, element_size=4)
    ctl = e.RankControllerState(bounds=bounds, window=case["window"], step_limit=case["step_limit"],
                                warmup_floor=case["warmup_floor"], total_iterations=case["iterations"])
    tracker = e.EntropyTracker(e.SamplerConfig(alpha=case["alpha"], beta=case["beta"],
                                               rng_seed=case["sampler_seed"]), case["window"])
    period = sampling_period(case["alpha"])
    trace, means = [], []

    def on_close(win):
        means.append(win.mean_entropy)
        if ctl.phase == ctl_mod.PHASE_WARMUP:
            e.warmup_step(ctl, win.mean_entropy, (win.window_index + 1) * ctl.window, table)
            trace.append(ctl.r_prev if ctl.phase == ctl_mod.PHASE_ACTIVE else None)
        else:
            trace.append(e.adjust_rank_window(ctl, win.mean_entropy, table, model)[0])

    for t in range(case["iterations"]):
        mats = [torch.from_numpy(rank_case_matrix(case, t)).cuda()] if t % period == 0 else []
        w = tracker.observe(t, mats)
        if w is not None:
            on_close(w)
    w = tracker.flush()
    if w is not None:
        on_close(w)
    return trace, means


@pytest.mark.parametrize("ci", range(len(RANK_CASES)), ids=lambda i: f"tau{RANK_CASES[i]['tau']:g}")
def test_rank_trace_identical_to_reference(ci):
    trace, means = run_case(RANK_CASES[ci])
    gold = GOLD[ci]
    assert trace == gold["trace"]
    for a, b in zip(means, [w["mean"] for w in gold["windows"]]):
        assert abs(a - b) <= 1e-9
