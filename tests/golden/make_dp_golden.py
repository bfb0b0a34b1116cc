"""Generate tests/golden/dp.json from the LIVE reference (build container only).

    python tests/golden/make_dp_golden.py

Pins the DP driver's control plane to the reference's own code:

* ``bounds``: train_toy's EDGC setup (grad_source.py:311-327) — Eq. 2 rank
  bounds from the cost-free byte model (controller.py:111-163), the g-table of
  the largest matrix and the r_max clamp below table.m — for the GPT2-2.5B and
  GPT2-12.1B bucket sets and the small test sets;
* ``history``: the window-rank decisions the reference's EntropyTracker
  (entropy.py:135-192, Gaussian plug-in on worker-0 raw gradients) and
  controller (controller.py:205-262) make on DP_SCENARIO's decaying-entropy
  gradients.  The decisions depend only on worker 0's gradients, so the same
  history holds at every world size.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from edgc import controller as rctl  # noqa: E402  (the reference)
from edgc import entropy as rent  # noqa: E402
from edgc import rank_model as rrm  # noqa: E402

from tests.golden.specs import DP_BOUND_SETS, DP_SCENARIO, dp_scenario_grads  # noqa: E402


def train_toy_setup(shapes, trials=64, seed=0):
    """grad_source.py:311-327, verbatim arithmetic through the reference's functions."""
    element_size, bandwidth = 4, 1e9
    raw = sum(m * n for m, n in shapes)
    per_rank = sum(m + n for m, n in shapes)
    model = rctl.CommModel(eta=element_size * per_rank / bandwidth, bandwidth=bandwidth, element_size=element_size)
    bounds = rctl.compute_rank_bounds(model, element_size * raw, shapes)
    big = max(shapes, key=lambda s: s[0] * s[1])
    table = rrm.g_table(min(big), max(big), trials, seed)
    unclamped = (bounds.r_min, bounds.r_max)
    if bounds.r_max >= table.m:
        r_max = table.m - 1
        bounds = rctl.RankBounds(r_min=min(bounds.r_min, r_max), r_max=r_max)
    return model, bounds, table, unclamped


def make_bounds():
    out = {}
    for name, shapes in DP_BOUND_SETS.items():
        _, b, table, raw = train_toy_setup(shapes)
        out[name] = {"r_min": b.r_min, "r_max": b.r_max, "unclamped": list(raw), "table_m": table.m}
    return out


def make_history():
    sc = DP_SCENARIO
    shapes = [tuple(s) for s in sc["shapes"]]
    model, bounds, table, _ = train_toy_setup(shapes)
    ctl = rctl.RankControllerState(bounds=bounds, window=sc["window"], total_iterations=sc["iters"])
    cfg = rent.SamplerConfig(alpha=sc["alpha"], beta=sc["beta"], rng_seed=0)
    tracker = rent.EntropyTracker(cfg, sc["window"])
    hist, entropies = [], []

    def update(win):
        # grad_source.py:450-479 without the write-only warm-up SVD probe (controller.py:231)
        entropies.append(win.mean_entropy)
        if ctl.phase == rctl.PHASE_WARMUP:
            rctl.warmup_step(ctl, win.mean_entropy, (win.window_index + 1) * ctl.window, table)
            hist.append(ctl.r_prev if ctl.phase == rctl.PHASE_ACTIVE else None)
        else:
            r, _ = rctl.adjust_rank_window(ctl, win.mean_entropy, table, model)
            hist.append(int(r))

    for t in range(sc["iters"]):
        gs = [g.astype(np.float64) for g in dp_scenario_grads(t, 0)]
        win = tracker.observe(t, gs)
        if win is not None:
            update(win)
    win = tracker.flush()
    if win is not None:
        update(win)
    return {"scenario": sc, "bounds": [bounds.r_min, bounds.r_max], "history": hist,
            "window_entropies": entropies}


def main():
    out = {"numpy": np.__version__, "bounds": make_bounds(), "driver": make_history()}
    with open(os.path.join(HERE, "dp.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps({"bounds": out["bounds"], "history": out["driver"]["history"]}))


if __name__ == "__main__":
    _ = math
    main()
