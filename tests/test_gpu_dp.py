"""GPU: EdgcDataParallel (train_toy's EDGC wiring, grad_source.py:311-479) at W = 1.

The rank history must equal the one the LIVE reference's tracker and controller
produce on the same inputs (tests/golden/dp.json, make_dp_golden.py), and the
averaged gradients must match the oracle's per-step DP average (uncompressed
during warm-up, compressed after).
"""

import numpy as np
import pytest
import torch

import oracle
from tests.golden.specs import DP_SCENARIO, dp_scenario_grads
from tests.helpers import load_json, rel_err

pytestmark = pytest.mark.gpu

SHAPES = [tuple(s) for s in DP_SCENARIO["shapes"]]


def grads_at(t):
    return dp_scenario_grads(t, 0)


def test_dp_driver_rank_history_and_averages():
    """Rank history identical to the reference control flow; averaged gradients equal to the
    oracle's per step: uncompressed during warm-up, and once compressing, one reference DP step
    from the device's own state (re-synced): at r ~ 0.8 min(m, n) the error-feedback iteration
    amplifies fp32 rounding ~1.5x per step even in the fp64 reference (tests/test_gpu_debug_rank.py),
    so chained trajectories are not a meaningful bar there."""
    from paper_2511_10333_b200.controller import PHASE_ACTIVE
    from paper_2511_10333_b200.dp import EdgcDataParallel
    from paper_2511_10333_b200.entropy import SamplerConfig
    from tests.test_gpu_debug_rank import resync
    sc = DP_SCENARIO
    iters, window, alpha, beta = sc["iters"], sc["window"], sc["alpha"], sc["beta"]
    ref_hist = load_json("dp.json")["driver"]["history"]
    dp = EdgcDataParallel(SHAPES, total_iterations=iters, seed=0, sampler=SamplerConfig(alpha, beta, 0),
                          window=window)
    seeds = oracle.state_seeds(0, 1, len(SHAPES))
    ost = None
    worst, where = 0.0, None
    for t in range(iters):
        gs = grads_at(t)
        active = dp.ctl.phase == PHASE_ACTIVE
        if active:
            if ost is None:
                r0 = dp.engine.ranks
                ost = [oracle.OracleState(m, n, r0[k], seeds[(0, k)]) for k, (m, n) in enumerate(SHAPES)]
            else:
                resync(dp.engine, ost)
            ref = oracle.dp_step([[g.astype(np.float64) for g in gs]], [ost])
        else:
            ref = [g.astype(np.float64) for g in gs]
        outs = dp.step(t, [torch.from_numpy(g).cuda() for g in gs])
        for k, (o, r) in enumerate(zip(outs, ref)):
            e = rel_err(o, r)
            if e > worst:
                worst, where = e, (t, k, active, list(dp.engine.ranks))
    dp.flush()
    dp.check_status()
    got = [None if d.ranks is None else d.ranks[0] for d in dp.rank_history]
    assert got == ref_hist
    assert any(r is not None for r in got), "controller never activated"
    assert worst <= 1e-4, (worst, where, got)
