"""GPU: wide-rank engine across rank shrinks (the DP driver's 109 -> 101 -> 93 schedule) vs the oracle."""

import numpy as np
import pytest
import torch

import oracle
from tests.helpers import rel_err

pytestmark = pytest.mark.gpu

SHAPES = [(128, 512), (512, 128), (256, 256)]


def test_engine_wide_rank_shrinks_match_oracle():
    from paper_2511_10333_b200.engine import BucketEngine
    eng = BucketEngine(SHAPES, rank=109, seed=0, rank_cap=109)
    seeds = oracle.state_seeds(0, 1, len(SHAPES))
    ost = [[oracle.OracleState(m, n, 109, seeds[(0, k)]) for k, (m, n) in enumerate(SHAPES)]]
    errs = []
    for t in range(30):
        if t in (10, 20):
            r = {10: 101, 20: 93}[t]
            eng.set_rank(r)
            for s in ost[0]:
                oracle.set_rank(s, r)
        gs = [oracle.synth_matrix(7, t, k, 0, m, n, 1e-2) for k, (m, n) in enumerate(SHAPES)]
        outs = eng.step([torch.from_numpy(g).cuda() for g in gs], check=True)
        ref = oracle.dp_step([[g.astype(np.float64) for g in gs]], ost)
        errs.append([rel_err(o, r_) for o, r_ in zip(outs, ref)])
    print("per-step errors:", [round(max(e), 7) for e in errs])
    assert max(max(e) for e in errs) <= 1e-4
