"""GPU: the bucket engine (grouped compress + reconstruct) against the oracle's DP step.

W = 1 here (multi-rank exchange is covered by tests/test_dist.py on CPU/gloo
and by the multi-GPU bench).  Worker-w states are seeded as the reference
seeds them (grad_source.py:440-447), so a W-rank engine's rank-w factors are
the reference worker w's.
"""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
from tests.helpers import rel_err

pytestmark = pytest.mark.gpu


def _shapes():
    return [(256, 768), (256, 256), (256, 1024), (1024, 256), (48, 36), (7, 9)]


@pytest.mark.parametrize("rank", [1, 4, 5, 6, 8, 12, 16, 24, 32, 64, 128])
def test_engine_matches_oracle_dp_step_chained(rank):
    from paper_2511_10333_b200.engine import BucketEngine
    shapes = _shapes()
    eng = BucketEngine(shapes, rank=rank, seed=3)
    seeds = oracle.state_seeds(3, 1, len(shapes))
    ost = [[oracle.OracleState(m, n, min(rank, m, n), seeds[(0, k)]) for k, (m, n) in enumerate(shapes)]]
    worst = 0.0
    for t in range(6):
        gs = [oracle.synth_matrix(1, t, k, 0, m, n, 1e-2) for k, (m, n) in enumerate(shapes)]
        for dst, g in zip(eng.grads, gs):
            dst.copy_(torch.from_numpy(g))
        outs = eng.step(check=True)
        ref = oracle.dp_step([[g.astype(np.float64) for g in gs]], ost)
        for k, (o, r) in enumerate(zip(outs, ref)):
            worst = max(worst, rel_err(o, r))
            if t == 5:
                ref_res = ost[0][k].residual
                if np.linalg.norm(ref_res) > 1e-9 * np.linalg.norm(gs[k]):
                    worst = max(worst, rel_err(eng.residual(k), ref_res))
                else:  # full-rank compression: the reference residual is fp64 round-off
                    assert float(torch.linalg.norm(eng.residual(k))) <= 1e-5 * np.linalg.norm(gs[k])
    assert worst <= 5e-5, worst


@pytest.mark.parametrize("rank", [6, 8])
def test_engine_narrow_passes_match_oracle(rank):
    """Ranks 5..8 run the skinny GEMMs by default; EDGC_NARROW_MAX=8 pins them to the
    register-tiled narrow passes (k_pass1 / k_pass2 with 8 ranks per thread)."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, EDGC_NARROW_MAX="8")
    code = (f"import sys; sys.path.insert(0, {root!r}); "
            f"from tests.test_gpu_engine import test_engine_matches_oracle_dp_step_chained as t; t({rank})")
    res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]


@pytest.mark.parametrize("rank", [24, 32])
def test_engine_rank32_tensor_core_path_matches_oracle(rank):
    """16 < r <= 32 take the fused CUDA-core EF + P_raw pass (k_skinny_ef, 64 x 32 tiles) by
    default; EDGC_SKEF32=0 keeps them on the tcgen05 TcEF / TcPraw / TcQ kernels."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, EDGC_SKEF32="0")
    code = (f"import sys; sys.path.insert(0, {root!r}); "
            f"from tests.test_gpu_engine import test_engine_matches_oracle_dp_step_chained as t; t({rank})")
    res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]


@pytest.mark.parametrize("rank", [8, 16])
def test_engine_separate_ef_pass_matches_oracle(rank):
    """4 < r <= 16 fuse the EF update into the P_raw partials (k_skinny_ef) by default;
    EDGC_SKINNY_EF_OFF=1 keeps the separate EF pass (k_ef) that rank transitions still use."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, EDGC_SKINNY_EF_OFF="1")
    code = (f"import sys; sys.path.insert(0, {root!r}); "
            f"from tests.test_gpu_engine import test_engine_matches_oracle_dp_step_chained as t; t({rank})")
    res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]


@pytest.mark.parametrize("rank", [96, 256])
def test_engine_tensor_core_ranks_match_oracle(rank):
    """Wide ranks on the tcgen05 path (EF update, P_raw, Q, reconstruction: 3xTF32 with
    chunked accumulation) and the multi-CTA fp64 factorisation, r < min(m, n), with
    K = n, m long enough for several 128-K accumulation chunks and r = 256 split over two
    128-column tiles."""
    from paper_2511_10333_b200.engine import BucketEngine
    shapes = [(512, 1024), (1024, 512), (384, 640)]
    eng = BucketEngine(shapes, rank=rank, seed=5)
    seeds = oracle.state_seeds(5, 1, len(shapes))
    ost = [[oracle.OracleState(m, n, rank, seeds[(0, k)]) for k, (m, n) in enumerate(shapes)]]
    worst = 0.0
    for t in range(4):
        gs = [oracle.synth_matrix(6, t, k, 0, m, n, 1e-2) for k, (m, n) in enumerate(shapes)]
        for dst, g in zip(eng.grads, gs):
            dst.copy_(torch.from_numpy(g))
        outs = eng.step(check=True)
        ref = oracle.dp_step([[g.astype(np.float64) for g in gs]], ost)
        for k, (o, r) in enumerate(zip(outs, ref)):
            worst = max(worst, rel_err(o, r))
            if t == 3:
                worst = max(worst, rel_err(eng.residual(k), ost[0][k].residual))
    assert worst <= 5e-5, worst


def test_engine_set_rank_matches_oracle():
    from paper_2511_10333_b200.engine import BucketEngine
    shapes = [(128, 384), (384, 128)]
    eng = BucketEngine(shapes, rank=8, seed=0, rank_cap=8)
    seeds = oracle.state_seeds(0, 1, 2)
    ost = [[oracle.OracleState(m, n, 8, seeds[(0, k)]) for k, (m, n) in enumerate(shapes)]]
    schedule = {2: 4, 4: 12, 5: 6}
    for t in range(7):
        if t in schedule:
            eng.set_rank(schedule[t])
            for s in ost[0]:
                oracle.set_rank(s, schedule[t])
        gs = [oracle.synth_matrix(2, t, k, 0, m, n, 1e-2) for k, (m, n) in enumerate(shapes)]
        outs = eng.step([torch.from_numpy(g).cuda() for g in gs], check=True)
        ref = oracle.dp_step([[g.astype(np.float64) for g in gs]], ost)
        for o, r in zip(outs, ref):
            assert rel_err(o, r) <= 5e-5


def test_engine_nonfinite_raises_divergence():
    from paper_2511_10333_b200.engine import BucketEngine
    from paper_2511_10333_b200.errors import DivergenceError
    eng = BucketEngine([(64, 64)], rank=4)
    eng.grads[0].fill_(1.0)
    eng.grads[0][3, 3] = float("nan")
    with pytest.raises(DivergenceError):
        eng.step(check=True)


def test_engine_gpt2_layer_one_step():
    """One full GPT2-2.5B layer (4 matrices, 30.7M elements) against the oracle."""
    from paper_2511_10333_b200.engine import GPT2_2P5B_LAYER, BucketEngine
    eng = BucketEngine(list(GPT2_2P5B_LAYER), rank=4, seed=0)
    seeds = oracle.state_seeds(0, 1, 4)
    ost = [[oracle.OracleState(m, n, 4, seeds[(0, k)]) for k, (m, n) in enumerate(GPT2_2P5B_LAYER)]]
    for t in range(2):
        gs = [oracle.synth_matrix(0, t, k, 0, m, n, 1e-2) for k, (m, n) in enumerate(GPT2_2P5B_LAYER)]
        outs = eng.step([torch.from_numpy(g).cuda() for g in gs], check=True)
        ref = oracle.dp_step([[g.astype(np.float64) for g in gs]], ost)
        for o, r in zip(outs, ref):
            assert rel_err(o, r) <= 1e-4


def test_rank_changes_do_not_accumulate_plans():
    """Every controller decision used to leave its transition and steady-state plans (each with its
    own fp64 scratch) cached forever; now only the current ranks' plans survive, so HBM use is
    flat across many rank changes."""
    from paper_2511_10333_b200.engine import BucketEngine
    shapes = _shapes()
    eng = BucketEngine(shapes, rank=24, seed=3, rank_cap=48)
    gs = [torch.from_numpy(oracle.synth_matrix(1, 0, k, 0, m, n, 1e-2)).cuda() for k, (m, n) in enumerate(shapes)]
    mem = []
    for i, r in enumerate([24, 30, 17, 48, 9, 33, 24, 40, 12, 36, 20, 44, 28]):
        eng.set_rank(r)
        for _ in range(3):
            eng.step(gs)
        torch.cuda.synchronize()
        assert len(eng._plans) <= 4, sorted(k[:3] for k in eng._plans)
        mem.append(torch.cuda.memory_allocated())
    eng.check_status()
    # bounded by the largest configuration visited, not growing with the number of decisions
    assert mem[-1] <= max(mem[:4]) * 1.05, mem


def test_compress_factors_do_not_alias_the_residual():
    """Editing the returned factors in place (e.g. a caller scaling P) must not change the state's
    error-feedback residual (compressor.py:112 stores an array of its own)."""
    import paper_2511_10333_b200 as e
    m, n, r = 96, 160, 4
    g = oracle.synth_matrix(2, 0, 0, 0, m, n, 1e-2)
    st = e.CompressorState(m, n, r, rng_seed=5)
    f = e.compress(torch.from_numpy(g).cuda(), st)
    before = st.residual.clone()
    f.p.mul_(3.0)
    f.q.zero_()
    assert torch.equal(st.residual, before)
    ost = oracle.OracleState(m, n, r, 5)
    oracle.compress(g.astype(np.float64), ost)
    g2 = oracle.synth_matrix(2, 1, 0, 0, m, n, 1e-2)
    f2 = e.compress(torch.from_numpy(g2).cuda(), st)
    p2, q2, _ = oracle.compress(g2.astype(np.float64), ost)
    assert rel_err(f2.p @ f2.q.T, p2 @ q2.T) <= 2e-5


@pytest.mark.parametrize("rank", [4, 32])
def test_cuda_graph_step_equals_eager(rank):
    """The steady-state step recorded as CUDA graphs (one per factor-buffer parity) and replayed
    gives bit-identical averages and residuals to the eager step."""
    from paper_2511_10333_b200.engine import BucketEngine
    shapes = _shapes()
    eager = BucketEngine(shapes, rank=rank, seed=3)
    graph = BucketEngine(shapes, rank=rank, seed=3)
    for t in range(7):
        gs = [torch.from_numpy(oracle.synth_matrix(1, t, k, 0, m, n, 1e-2)).cuda() for k, (m, n) in enumerate(shapes)]
        for dst, g in zip(graph.grads, gs):
            dst.copy_(g)
        a = eager.step(gs)
        if t < 1:
            b = graph.step()
        else:
            if t == 1:
                graph.capture_graphs()
            b = graph.graph_step()
        torch.cuda.synchronize()
        for x, y in zip(a, b):
            assert torch.equal(x, y), t
    eager.check_status()
    graph.check_status()
    for k in range(len(shapes)):
        assert torch.equal(eager.residual(k), graph.residual(k))
