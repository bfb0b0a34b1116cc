"""GPU: low-rank compress / decompress / error feedback / set_rank (compressor.py:94-160).

Tolerances (fp32 storage, fp64 reductions):
  * P, Q, residual, reconstruction vs the reference on fp32-representable
    inputs: relative Frobenius error <= 2e-5 per step, chained through the
    golden error-feedback sequences;
  * config 1 (1024x4096, r=4) chained over 50 EF steps vs the oracle:
    <= 1e-4;
  * properties the reference tests pin: orthonormal P (<= 2e-6 off-diagonal),
    exact zero matrix, exact power-of-two scale equivariance, exact-rank
    round trips (<= 1e-6), dead columns zeroed and re-seeded.
"""

import numpy as np
import pytest
import torch

import oracle
from tests.golden.specs import COMPRESS_CASES, compress_inputs
from tests.helpers import load_npz, rel_err, to_np

pytestmark = pytest.mark.gpu

NPZ = load_npz("compress.npz")
TOL_STEP = 2e-5


def _api():
    import paper_2511_10333_b200 as e
    return e


@pytest.mark.parametrize("ci", range(len(COMPRESS_CASES)))
def test_compress_matches_reference_golden(ci):
    e = _api()
    case = COMPRESS_CASES[ci]
    st = e.CompressorState(case["m"], case["n"], case["rank"], rng_seed=case["seed"])
    np.testing.assert_array_equal(to_np(st.q_warm), NPZ[f"c{ci}_q0"].astype(np.float32))
    for t in range(case["steps"]):
        if t in case.get("set_rank_at", {}):
            e.set_rank(st, case["set_rank_at"][t])
        g = compress_inputs(case, t).astype(np.float32)
        f = e.compress(g, st)
        p_ref, q_ref = NPZ[f"c{ci}_t{t}_p"], NPZ[f"c{ci}_t{t}_q"]
        if case["kind"] == "zero":
            assert torch.count_nonzero(f.p @ f.q.T) == 0
            assert torch.count_nonzero(st.residual) == 0
            continue
        assert rel_err(f.p, p_ref) <= TOL_STEP, (t, rel_err(f.p, p_ref))
        assert rel_err(f.q, q_ref) <= TOL_STEP, (t, rel_err(f.q, q_ref))
        out = e.decompress(f).data
        if f"c{ci}_t{t}_out" in NPZ:
            assert rel_err(out, NPZ[f"c{ci}_t{t}_out"]) <= TOL_STEP
            res_ref = NPZ[f"c{ci}_t{t}_res"]
            if np.linalg.norm(res_ref) > 1e-9 * max(1.0, np.linalg.norm(g)):
                assert rel_err(st.residual, res_ref) <= 1e-4
            else:  # exact-rank input: the reference residual is fp64 round-off
                assert float(torch.linalg.norm(st.residual)) <= 1e-6 * np.linalg.norm(g)


def test_config1_chained_50_steps_vs_oracle():
    e = _api()
    m, n, r, seed = 1024, 4096, 4, 11
    st = e.CompressorState(m, n, r, rng_seed=seed)
    ost = oracle.OracleState(m, n, r, seed)
    worst = 0.0
    for t in range(50):
        g = oracle.synth_matrix(0, t, 0, 0, m, n, 1e-2)
        f = e.compress(g, st)
        p, q, _ = oracle.compress(g.astype(np.float64), ost)
        worst = max(worst, rel_err(f.p, p), rel_err(f.q, q), rel_err(e.decompress(f).data, p @ q.T))
        if t in (0, 9, 49):
            worst = max(worst, rel_err(st.residual, ost.residual))
    assert worst <= 1e-4, worst


def test_orthonormal_columns():
    e = _api()
    m = np.random.default_rng(7).standard_normal((32, 48)).astype(np.float32)
    p = e.compress(m, e.CompressorState(32, 48, 8, rng_seed=1)).p.double()
    gram = p.T @ p
    off = gram - torch.diag(torch.diag(gram))
    assert float(off.abs().max()) <= 2e-6
    assert float((torch.diag(gram) - 1).abs().max()) <= 2e-6


def test_power_of_two_scale_equivariance_exact():
    e = _api()
    m = np.random.default_rng(21).standard_normal((48, 32)).astype(np.float32)

    def err(x):
        st = e.CompressorState(48, 32, 8, rng_seed=9)
        f = e.compress(x, st)
        return torch.from_numpy(x).cuda() - f.p @ f.q.T, f

    base, fb = err(m)
    for c in (0.5, 2.0, 4.0):
        scaled, fs = err(np.float32(c) * m)
        assert torch.equal(fs.p, fb.p)
        assert torch.equal(fs.q, np.float32(c) * fb.q)


def test_exact_rank_one_roundtrip():
    e = _api()
    rng = np.random.default_rng(0)
    m = np.outer(rng.integers(-8, 9, 12), rng.integers(-8, 9, 9)).astype(np.float32)
    out = e.decompress(e.compress(m, e.CompressorState(12, 9, 1, rng_seed=3))).data
    assert rel_err(out, m) <= 1e-6


def test_rank_deficient_dead_columns_zeroed_and_reseeded():
    e = _api()
    rng = np.random.default_rng(3)
    m = (rng.integers(-3, 4, (64, 16)) @ rng.integers(-3, 4, (16, 256))).astype(np.float32)
    st = e.CompressorState(64, 256, 64, rng_seed=2)
    f = e.compress(m, st)
    assert rel_err(f.p @ f.q.T, m) <= 5e-6   # fp32 factors of an exact rank-16 integer matrix
    pn = torch.linalg.norm(f.p, dim=0)
    dead = (pn == 0).cpu().numpy()
    assert dead.sum() == 64 - 16
    basis = oracle.basis_column
    for j in np.flatnonzero(dead)[:4]:
        assert np.array_equal(to_np(f.q[:, j]), basis(2, int(j), 256).astype(np.float32))


def test_refactor_idempotent_on_exact_rank_input():
    e = _api()
    m = np.random.default_rng(11).standard_normal((20, 15)).astype(np.float32)
    first = e.compress(m, e.CompressorState(20, 15, 15, rng_seed=5))
    prod = (first.p @ first.q.T).cpu().numpy()
    second = e.compress(prod, e.CompressorState(20, 15, 15, rng_seed=5))
    assert rel_err(second.p @ second.q.T, prod) <= 1e-5


def test_error_feedback_accumulates():
    e = _api()
    m = np.random.default_rng(42).standard_normal((64, 64)).astype(np.float32)
    st = e.CompressorState(64, 64, 8, rng_seed=1)
    acc = torch.zeros(64, 64, dtype=torch.float64, device="cuda")
    mt = torch.from_numpy(m).cuda().double()
    rels = []
    for t in range(1, 101):
        f = e.compress(m, st)
        acc += (f.p @ f.q.T).double()
        rels.append(float(torch.linalg.norm(acc - t * mt) / (t * torch.linalg.norm(mt))))
    assert np.mean(rels[:25]) > np.mean(rels[25:50]) > np.mean(rels[50:])
    assert rels[99] <= 0.05


def test_nonfinite_raises_before_mutation():
    e = _api()
    st = e.CompressorState(8, 8, 2, rng_seed=0)
    e.compress(np.random.default_rng(0).standard_normal((8, 8)).astype(np.float32), st)
    res, qw = st.residual.clone(), st.q_warm.clone()
    bad = np.ones((8, 8), np.float32)
    bad[3, 4] = np.inf
    with pytest.raises(ValueError):
        e.compress(bad, st)
    assert torch.equal(st.residual, res) and torch.equal(st.q_warm, qw)


def test_shape_and_rank_errors():
    e = _api()
    with pytest.raises(ValueError):
        e.compress(np.zeros((4, 5), np.float32), e.CompressorState(4, 4, 2))
    with pytest.raises(ValueError):
        e.CompressorState(4, 8, 5)
    st = e.CompressorState(8, 8, 4)
    for bad in (0, 9):
        with pytest.raises(ValueError):
            e.set_rank(st, bad)


def test_set_rank_semantics():
    e = _api()
    st = e.CompressorState(64, 64, 64, rng_seed=1)
    e.compress(np.random.default_rng(0).standard_normal((64, 64)).astype(np.float32), st)
    before = st.q_warm.clone()
    e.set_rank(st, 32)
    assert st.rank == 32 and torch.equal(st.q_warm, before[:, :32])
    a = e.CompressorState(64, 64, 32, rng_seed=7)
    e.set_rank(a, 64)
    b = e.CompressorState(64, 64, 64, rng_seed=7)
    assert torch.equal(a.q_warm[:, 32:], b.q_warm[:, 32:])
    s = e.CompressorState(16, 24, 8, rng_seed=1)
    e.compress(np.random.default_rng(5).standard_normal((16, 24)).astype(np.float32), s)
    res = s.residual.clone()
    e.set_rank(s, 4)
    e.set_rank(s, 8)
    assert torch.equal(s.residual, res)


def test_decompress_unit_factors_and_metadata():
    e = _api()
    p = np.zeros((5, 1))
    q = np.zeros((7, 1))
    p[0, 0] = q[0, 0] = 1.0
    out = to_np(e.decompress(e.LowRankFactors(p=p, q=q)).data)
    exp = np.zeros((5, 7), np.float32)
    exp[0, 0] = 1.0
    assert np.array_equal(out, exp)
    g = e.GradientMatrix(np.ones((3, 4)), layer_id=2, stage_id=1, iteration=9)
    d = e.decompress(e.compress(g, e.CompressorState(3, 4, 1)))
    assert (d.layer_id, d.stage_id, d.iteration) == (2, 1, 9)


def test_error_sandwich():
    e = _api()
    m = np.random.default_rng(42).standard_normal((64, 64)).astype(np.float32)
    f = e.compress(m, e.CompressorState(64, 64, 16, rng_seed=1))
    err = float(torch.linalg.norm(torch.from_numpy(m).cuda() - f.p @ f.q.T))
    assert e.optimal_rank_r_error(m, 16) <= err <= e.frobenius_norm(m)


def _graded_matrix(m, n, sigmas, seed):
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((m, len(sigmas))))
    v, _ = np.linalg.qr(rng.standard_normal((n, len(sigmas))))
    a = (u * np.asarray(sigmas)) @ v.T + 1e-4 * rng.standard_normal((m, n))
    return a.astype(np.float32)


@pytest.mark.parametrize("sigmas,tol", [((1e3, 1e2, 10.0, 1.0, 0.5), 1e-3), ((1.0, 1.0, 1.0, 1.0), 1e-4),
                                        ((1e2, 30.0, 10.0, 3.0, 1.0), 1e-4)])
def test_graded_spectrum_chained_vs_oracle(sigmas, tol):
    """Ill-conditioned warm starts (the one-sweep path's kappa fallback) stay within tolerance.

    With sigma_1 / sigma_4 = 1e3 the fp32 representation of w alone perturbs the
    4th direction by ~1e-4 relative, hence the looser bound for that spectrum.
    Spectra whose trailing sigma falls under DEVICE_COLUMN_TOL * ||P|| are a
    documented semantic delta (dead column here, kept by the fp64 reference).
    """
    e = _api()
    m, n, r = 256, 512, 4
    st = e.CompressorState(m, n, r, rng_seed=4)
    ost = oracle.OracleState(m, n, r, 4)
    for t in range(4):
        g = _graded_matrix(m, n, sigmas, 100 + t)
        f = e.compress(g, st)
        p, q, _ = oracle.compress(g.astype(np.float64), ost)
        out = p @ q.T
        assert rel_err(e.decompress(f).data, out) <= tol, (t, rel_err(e.decompress(f).data, out))
        assert rel_err(f.q, q) <= tol
