"""Input specifications for the golden fixtures (shared by the generator and the tests).

Inputs are regenerated from these specs on whichever machine runs the tests;
every value is fp32-representable, so the device path (fp32 storage) and the
reference (float64) see identical numbers.  No dependency on /root/reference.
"""

from __future__ import annotations

import math

import numpy as np

# (N, beta, seed): both NumPy branches, the count == N//20 boundary (Floyd),
# the N <= 10000 rule, beta = 1 (copy), and GPT-2-shaped sizes.
CHOICE_GRID = [
    (1, 0.5, 0), (2, 0.5, 0), (7, 0.3, 5), (64, 1.0, 0), (100, 0.5, 3),
    (4096, 0.25, 1), (10000, 0.5, 4), (10001, 0.06, 4), (12000, 0.25, 5),
    (20000, 0.05, 9), (20000, 0.0501, 11), (40000, 0.999, 2), (65536, 0.25, 13),
    (262144, 0.05, 6), (262144, 0.5, 8),
    (4194304, 0.25, 17),                       # config 1 (1024x4096, tail)
    (3686400, 0.25, 0), (3686400, 0.05, 1),     # 1920x1920
    (11059200, 0.05, 19), (11059200, 0.25, 3), (11059200, 0.5, 2),  # 1920x5760
    (14745600, 0.25, 23),                      # 1920x7680
]

HIST_SETS = [
    {"kind": "gauss", "n": 1_000_003, "seed": 0, "scale": 1.0},
    {"kind": "gauss", "n": 1_000_003, "seed": 1, "scale": 1.0},
    {"kind": "gauss", "n": 1_048_576, "seed": 5, "scale": 1e-3},
    {"kind": "t3", "n": 777_777, "seed": 2, "scale": 1.0},
    {"kind": "t3", "n": 2_764_800, "seed": 7, "scale": 1e-2},
    {"kind": "uniform", "n": 250_000, "seed": 3, "scale": 1.0},
    {"kind": "quant", "n": 100_000, "seed": 4, "scale": 1.0},
    {"kind": "gauss", "n": 2, "seed": 8, "scale": 1.0},
    {"kind": "gauss", "n": 3, "seed": 9, "scale": 1.0},
    {"kind": "gauss", "n": 17, "seed": 10, "scale": 1.0},
    {"kind": "gauss", "n": 1000, "seed": 11, "scale": 1.0},
    {"kind": "quant", "n": 5, "seed": 12, "scale": 1.0},
    {"kind": "const", "n": 64, "seed": 0, "scale": 3.25},
]


def hist_samples(spec) -> np.ndarray:
    rng = np.random.default_rng([spec["seed"], 77])
    n, kind, scale = spec["n"], spec["kind"], np.float32(spec["scale"])
    if kind == "gauss":
        x = rng.standard_normal(n, dtype=np.float32) * scale
    elif kind == "t3":
        x = rng.standard_t(3, n).astype(np.float32) * scale
    elif kind == "uniform":
        x = rng.random(n, dtype=np.float32) * scale
    elif kind == "quant":
        x = (np.clip(np.rint(rng.standard_normal(n) * 8), -50, 50) * 0.125).astype(np.float32)
    elif kind == "const":
        x = np.full(n, scale, dtype=np.float32)
    else:
        raise ValueError(kind)
    return x.astype(np.float64)


COMPRESS_CASES = [
    {"m": 64, "n": 96, "rank": 4, "seed": 3, "steps": 6, "kind": "gauss"},
    {"m": 96, "n": 64, "rank": 8, "seed": 5, "steps": 4, "kind": "gauss"},
    {"m": 64, "n": 64, "rank": 8, "seed": 7, "steps": 5, "kind": "gauss", "set_rank_at": {2: 4, 3: 12}},
    {"m": 48, "n": 32, "rank": 8, "seed": 9, "steps": 1, "kind": "lowrank", "true_rank": 3},
    {"m": 6, "n": 8, "rank": 2, "seed": 0, "steps": 2, "kind": "zero"},
    {"m": 12, "n": 9, "rank": 1, "seed": 3, "steps": 1, "kind": "rank1"},
    {"m": 160, "n": 272, "rank": 16, "seed": 11, "steps": 3, "kind": "gauss"},
]


def compress_inputs(case, t: int) -> np.ndarray:
    m, n = case["m"], case["n"]
    rng = np.random.default_rng([case["seed"], 1, t, 0, 0])
    kind = case["kind"]
    if kind == "gauss":
        x = rng.standard_normal((m, n), dtype=np.float32) * np.float32(1e-2)
    elif kind == "lowrank":
        k = case["true_rank"]
        u = rng.integers(-2, 3, size=(m, k)).astype(np.float64)
        v = rng.integers(-2, 3, size=(k, n)).astype(np.float64)
        x = (u @ v).astype(np.float32)
    elif kind == "rank1":
        u = rng.integers(-4, 5, size=m).astype(np.float64)
        v = rng.integers(-4, 5, size=n).astype(np.float64)
        x = np.outer(u, v).astype(np.float32)
    elif kind == "zero":
        x = np.zeros((m, n), dtype=np.float32)
    else:
        raise ValueError(kind)
    return x.astype(np.float64)


_RANK_BASE = {
    "shape": [1024, 4096], "iterations": 200, "alpha": 0.1, "beta": 0.25, "window": 20,
    "step_limit": 8, "warmup_floor": 0.10, "r_min": 26, "r_max": 128, "trials": 64,
    "table_seed": 0, "sampler_seed": 0, "synth_seed": 0, "sigma0": 1e-2,
}
RANK_CASES = [_RANK_BASE | {"tau": 100.0}, _RANK_BASE | {"tau": 4000.0}]


def rank_case_sigma(case, t: int) -> float:
    return case["sigma0"] * math.exp(-t / case["tau"])


def rank_case_matrix(case, t: int) -> np.ndarray:
    """SynthSchedule(kind="exp") (grad_source.py:135-171) on the fp32 generator of SURVEY §8(d)."""
    m, n = case["shape"]
    z = np.random.default_rng([case["synth_seed"], 1, t, 0, 0]).standard_normal((m, n), dtype=np.float32)
    return z * np.float32(rank_case_sigma(case, t))


# EDGT trace replay + analyze-trace (grad_source.py:44-131, cli.py:579-659).
# Layers 0 and 1 share an element count (correlation pairs), layer 1 is
# correlated with layer 0, every layer decays like SynthSchedule's "exp" kind.
TRACE_SPEC = {"shapes": [(24, 40), (40, 24), (16, 16)], "iterations": 30, "seed": 7, "tau": 12.0,
              "window": 10, "alpha": 0.1, "beta": 0.25, "correlation_iterations": 4}


def trace_frames(spec=TRACE_SPEC):
    rng = np.random.default_rng(spec["seed"])
    frames = []
    for t in range(spec["iterations"]):
        s = np.float32(2.0 * math.exp(-t / spec["tau"]))
        a = rng.standard_normal(spec["shapes"][0]).astype(np.float32) * s
        noise = rng.standard_normal(spec["shapes"][1]).astype(np.float32) * s
        b = (np.float32(0.6) * a.reshape(spec["shapes"][1]) + np.float32(0.8) * noise).astype(np.float32)
        c = rng.standard_normal(spec["shapes"][2]).astype(np.float32) * s
        frames.append([a, b, c])
    return frames


# ---------------------------------------------------------------- DP driver
# train_toy's EDGC setup (grad_source.py:311-327) on these bucket sets pins the
# rank bounds (controller.py:111-163); DP_SCENARIO pins the window decisions.
def _gpt2(layer, layers):
    return [s for _ in range(layers) for s in layer]


DP_BOUND_SETS = {
    "gpt2_2p5b": _gpt2(((1920, 5760), (1920, 1920), (1920, 7680), (7680, 1920)), 52),
    "gpt2_12p1b": _gpt2(((3584, 10752), (3584, 3584), (3584, 14336), (14336, 3584)), 76),
    "gpt2_2p5b_layer": _gpt2(((1920, 5760), (1920, 1920), (1920, 7680), (7680, 1920)), 1),
    "dp_small": [(128, 512), (512, 128), (256, 256)],
    "dp_check": [(192, 576), (192, 192), (192, 768), (768, 192), (50, 70)],
}

DP_SCENARIO = {"shapes": [[128, 512], [512, 128], [256, 256]], "iters": 80, "window": 20, "alpha": 0.1,
               "beta": 0.25, "sigma0": 1e-2, "tau": 60.0, "synth_seed": 7}


def dp_scenario_grads(t: int, w: int):
    """Worker w's fp32 gradients at iteration t: sigma0 exp(-t / tau) standard normals (oracle.synth_matrix)."""
    import oracle
    sc = DP_SCENARIO
    s = sc["sigma0"] * math.exp(-t / sc["tau"])
    return [oracle.synth_matrix(sc["synth_seed"], t, k, w, m, n, s) for k, (m, n) in enumerate(sc["shapes"])]
