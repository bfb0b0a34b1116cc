"""Seed derivation (host side).

Every random stream of the reference derives from one run seed as
``np.random.default_rng([seed, tag, *indices])`` (pkg/src/edgc/seeds.py:1-28).
The device path must consume exactly the same streams, so these derivations
stay in NumPy on the host; what crosses into the CUDA library is the
resulting PCG64 (state, inc) pair (``pcg64_words``), never a re-implemented
SeedSequence.
"""

from __future__ import annotations

import numpy as np

__all__ = ["TAG_SYNTH", "TAG_SUBSAMPLE", "TAG_BASIS", "TAG_DATA", "TAG_TEACHER", "TAG_INIT", "TAG_BATCH",
           "TAG_TABLE", "TAG_NOISE", "TAG_LABEL_NOISE", "rng", "pcg64_words", "subsample_seed", "state_seeds"]

# stream tags — values fixed by the reference (seeds.py:14-23)
TAG_SYNTH, TAG_SUBSAMPLE, TAG_BASIS, TAG_DATA, TAG_TEACHER = 1, 2, 3, 4, 5
TAG_INIT, TAG_BATCH, TAG_TABLE, TAG_NOISE, TAG_LABEL_NOISE = 6, 7, 8, 9, 10

_MASK64 = (1 << 64) - 1


def rng(seed: int, tag: int, *indices: int) -> np.random.Generator:
    """The Generator of stream (seed, tag, *indices); indices must be >= 0."""
    return np.random.default_rng([seed, tag, *indices])


def pcg64_words(seed) -> tuple[int, int, int, int]:
    """(state_hi, state_lo, inc_hi, inc_lo) of default_rng(seed)'s PCG64, for the device sampler."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    return (s >> 64) & _MASK64, s & _MASK64, (inc >> 64) & _MASK64, inc & _MASK64


def subsample_seed(run_seed: int, iteration: int, layer: int) -> int:
    """Sampler seed of (iteration, layer): entropy.py:170-174."""
    return int(rng(run_seed, TAG_SUBSAMPLE, iteration, layer).integers(2**31))


def state_seeds(seed: int, workers: int, layers: int) -> dict[tuple[int, int], int]:
    """Basis seed of every (worker, layer) CompressorState: grad_source.py:440-447."""
    children = np.random.SeedSequence([seed, TAG_BASIS]).spawn(workers * layers)
    out = {}
    for w in range(workers):
        for k in range(layers):
            out[(w, k)] = int(children[w * layers + k].generate_state(1)[0])
    return out
