"""Seed derivation (host side).

Every random stream of the reference derives from one run seed as
``np.random.default_rng([seed, tag, *indices])`` (pkg/src/edgc/seeds.py:1-28).
The device path must consume exactly the same streams; what crosses into the
CUDA library is the resulting PCG64 (state, inc) pair.  ``pcg64_words`` reads
it from NumPy; ``pcg64_words_many`` / ``subsample_seeds`` restate NumPy's
SeedSequence pool hashing and PCG64 seeding (numpy/random/bit_generator.pyx,
``_pcg64.pyx`` / ``pcg64.h``, NumPy 2.x) vectorised over many seeds, because a
sampled iteration needs one stream per matrix (208 for GPT2-2.5B: ~20 ms of
host time through ``default_rng``, ~1 ms here).  Both are pinned to NumPy
word for word in tests/test_host.py.
"""

from __future__ import annotations

import numpy as np

__all__ = ["TAG_SYNTH", "TAG_SUBSAMPLE", "TAG_BASIS", "TAG_DATA", "TAG_TEACHER", "TAG_INIT", "TAG_BATCH",
           "TAG_TABLE", "TAG_NOISE", "TAG_LABEL_NOISE", "rng", "pcg64_words", "pcg64_words_many", "subsample_seed",
           "subsample_seeds", "state_seeds"]

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


# SeedSequence constants (bit_generator.pyx) and the PCG64 multiplier (pcg64.h)
_INIT_A, _MULT_A, _INIT_B, _MULT_B = 0x43B0D7E5, 0x931E8875, 0x8B51F9DD, 0x58F38DED
_MIX_L, _MIX_R = 0xCA01F9DD, 0x4973F715
_M32 = np.uint64(0xFFFFFFFF)
_PCG_MULT = (2549297995355413924 << 64) + 4865540595714422341
_MASK128 = (1 << 128) - 1


def _words32(x: int) -> list[int]:
    """An entropy int as SeedSequence coerces it: little-endian 32-bit words, 0 -> [0]."""
    if x < 0:
        raise ValueError("seeds must be non-negative")
    out = [x & 0xFFFFFFFF]
    x >>= 32
    while x:
        out.append(x & 0xFFFFFFFF)
        x >>= 32
    return out


def _seedseq_state(entropy: np.ndarray) -> np.ndarray:
    """SeedSequence(entropy_row).generate_state(4, uint64) for every row of a (B, L) uint64 array
    of 32-bit words (all rows the same length): the mix_entropy pool, then the output hash."""
    e = entropy.astype(np.uint64)
    B, L = e.shape
    hc = _INIT_A

    def hashmix(v):
        nonlocal hc
        v = v ^ np.uint64(hc)
        hc = (hc * _MULT_A) & 0xFFFFFFFF
        v = (v * np.uint64(hc)) & _M32
        return v ^ (v >> np.uint64(16))

    def mix(x, y):
        r = (np.uint64(_MIX_L) * x - np.uint64(_MIX_R) * y) & _M32   # uint64 wraps mod 2^64
        return r ^ (r >> np.uint64(16))

    pool = [hashmix(e[:, i] if i < L else np.zeros(B, np.uint64)) for i in range(4)]
    for src in range(4):
        for dst in range(4):
            if src != dst:
                pool[dst] = mix(pool[dst], hashmix(pool[src]))
    for src in range(4, L):
        for dst in range(4):
            pool[dst] = mix(pool[dst], hashmix(e[:, src]))
    hb = _INIT_B
    words = []
    for i in range(8):
        v = pool[i % 4] ^ np.uint64(hb)
        hb = (hb * _MULT_B) & 0xFFFFFFFF
        v = (v * np.uint64(hb)) & _M32
        words.append(v ^ (v >> np.uint64(16)))
    return np.stack([words[2 * j] | (words[2 * j + 1] << np.uint64(32)) for j in range(4)], axis=1)


def _entropy_rows(seeds) -> dict[int, tuple[list[int], np.ndarray]]:
    """Group seeds (ints or int sequences) by the length of their word expansion."""
    groups: dict[int, tuple[list[int], list[list[int]]]] = {}
    for i, sd in enumerate(seeds):
        parts = [sd] if isinstance(sd, (int, np.integer)) else list(sd)
        w = [x for p in parts for x in _words32(int(p))]
        groups.setdefault(len(w), ([], []))
        groups[len(w)][0].append(i)
        groups[len(w)][1].append(w)
    return {k: (ix, np.array(rows, dtype=np.uint64)) for k, (ix, rows) in groups.items()}


def _pcg64_seeded(v: np.ndarray) -> tuple[int, int]:
    """PCG64 (state, inc) after pcg64_set_seed(seed = v[0:2], inc = v[2:4])."""
    initstate = (int(v[0]) << 64) | int(v[1])
    initseq = (int(v[2]) << 64) | int(v[3])
    inc = ((initseq << 1) | 1) & _MASK128
    state = inc                                            # step from 0
    state = (state + initstate) & _MASK128
    state = (state * _PCG_MULT + inc) & _MASK128
    return state, inc


def pcg64_words_many(seeds) -> list[tuple[int, int, int, int]]:
    """``[pcg64_words(s) for s in seeds]`` without a Generator per seed (entries: ints or int lists)."""
    out: list = [None] * len(seeds)
    for _, (ix, rows) in _entropy_rows(seeds).items():
        st = _seedseq_state(rows)
        for i, v in zip(ix, st):
            s, inc = _pcg64_seeded(v)
            out[i] = ((s >> 64) & _MASK64, s & _MASK64, (inc >> 64) & _MASK64, inc & _MASK64)
    return out


def _xsl_rr(state: int) -> int:
    x = ((state >> 64) ^ state) & _MASK64
    rot = state >> 122
    return ((x >> rot) | (x << ((64 - rot) & 63))) & _MASK64


def subsample_seeds(run_seed: int, iteration: int, layers: int) -> list[int]:
    """``[subsample_seed(run_seed, iteration, k) for k in range(layers)]``: integers(2**31) of each
    stream is the low 32 bits of its first PCG64 output (the buffered next_uint32) times 2^31
    >> 32 (Lemire with rng_excl = 2^31 never rejects)."""
    seeds = [(run_seed, TAG_SUBSAMPLE, iteration, k) for k in range(layers)]
    out = []
    for w in pcg64_words_many(seeds):
        state, inc = (w[0] << 64) | w[1], (w[2] << 64) | w[3]
        state = (state * _PCG_MULT + inc) & _MASK128
        out.append((_xsl_rr(state) & 0xFFFFFFFF) >> 1)
    return out


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
