"""CPU: the device sample-plan ALGORITHM (csrc/sample_plan.cu phases P2-P4),
emulated step for step in Python on the oracle's u32 stream, against NumPy.

This pins the parallel decomposition (walk with first-rejection windows, hash
lists, tail-shuffle chains, Floyd collision chains) independently of the GPU.
"""

import math

import numpy as np
import pytest

import oracle


def lemire(x, rng):
    excl = rng + 1
    m = x * excl
    val, left = m >> 32, m & 0xFFFFFFFF
    if left >= excl:
        return True, val
    thr = (0xFFFFFFFF - rng) % excl
    return left >= thr, val


def walk(seed, n_elems, count, window=64, K=8):
    """k_walk: bounded value of every step (speculative shifts, first-rejection windows)."""
    tail = n_elems > 10000 and count > n_elems // 20
    draws = oracle.pcg64_u32(seed, count + 4096 + 2 * count).astype(np.int64)
    step_rng = (lambda s: n_elems - 1 - s) if tail else (lambda s: n_elems - count + s)
    rv = [0] * count
    s = u = 0
    while s < count:                      # k_walk (speculative shifts 0..K-1)
        nvalid = min(window, count - s)
        vals = [[0] * window for _ in range(K)]
        rej = [[False] * window for _ in range(K)]
        for lane in range(nvalid):
            for j in range(K):
                ok, v = lemire(int(draws[u + lane + j]), step_rng(s + lane))
                vals[j][lane], rej[j][lane] = v, not ok
        cur, d, events, length = 0, 0, [], nvalid
        while True:
            f = next((l for l in range(cur, nvalid) if rej[d][l]), None)
            if f is None:
                break
            events.append(f)
            d += 1
            if d == K:
                length = f
                break
            cur = f
        for lane in range(length):
            sh = sum(1 for e in events if e <= lane)
            rv[s + lane] = vals[sh][lane]
        s += length
        u += length + len(events)
    return rv, tail


def emulate(seed, n_elems, count, window=64, K=8):
    rv, tail = walk(seed, n_elems, count, window, K)
    lists = {}                            # k_index (hash lists)
    for st in range(count):
        lists.setdefault(rv[st], []).append(st)

    def latest_before(key, before):
        c = [e for e in lists.get(key, []) if e < before]
        return max(c) if c else -1

    out = [0] * count                     # k_resolve
    base = n_elems - count
    for st in range(count):
        if tail:
            j = rv[st]
            t = latest_before(j, st)
            val = j
            if t >= 0:
                while True:
                    pos_t = n_elems - 1 - t
                    t2 = latest_before(pos_t, t)
                    if t2 < 0:
                        val = pos_t
                        break
                    t = t2
            out[count - 1 - st] = val
        else:
            cur, collide = st, False
            while True:
                v = rv[cur]
                if latest_before(v, cur) >= 0:
                    collide = True
                    break
                if v < base or v - base >= cur:
                    break
                cur = v - base
            out[st] = base + st if collide else rv[st]
    return np.asarray(out, dtype=np.int64)


@pytest.mark.parametrize("window,K", [(64, 8), (7, 4), (2048, 8)])
@pytest.mark.parametrize("n_elems,beta,seed", [
    (100, 0.5, 3), (101, 0.9, 1), (4096, 0.25, 1), (10000, 0.5, 4), (10001, 0.06, 4), (12000, 0.25, 5),
    (20000, 0.05, 9), (20000, 0.0501, 11), (40000, 0.999, 2), (7, 0.3, 5), (2, 0.5, 0), (300, 0.99, 8)])
def test_plan_algorithm_matches_numpy(n_elems, beta, seed, window, K):
    count = min(n_elems, math.ceil(beta * n_elems))
    if count == n_elems:
        pytest.skip("copy branch")
    ref = np.random.default_rng(seed).choice(n_elems, size=count, replace=False, shuffle=False)
    assert np.array_equal(emulate(seed, n_elems, count, window, K), ref)


def resolve_buckets(rv, n_elems, count, tail, bbits, order_seed=0):
    """k_bucket_hist / k_bucket_scan / k_bucket_resolve / k_bucket_out with 2^bbits-position
    buckets; the scatter order inside a bucket is deliberately shuffled (the device's is
    arbitrary)."""
    nb = -(-n_elems // (1 << bbits))
    buckets = [[] for _ in range(nb)]
    order = np.random.default_rng(order_seed).permutation(count)
    for st in order:                      # histogram + scatter (any order)
        buckets[rv[st] >> bbits].append(st)
    pred = [-1] * count
    z0 = n_elems - count
    wtail = [-1] * count
    for b, steps in enumerate(buckets):   # one CTA per bucket
        head = {}
        for st in steps:
            head.setdefault(rv[st], []).append(st)
        for st in steps:
            c = [t for t in head[rv[st]] if t < st]
            pred[st] = max(c) if c else -1
        if tail:
            for pos in range(max(b << bbits, z0), min((b + 1) << bbits, n_elems)):
                lim = n_elems - 1 - pos
                c = [t for t in head.get(pos, []) if t < lim]
                wtail[pos - z0] = max(c) if c else -1
    out = [0] * count                     # k_bucket_out
    base = n_elems - count
    for st in range(count):
        if tail:
            t, val = pred[st], rv[st]
            while t >= 0:
                pos = n_elems - 1 - t
                t2 = wtail[pos - z0]
                if t2 < 0:
                    val = pos
                    break
                t = t2
            out[count - 1 - st] = val
        else:
            cur, collide = st, False
            while True:
                if pred[cur] >= 0:
                    collide = True
                    break
                v = rv[cur]
                if v < base or v - base >= cur:
                    break
                cur = v - base
            out[st] = base + st if collide else rv[st]
    return np.asarray(out, dtype=np.int64)


@pytest.mark.parametrize("bbits", [3, 14])
@pytest.mark.parametrize("n_elems,beta,seed", [
    (100, 0.5, 3), (101, 0.9, 1), (4096, 0.25, 1), (10000, 0.5, 4), (10001, 0.06, 4), (12000, 0.25, 5),
    (20000, 0.05, 9), (20000, 0.0501, 11), (40000, 0.999, 2), (7, 0.3, 5), (2, 0.5, 0), (300, 0.99, 8)])
def test_bucketed_resolve_matches_numpy(n_elems, beta, seed, bbits):
    count = min(n_elems, math.ceil(beta * n_elems))
    if count == n_elems:
        pytest.skip("copy branch")
    ref = np.random.default_rng(seed).choice(n_elems, size=count, replace=False, shuffle=False)
    rv, tail = walk(seed, n_elems, count)
    assert np.array_equal(resolve_buckets(rv, n_elems, count, tail, bbits, order_seed=seed), ref)


def lemire_threshold(excl):
    """csrc/sample_plan.cu:lemire_threshold, restated with float32 rounding."""
    if excl < 65536:
        return (2**32 - excl) % excl
    q = int(np.float32(4294967296.0) * (np.float32(1.0) / np.float32(excl)))
    r = 2**32 - q * excl
    for _ in range(2):
        r += excl if r < 0 else 0
    for _ in range(2):
        r -= excl if r >= excl else 0
    return r


def test_lemire_threshold_fast_path():
    rng = np.random.default_rng(0)
    xs = list(rng.integers(1, 2**31, size=20000)) + [1, 2, 3, 65535, 65536, 65537, 2**31 - 1, 2**30, 3 << 29]
    xs += [int(x) for x in np.arange(65536, 65536 + 2000)]
    for x in xs:
        x = int(x)
        assert lemire_threshold(x) == (2**32 - x) % x, x
