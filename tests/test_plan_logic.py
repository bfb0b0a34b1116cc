"""CPU: the device sample-plan ALGORITHM (csrc/sample_plan.cu), emulated step
for step in Python on the oracle's u32 stream, against NumPy.

This pins the parallel decomposition (the warp walk with first-rejection chunks,
hash lists, tail-shuffle chains, Floyd collision chains, and the order-free
set-mode resolve) independently of the GPU.
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


def walk(seed, n_elems, count, chunk=256, max_rej=8):
    """k_walk: bounded value of every step.  A warp takes `chunk` consecutive steps against
    consecutive draws; rejections are settled in step order inside the chunk (from a rejecting
    step on, every step moves to the next draw and is tested again), up to `max_rej` per chunk,
    beyond which the chunk ends at the rejecting step."""
    tail = n_elems > 10000 and count > n_elems // 20
    draws = oracle.pcg64_u32(seed, 2 * count + 4096).astype(np.int64)
    step_rng = (lambda s: n_elems - 1 - s) if tail else (lambda s: n_elems - count + s)
    rv = [0] * count
    s = k = 0
    while s < count:
        ln = min(chunk, count - s)
        vals = [lemire(int(draws[k + p]), step_rng(s + p)) for p in range(ln)]
        adv, shift, skip, frm = ln, 0, 0, 0
        while True:
            first = next((p for p in range(frm, ln) if not vals[p][0]), None)
            if first is None:
                break
            if shift == max_rej:
                adv, skip = first, 1
                break
            shift += 1
            for p in range(first, ln):
                vals[p] = lemire(int(draws[k + p + shift]), step_rng(s + p))
            frm = first
        rv[s:s + adv] = [v for _, v in vals[:adv]]
        s += adv
        k += adv + shift + skip
    return rv, tail


def emulate(seed, n_elems, count, chunk=256, max_rej=8):
    rv, tail = walk(seed, n_elems, count, chunk, max_rej)
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


@pytest.mark.parametrize("chunk,max_rej", [(256, 8), (32, 1), (7, 0), (1, 0), (300, 2)])
@pytest.mark.parametrize("n_elems,beta,seed", [
    (100, 0.5, 3), (101, 0.9, 1), (4096, 0.25, 1), (10000, 0.5, 4), (10001, 0.06, 4), (12000, 0.25, 5),
    (20000, 0.05, 9), (20000, 0.0501, 11), (40000, 0.999, 2), (7, 0.3, 5), (2, 0.5, 0), (300, 0.99, 8),
    (2_000_000_000, 0.00001, 6)])
def test_plan_algorithm_matches_numpy(n_elems, beta, seed, chunk, max_rej):
    count = min(n_elems, math.ceil(beta * n_elems))
    if count == n_elems:
        pytest.skip("copy branch")
    ref = np.random.default_rng(seed).choice(n_elems, size=count, replace=False, shuffle=False)
    assert np.array_equal(emulate(seed, n_elems, count, chunk, max_rej), ref)


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


def sequential_rv(seed, n_elems, count):
    """Tail-shuffle bounded values j_s in step order (NumPy's sequential Lemire loop, vectorised
    between rejections): the walk's output, whose chunked form test_plan_algorithm_matches_numpy pins."""
    draws = oracle.pcg64_u32(seed, count + 8192 + count // 64).astype(np.uint64)
    excl = (n_elems - np.arange(count, dtype=np.uint64))          # i + 1 for step s
    rv = np.empty(count, dtype=np.int64)
    s = u = 0
    while s < count:
        k = min(count - s, 1 << 16)
        m = draws[u:u + k] * excl[s:s + k]
        left = m & np.uint64(0xFFFFFFFF)
        thr = (np.uint64(1 << 32) - excl[s:s + k]) % excl[s:s + k]
        bad = np.flatnonzero(left < thr)
        take = k if bad.size == 0 else int(bad[0])
        rv[s:s + take] = (m[:take] >> np.uint64(32)).astype(np.int64)
        s += take
        u += take + (0 if bad.size == 0 else 1)
    return rv.tolist()


def resolve_set(rv, n_elems, count, sbits):
    """k_set_sort / k_set_resolve / k_set_tail: the membership set of a tail-shuffle plan without
    NumPy's order.  Buckets of 2^sbits positions hold the packed (step in chunk, position) entries
    of every sort chunk; each computes M (latest non-self step per position) in any entry order,
    stores its D bits and marks the !last steps; the tail pass finishes positions >= z0."""
    chunk = 1 << sbits
    z0 = n_elems - count
    nb = -(-n_elems // chunk)
    bits = np.zeros(n_elems, dtype=np.uint8)
    notlast = np.zeros(count, dtype=bool)
    segs = [[] for _ in range(nb)]       # bucket b: (chunk, packed entry) of every sort chunk
    for i in range(count):                # k_set_sort: one chunk of steps per CTA
        c = i // chunk
        segs[rv[i] >> sbits].append((c, ((i - c * chunk) << sbits) | (rv[i] & (chunk - 1))))
    rng = np.random.default_rng(sbits)
    for b in range(nb):                   # k_set_resolve: one CTA per bucket
        ents = [(c * chunk + (e >> sbits), e & (chunk - 1)) for c, e in segs[b]]
        ents = [ents[k] for k in rng.permutation(len(ents))]   # atomics: any order
        ibase = n_elems - 1 - (b << sbits)
        M = {}
        for st, l in ents:
            if st != ibase - l:
                M[l] = max(M.get(l, -1), st)
        for l in M:
            bits[(b << sbits) + l] = 1
        for st, l in ents:
            if st != ibase - l and M[l] != st:
                notlast[st] = True
    for q in range(z0, n_elems):          # k_set_tail
        if bits[q]:
            continue
        s, good = n_elems - 1 - q, False
        while True:
            j = rv[s]
            if j == n_elems - 1 - s or notlast[s]:
                break
            if j < z0:
                good = True
                break
            s = n_elems - 1 - j
        if not good:
            bits[q] = 1
    return bits


@pytest.mark.parametrize("sbits", [2, 5, 15])
@pytest.mark.parametrize("n_elems,beta,seed", [
    (10001, 0.06, 4), (12000, 0.25, 5), (20000, 0.0501, 11), (40000, 0.999, 2), (65536, 0.25, 13),
    (262144, 0.5, 8), (30000, 0.75, 1)])
def test_set_resolve_matches_numpy_set(n_elems, beta, seed, sbits):
    count = min(n_elems, math.ceil(beta * n_elems))
    rv = sequential_rv(seed, n_elems, count)
    assert n_elems > 10000 and count > n_elems // 20
    ref = np.random.default_rng(seed).choice(n_elems, size=count, replace=False, shuffle=False)
    want = np.zeros(n_elems, dtype=np.uint8)
    want[ref] = 1
    got = resolve_set(rv, n_elems, count, sbits)
    assert np.array_equal(got, want)
    assert int(got.sum()) == count
    assert ref[-1] == rv[0]                # the bitmap-only plan's shift sample: step 0's own target
