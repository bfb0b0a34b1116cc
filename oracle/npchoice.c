/*
 * ORACLE — test infrastructure only. Never linked into the product path.
 *
 * Plain-C restatement of the index rule behind
 *     np.random.default_rng(seed).choice(N, size=count, replace=False, shuffle=False)
 * as called by the reference at /root/reference/pkg/src/edgc/entropy.py:78
 * (subsample_entries, entropy.py:67-79).
 *
 * The algorithm lives in the third-party dependency NumPy (pinned: numpy 2.3.5,
 * the version installed with the reference; `numpy>=1.24` in
 * /root/reference/pkg/pyproject.toml:10).  Its Cython/C source is not shipped in
 * site-packages, so this file restates the published algorithm:
 *
 *   PCG64 (pcg_setseq_128_xsl_rr_64): state <- state * MULT + inc, then
 *     out = rotr64(hi(state) ^ lo(state), state >> 122).
 *   next_uint32: low half of a fresh 64-bit draw first, buffered high half next.
 *   bounded(0..rng) (random_bounded_uint64 -> Lemire 32-bit for rng < 2^32-1):
 *     rng == 0 -> 0 without a draw; else m = u32 * (rng+1); if lo32(m) < rng+1,
 *     threshold = (2^32-1 - rng) % (rng+1); redraw while lo32(m) < threshold;
 *     return hi32(m).
 *   Branch: "tail shuffle" iff N > 10000 and count > N // 20, else Floyd.
 *   Tail shuffle: data = arange(N); for i = N-1 down to max(N-count, 1):
 *     j = bounded(0..i); swap(data[i], data[j]); output data[N-count:].
 *   Floyd: for j in [N-count, N): v = bounded(0..j); output v if not yet
 *     output, else output j.
 *
 * The restatement is pinned against NumPy itself by tests/golden/make_golden.py
 * (index checksums over a grid covering both branches and the count == N//20
 * boundary) and tests/test_oracle.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

#define PCG_MULT ((((u128)0x2360ED051FC65DA4ULL) << 64) | (u128)0x4385DF649FCCF645ULL)

typedef struct {
    u128 state;
    u128 inc;
    int has32;
    uint32_t buf32;
} pcg64_t;

static inline uint64_t pcg64_next64(pcg64_t *g) {
    g->state = g->state * PCG_MULT + g->inc;
    uint64_t hi = (uint64_t)(g->state >> 64), lo = (uint64_t)g->state;
    unsigned rot = (unsigned)(g->state >> 122);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64 - rot) & 63));
}

static inline uint32_t pcg64_next32(pcg64_t *g) {
    if (g->has32) {
        g->has32 = 0;
        return g->buf32;
    }
    uint64_t v = pcg64_next64(g);
    g->has32 = 1;
    g->buf32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
}

static inline uint64_t bounded(pcg64_t *g, uint64_t rng, uint64_t *ndraws) {
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFULL) { (*ndraws)++; return pcg64_next32(g); }
    const uint32_t excl = (uint32_t)rng + 1u;
    uint64_t m = (uint64_t)pcg64_next32(g) * excl;
    (*ndraws)++;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
        const uint32_t thr = (uint32_t)(0xFFFFFFFFu - (uint32_t)rng) % excl;
        while (left < thr) {
            m = (uint64_t)pcg64_next32(g) * excl;
            (*ndraws)++;
            left = (uint32_t)m;
        }
    }
    return m >> 32;
}

/* 1 = tail shuffle, 0 = Floyd (NumPy's branch rule). */
int oracle_choice_branch(int64_t N, int64_t count) {
    return (N > 10000 && count > N / 20) ? 1 : 0;
}

/*
 * Writes `count` indices into out.  Returns the number of u32 draws consumed,
 * or -1 on invalid arguments (N >= 2^32 is outside what this restatement covers:
 * NumPy would switch to 64-bit draws there).
 */
int64_t oracle_choice(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                      int64_t N, int64_t count, int64_t *out) {
    if (N < 1 || count < 0 || count > N || N > 0xFFFFFFFFLL) return -1;
    pcg64_t g;
    g.state = (((u128)state_hi) << 64) | state_lo;
    g.inc = (((u128)inc_hi) << 64) | inc_lo;
    g.has32 = 0;
    g.buf32 = 0;
    uint64_t ndraws = 0;
    if (oracle_choice_branch(N, count)) {
        int64_t *data = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
        if (!data) return -1;
        for (int64_t i = 0; i < N; i++) data[i] = i;
        int64_t first = N - count > 1 ? N - count : 1;
        for (int64_t i = N - 1; i >= first; i--) {
            int64_t j = (int64_t)bounded(&g, (uint64_t)i, &ndraws);
            int64_t t = data[i];
            data[i] = data[j];
            data[j] = t;
        }
        memcpy(out, data + (N - count), sizeof(int64_t) * (size_t)count);
        free(data);
    } else {
        /* open-addressing set sized like NumPy's (power of two >= 1.2*count) */
        int64_t cap = 1;
        while (cap < count + count / 5 + 1) cap <<= 1;
        int64_t *set = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
        if (!set) return -1;
        for (int64_t i = 0; i < cap; i++) set[i] = -1;
        const int64_t mask = cap - 1;
        for (int64_t j = N - count; j < N; j++) {
            int64_t v = (int64_t)bounded(&g, (uint64_t)j, &ndraws);
            int64_t loc = v & mask;
            while (set[loc] != -1 && set[loc] != v) loc = (loc + 1) & mask;
            if (set[loc] == -1) {
                set[loc] = v;
                out[j - (N - count)] = v;
            } else {
                loc = j & mask;
                while (set[loc] != -1) loc = (loc + 1) & mask;
                set[loc] = j;
                out[j - (N - count)] = j;
            }
        }
        free(set);
    }
    return (int64_t)ndraws;
}

/* Raw u32 stream (next_uint32 semantics) — used to pin the device generator. */
void oracle_pcg64_u32(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                      int64_t n, uint32_t *out) {
    pcg64_t g;
    g.state = (((u128)state_hi) << 64) | state_lo;
    g.inc = (((u128)inc_hi) << 64) | inc_lo;
    g.has32 = 0;
    g.buf32 = 0;
    for (int64_t i = 0; i < n; i++) out[i] = pcg64_next32(&g);
}
