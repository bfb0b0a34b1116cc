// Sample plan: NumPy-exact sampled indices on the device.
//
// Replaces np.random.default_rng(seed).choice(N, count, replace=False,
// shuffle=False) at /root/reference/pkg/src/edgc/entropy.py:78.  The NumPy
// algorithm (restated in oracle/npchoice.c) is sequential: a partial
// Fisher-Yates over arange(N) ("tail", N > 10000 and count > N//20) or
// Floyd's algorithm, each step consuming Lemire-bounded 32-bit draws from
// PCG64 with rare, value-dependent rejections.  The device plan splits it
// into four data-parallel phases:
//   P1 draws    every thread jumps PCG64 ahead to its own chunk and writes the
//               u32 stream (low half first, as next_uint32 buffers it);
//   P2 walk     one CTA per plan assigns draws to steps: 1024 lanes test 1024
//               consecutive steps against their draws in parallel, a CTA-wide
//               vote finds the first Lemire rejection, and the window slides
//               past it (rejections are ~1e-3 per step at GPT-2 sizes);
//   P3 index    (key = bounded value, step) pairs go into an open-addressing
//               hash table with per-key step lists;
//   P4 resolve  tail: out[i] = value at position j just before step i, found
//               by following "last earlier writer" links (chains are a few
//               links deep); Floyd: a draw collides iff it equals an earlier
//               draw or an earlier collided step's j.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "ptx.cuh"

namespace edgc {
namespace {

typedef unsigned __int128 u128;

__host__ __device__ __forceinline__ u128 pcg_mult() {
    return (((u128)0x2360ED051FC65DA4ULL) << 64) | (u128)0x4385DF649FCCF645ULL;
}

__device__ __forceinline__ uint64_t pcg_output(u128 s) {
    const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
    const unsigned rot = (unsigned)(s >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

// affine map of `delta` LCG steps: state -> mult * state + plus (pcg_advance_lcg_128)
__device__ __forceinline__ void pcg_affine(u128 inc, uint64_t delta, u128 &mult, u128 &plus) {
    u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
    while (delta) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    mult = acc_mult;
    plus = acc_plus;
}

__device__ __forceinline__ u128 pcg_jump(u128 state, u128 inc, uint64_t delta) {
    u128 a, c;
    pcg_affine(inc, delta, a, c);
    return a * state + c;
}

struct PlanDev {
    u128 state, inc;
    int64_t n_elems, count;
    int32_t *idx;
    uint32_t *bitmap;  // optional membership bits
    int32_t *rv;       // [count] bounded values
    int32_t *next;     // [count]
    int32_t *head;     // [n_elems] latest step targeting each position (-1: none)
    int32_t tail;      // 1 = tail shuffle, 0 = Floyd
    int64_t step_block0;  // first P3/P4 block index of this plan
    // bucketed resolve (tail-shuffle plans; see k_bucket_sort)
    int32_t *lst_s, *lst_j;   // [count] each chunk's steps sorted by bucket, and their bounded values
    int32_t *segoff;          // [nch][nb + 1] per chunk: start of each bucket's segment in the chunk
    int32_t *pred;            // chain list: latest earlier step that wrote the step's target
    int32_t *wtail;           // [count] latest step before N-1-p that wrote tail position p >= N-count
    int32_t *nchain;          // chain list length
    int32_t nb, nch;          // buckets, sort chunks
    int32_t bucketed;         // 1: bucket path, 0: global head-table path
    int32_t setmode;          // 1: membership set only (k_set_*), the order-free resolve
    uint32_t *lst_pk;         // set mode: [count] (step in chunk << kSBits) | position in bucket
    uint32_t *notlast;        // set mode: [ceil(count/32)] bit s: a later step hits rv[s] again
    int32_t full_idx;         // 0: EDGC_PLAN_BITMAP_ONLY (only idx[0] is written)
    int64_t chunk0;           // first sort CTA of this plan
    int64_t bucket0;          // first bucket-resolve CTA of this plan
    int64_t oblock0;          // first chain-pass CTA of this plan
};

constexpr int kStepThreads = 256;

__device__ __forceinline__ int find_plan(const PlanDev *plans, int n, int64_t blk) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (plans[mid].step_block0 <= blk) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// 2^32 mod excl (NumPy's Lemire threshold (2^32 - excl) % excl), excl >= 1.  For
// excl >= 2^16 the quotient is < 2^16, so a float reciprocal estimate is within
// +-2 of it and two exact corrections finish; smaller excl take the division.
__device__ __forceinline__ uint32_t lemire_threshold(uint32_t excl) {
    if (excl < 65536u) return (0u - excl) % excl;
    const uint32_t q = (uint32_t)(4294967296.0f * __frcp_rn((float)excl));
    int64_t r = (int64_t)4294967296ll - (int64_t)q * (int64_t)excl;
    r += (r < 0) ? (int64_t)excl : 0;
    r += (r < 0) ? (int64_t)excl : 0;
    r -= (r >= (int64_t)excl) ? (int64_t)excl : 0;
    r -= (r >= (int64_t)excl) ? (int64_t)excl : 0;
    return (uint32_t)r;
}

// ---- P1: the walk -- bounded value of every step ------------------------------
// The NumPy walk is sequential: step s takes the next unused u32 draw (NumPy's
// next_uint32: low half of each PCG64 output first) and a Lemire rejection
// consumes one extra draw.  Rejections are rare (first-stage test p ~ excl/2^32,
// ~3e-3 at GPT-2 sizes), so one walker warp takes kWalkQ * 32 consecutive steps
// per chunk -- lane l steps s + l + 32 q against draws k + l + 32 q: one multiply
// and compare per step, one ballot per chunk -- and when a step rejects, the chunk
// ends at the first rejecting step (in step order), whose draw is skipped.
// Generating the draws is most of the arithmetic (a 128-bit LCG step per two
// draws) and does not depend on the walk, so a producer warp per plan fills a
// shared ring of kWalkBlk-draw blocks ahead of the walker (smem counters, no HBM
// draw buffer).  Plans per CTA: kWalkPlans for plans built ahead on a side stream
// (few SMs held for the longer walk), 1 with EDGC_PLAN_LATENCY (the walk is on
// the step's critical path: every SM to itself).
#ifndef EDGC_WALK_PLANS
#define EDGC_WALK_PLANS 16
#endif
constexpr int kWalkPlans = EDGC_WALK_PLANS;  // plans per CTA (a walker and a producer warp each)
constexpr int kWalkQ = 8;                   // steps per walker lane per chunk
constexpr int kWalkChunk = 32 * kWalkQ;
constexpr int kWalkMaxRej = 8;              // rejections settled inside one chunk (ring lookahead)
constexpr int kWalkBlk = 512;               // draws per ring block
// ring blocks: 4 with kWalkPlans rings per CTA (plans built ahead), 32 with one (latency mode:
// the producer runs up to 16K draws ahead, so its back-off while the ring is full never
// starves the walker)
constexpr int kWalkNBlkAhead = 4, kWalkNBlkLat = 32;
constexpr int kWalkThreads = 64 * kWalkPlans;
static_assert(kWalkBlk % 64 == 0, "whole outputs per producer lane");
static_assert(kWalkChunk + kWalkMaxRej <= kWalkBlk, "a chunk spans at most two blocks");
static_assert((kWalkChunk + kWalkMaxRej) % 2 == 0, "the mirror copies whole outputs");

constexpr int kWalkPad = kWalkChunk + kWalkMaxRej;   // ring head mirrored past its end: no index wrap
template <int NBLK>
struct alignas(16) WalkRing {
    static constexpr int kRing = kWalkBlk * NBLK;
    uint32_t d[kRing + kWalkPad];
    uint64_t full[NBLK];    // producer -> walker: block written
    uint64_t empty[NBLK];   // walker -> producer: block consumed
    volatile int done;
};

// mbarrier probe that suspends the thread up to the hint (ns) while the phase is pending
__device__ __forceinline__ bool walk_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 2000;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(ptx::smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void walk_wait(uint64_t *bar, uint32_t parity) {
    while (!walk_try_wait(bar, parity)) {
    }
}

template <int NBLK, int BACKOFF_NS>
__global__ void __launch_bounds__(kWalkThreads) k_walk(const PlanDev *plans, int n_plans, const int32_t *order,
                                                       int ppc) {
    constexpr int kWalkNBlk = NBLK, kWalkRing = WalkRing<NBLK>::kRing;
    extern __shared__ __align__(16) unsigned char walk_raw[];
    const int g = threadIdx.x >> 6;                 // plan group in the CTA
    const bool producer = (threadIdx.x >> 5) & 1;
    const int lane = threadIdx.x & 31;
    const int slot = blockIdx.x * ppc + g;
    WalkRing<NBLK> &R = reinterpret_cast<WalkRing<NBLK> *>(walk_raw)[g];
    if ((threadIdx.x & 63) == 0) {
        for (int i = 0; i < kWalkNBlk; ++i) {
            ptx::mbar_init(&R.full[i], 1);
            ptx::mbar_init(&R.empty[i], 1);
        }
        R.done = 0;
    }
    __syncthreads();
    if (slot >= n_plans) return;   // whole group leaves (groups synchronise only among themselves)
    const PlanDev &P = plans[order[slot]];
    const uint32_t count = (uint32_t)P.count;
    if (producer) {
        // lane l writes outputs o = blk * kWalkBlk / 2 + l + 32 t of each block; output t comes from
        // chain t % kChains, each chain stepping 32 kChains outputs at a time, so the 128-bit LCG
        // steps of a block form kChains independent dependency chains instead of one
        constexpr int kPer = kWalkBlk / 64;                        // outputs per lane per block
        constexpr int kChains = 4;
        static_assert(kPer % kChains == 0, "whole chain rounds per block");
        u128 stc[kChains];
#pragma unroll
        for (int ch = 0; ch < kChains; ++ch)
            stc[ch] = pcg_jump(P.state, P.inc, (uint64_t)lane + 1u + 32u * ch);   // state after output lane + 32 ch
        u128 a, c;
        pcg_affine(P.inc, 32 * kChains, a, c);
        for (uint32_t blk = 0;; ++blk) {
            const uint32_t sl = blk % kWalkNBlk;
            // block blk - kWalkNBlk handed back?  The walker may finish first: it only sets done.
            // Lane 0 waits and decides for the warp (a lane-divergent exit would leave the others'
            // __syncwarp waiting on exited lanes); the __syncwarp orders its acquire before the writes
            int stop = 0;
            if (lane == 0) {
                if (blk >= kWalkNBlk)
                    while (!walk_try_wait(&R.empty[sl], ((blk / kWalkNBlk) - 1) & 1)) {
                        if (R.done) { stop = 1; break; }
                        __nanosleep(BACKOFF_NS);   // try_wait suspends only ~0.1 us: back off so the walkers issue
                    }
                if (R.done) stop = 1;
            }
            if (__shfl_sync(0xffffffffu, stop, 0)) return;
            __syncwarp();
            uint2 *dst = reinterpret_cast<uint2 *>(R.d + sl * kWalkBlk);
#pragma unroll
            for (int t = 0; t < kPer; ++t) {
                u128 &st = stc[t % kChains];
                const uint64_t v = pcg_output(st);
                st = a * st + c;
                const uint2 w = make_uint2((uint32_t)v, (uint32_t)(v >> 32));
                dst[lane + 32 * t] = w;
                // the ring's first kWalkPad draws again past its end, so a chunk reads one straight run
                if (sl == 0 && 2 * (lane + 32 * t) < kWalkPad)
                    *reinterpret_cast<uint2 *>(R.d + kWalkRing + 2 * (lane + 32 * t)) = w;
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&R.full[sl]);   // release: the block's writes before the arrival
        }
    }
    // walker
    const uint32_t tail = (uint32_t)P.tail;
    // excl = rng + 1 of step s: tail i + 1 = N - s; Floyd j + 1 = N - count + s + 1
    const uint32_t e0 = tail ? (uint32_t)P.n_elems : (uint32_t)(P.n_elems - P.count + 1);
    int32_t *rv = P.rv;
    uint32_t s = 0, k = 0;       // next step, next draw (N < 2^31)
    uint32_t have = 0, freed = 0; // blocks waited for / handed back
    while (s < count) {
        const uint32_t need = (k + kWalkChunk + kWalkMaxRej + kWalkBlk) / kWalkBlk;
        for (; have < need; ++have) walk_wait(&R.full[have % kWalkNBlk], (have / kWalkNBlk) & 1);
        const uint32_t base = s + lane;
        const uint32_t len = min((uint32_t)kWalkChunk, count - s);
        const bool full = len == kWalkChunk;
        const uint32_t *rp = R.d + (k & (kWalkRing - 1)) + lane;   // draw of step base + 32 q: rp[32 q]
        const uint32_t ex0 = tail ? e0 - base : e0 + base;
        const uint32_t dex = tail ? 0u - 32u : 32u;
        uint64_t m[kWalkQ];
        uint32_t excl[kWalkQ];
        uint32_t cm = 0;   // bit q: step base + 32 q is a rejection candidate
#pragma unroll
        for (int q = 0; q < kWalkQ; ++q) {
            excl[q] = ex0 + dex * q;
            m[q] = (uint64_t)rp[32 * q] * excl[q];
            cm |= (uint32_t)((uint32_t)m[q] < excl[q] && (full || lane + 32u * q < len)) << q;
        }
        uint32_t adv = len, shift = 0, skip = 0;   // shift: rejections so far in this chunk
        if (__ballot_sync(0xffffffffu, cm != 0)) {
            // settle rejections in step order: from the first rejecting step f on, every step
            // moves to the next draw (f itself retries) and is tested again
            uint32_t from = 0;
            while (true) {
                uint32_t first = 0xFFFFFFFFu;
                for (uint32_t c = cm; c; c &= c - 1) {   // candidates in step order
                    const int q = __ffs(c) - 1;
                    const uint32_t p = 32u * q + lane;
                    if (p >= from && (uint32_t)m[q] < lemire_threshold(excl[q])) { first = p; break; }
                }
                first = __reduce_min_sync(0xffffffffu, first);
                if (first == 0xFFFFFFFFu) break;
                if (shift == kWalkMaxRej) {   // burst beyond the ring's lookahead: end the chunk here
                    adv = first;
                    skip = 1;
                    break;
                }
                ++shift;
#pragma unroll
                for (int q = 0; q < kWalkQ; ++q) {
                    const uint32_t p = 32u * q + lane;
                    if (p >= first) {
                        m[q] = (uint64_t)rp[32 * q + shift] * excl[q];
                        cm = (cm & ~(1u << q)) | ((uint32_t)(p < len && (uint32_t)m[q] < excl[q]) << q);
                    }
                }
                from = first;
            }
        }
        int32_t *out = rv + base;
        if (adv == kWalkChunk) {
#pragma unroll
            for (int q = 0; q < kWalkQ; ++q) out[32 * q] = (int32_t)(m[q] >> 32);
        } else {
#pragma unroll
            for (int q = 0; q < kWalkQ; ++q)
                if (lane + 32u * q < adv) out[32 * q] = (int32_t)(m[q] >> 32);
        }
        s += adv;
        k += adv + shift + skip;
        __syncwarp();   // every lane's ring reads before blocks are handed back
        for (; freed < k / kWalkBlk; ++freed)
            if (lane == 0) ptx::mbar_arrive(&R.empty[freed % kWalkNBlk]);
    }
    if (lane == 0) R.done = 1;
}

__device__ __forceinline__ int find_plan_steps(const PlanDev *plans, int n, int64_t blk) {
    return find_plan(plans, n, blk);
}

// ---- P3: per-position lists of the steps whose bounded value is that position
// (direct-mapped heads: one atomic exchange per step, no probing)
__global__ void __launch_bounds__(kStepThreads) k_index(const PlanDev *plans, int p0, int p1, int64_t blk0) {
    const int p = p0 + find_plan_steps(plans + p0, p1 - p0, blk0 + blockIdx.x);
    const PlanDev P = plans[p];
    const int64_t s = (int64_t)(blk0 + blockIdx.x - P.step_block0) * kStepThreads + threadIdx.x;
    if (P.bucketed || s >= P.count) return;
    P.next[s] = atomicExch(P.head + P.rv[s], (int32_t)s);
}

__device__ __forceinline__ int32_t lookup_head(const PlanDev &P, int32_t key) { return P.head[key]; }

// largest step < before in the list of `key` (or -1)
__device__ __forceinline__ int32_t latest_before(const PlanDev &P, int32_t key, int32_t before) {
    int32_t best = -1;
    for (int32_t e = lookup_head(P, key); e >= 0; e = P.next[e])
        if (e < before && e > best) best = e;
    return best;
}

// ---- P4: resolve chains / collisions ---------------------------------------
__global__ void __launch_bounds__(kStepThreads) k_resolve(const PlanDev *plans, int p0, int p1, int64_t blk0) {
    const int p = p0 + find_plan_steps(plans + p0, p1 - p0, blk0 + blockIdx.x);
    const PlanDev P = plans[p];
    const int64_t s64 = (int64_t)(blk0 + blockIdx.x - P.step_block0) * kStepThreads + threadIdx.x;
    if (P.bucketed || s64 >= P.count) return;
    const int32_t s = (int32_t)s64;
    const int64_t N = P.n_elems, count = P.count;
    if (P.tail) {
        // step s swaps positions i = N-1-s and j = rv[s]; out[count-1-s] is the
        // value sitting at j just before step s.
        const int32_t j = P.rv[s];
        int32_t t = latest_before(P, j, s);
        int64_t val = j;
        if (t >= 0) {
            // value deposited at j by step t = value at position i_t before step t
            while (true) {
                const int32_t pos_t = (int32_t)(N - 1 - t);
                const int32_t t2 = latest_before(P, pos_t, t);
                if (t2 < 0) { val = pos_t; break; }
                t = t2;
            }
        }
        if (P.full_idx || s == count - 1) P.idx[count - 1 - s] = (int32_t)val;
        if (P.bitmap) atomicOr(P.bitmap + (val >> 5), 1u << (val & 31));
    } else {
        const int64_t base = N - count;
        int32_t cur = s;
        bool collide = false;
        // collision(t) = [v_t drawn at an earlier step] or [v_t == j_t' of an
        // earlier step t' that itself collided]; v_t == j_t (t' == t) is a fresh value
        while (true) {
            const int32_t v = P.rv[cur];
            if (latest_before(P, v, cur) >= 0) { collide = true; break; }
            if (v < base) break;
            const int32_t prev = (int32_t)(v - base);
            if (prev >= cur) break;
            cur = prev;
        }
        const int32_t outv = collide ? (int32_t)(base + s) : P.rv[s];
        if (P.full_idx || s == 0) P.idx[s] = outv;
        if (P.bitmap) atomicOr(P.bitmap + (outv >> 5), 1u << (outv & 31));
    }
}


// ---- P3/P4, bucketed (tail-shuffle plans, N <= 2^25) -------------------------
// The tail-shuffle resolve needs per-position list queries: pred(s) = the
// latest earlier step whose bounded value equals rv[s], and for each tail
// position p the latest step before N-1-p that targeted p.  Instead of a
// global N-entry head table (random L2/DRAM atomics, a memset per plan):
//   sort     each 32K-step chunk orders its steps by 8K-position bucket in
//            shared memory and writes the block back contiguously (full
//            sectors), with the per-bucket segment offsets;
//   resolve  one CTA per bucket gathers the bucket's segment from every chunk
//            into shared memory, builds the position lists there (int16
//            links) and answers all of the bucket's queries.  A step whose
//            target no earlier step wrote outputs the target itself -- a
//            position of the bucket -- so its membership bit is set in the
//            bucket's shared bitmap, which is then stored whole (no global
//            atomics, no pre-zeroed bitmap); the ~12% of steps whose target
//            was already written go to a chain list;
//   chain    value at j_s before step s = the value an earlier step t moved
//            there = the value at i_t = N-1-t before step t, recursively
//            through the tail-position answers.
// Every answer is a maximum, so no stage needs a stable order.
constexpr int kBBits = 14;
constexpr int kBSize = 1 << kBBits;          // positions per bucket
constexpr int kBWords = kBSize / 32;
constexpr int kBMaxBuckets = 2048;           // N <= 2^25 on the bucket path
constexpr int kBChunk = 32768;               // steps per sort CTA
constexpr int kBSortThreads = 1024;
constexpr int kBSortPer = kBChunk / kBSortThreads;
constexpr int kBResThreads = 512;
constexpr int kBCap = 8192;                  // entries per resolve pass (several passes if a bucket holds more)
constexpr int kBMaxChunks = (1 << 25) / kBChunk;
constexpr int kOutPerThread = 8;
constexpr int kOutPerBlock = kOutPerThread * kStepThreads;

struct BSortSmem {
    int32_t hist[kBMaxBuckets + 1];
    int32_t warp_tmp[33];
    uint16_t st_s[kBChunk];
    int32_t st_j[kBChunk];
};

constexpr int kBSub = 64;                    // position sub-ranges for sizing multi-pass resolves
constexpr int kBStage = 1024;                // chain-list entries staged per CTA
struct BResSmem {
    uint32_t head2[kBSize / 2];        // list heads, two int16 per word (0xFFFF: empty)
    uint32_t bits[kBWords];
    int32_t ls[kBCap];                 // step of entry e
    int16_t nx[kBCap];                 // list link
    uint16_t lp[kBCap];                // position (in the bucket) of entry e; single pass: first the chunk of entry e
    union {
        struct {
            int32_t segoff[kBMaxChunks + 1];   // entry prefix per sort chunk (+ total)
            int32_t segstart[kBMaxChunks];     // global start of the bucket's segment in each chunk
        } g;
        struct {
            int32_t cs[kBStage], ct[kBStage];  // staged chain entries (step, pred), after the gather
        } c;
    } u;
    int32_t sub[kBSub + 1];            // entries per sub-range, then pass boundaries
    int32_t warp_tmp[33];
    int32_t fill, err, npass, nchain, chain_base;
};

__device__ __forceinline__ int head_get(const BResSmem &sm, int l) {
    return (int)(int16_t)(sm.head2[l >> 1] >> ((l & 1) * 16));
}

// push entry e on position l's list; returns the previous head (-1: empty)
__device__ __forceinline__ int head_push(BResSmem &sm, int l, int e) {
    uint32_t *w = &sm.head2[l >> 1];
    const int sh = (l & 1) * 16;
    uint32_t old = *w, assumed;
    do {
        assumed = old;
        old = atomicCAS(w, assumed, (assumed & ~(0xFFFFu << sh)) | ((uint32_t)(uint16_t)e << sh));
    } while (old != assumed);
    return (int)(int16_t)(old >> sh);
}

// CTA -> plan: the host table gives the plan holding CTA (64 g) for every group
// g of 64 CTAs; a short forward scan skips the plans that start inside the
// group (zero-width ranges of the other path included).
constexpr int kLutShift = 6;
struct PlanLut {
    const int32_t *sort, *bucket, *chain;
};

__device__ __forceinline__ int64_t plan_off(const PlanDev &P, int which) {
    return which == 0 ? P.chunk0 : which == 1 ? P.bucket0 : P.oblock0;
}

__device__ __forceinline__ int find_plan_by(const PlanDev *plans, int n, const int32_t *lut, int64_t blk,
                                            int which) {
    int p = lut[blk >> kLutShift];
    while (p + 1 < n && plan_off(plans[p + 1], which) <= blk) ++p;
    return p;
}

// in-place exclusive scan of a[0..n) in shared memory by the whole block; returns the total
__device__ int32_t block_exclusive_scan(int32_t *a, int n, int32_t *warp_tmp) {
    const int T = blockDim.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int per = (n + T - 1) / T;
    const int i0 = min(n, threadIdx.x * per), i1 = min(n, i0 + per);
    int32_t sum = 0;
    for (int i = i0; i < i1; ++i) sum += a[i];
    int32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) warp_tmp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const int nw = T / 32;
        int32_t v = lane < nw ? warp_tmp[lane] : 0, x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane < nw) warp_tmp[lane] = x - v;
        if (lane == 31) warp_tmp[32] = x;   // the total
    }
    __syncthreads();
    int32_t run = warp_tmp[warp] + inc - sum;
    const int32_t total = warp_tmp[32];
    for (int i = i0; i < i1; ++i) {
        const int32_t v = a[i];
        a[i] = run;
        run += v;
    }
    __syncthreads();
    return total;
}

__device__ __forceinline__ void k_bucket_sort_body(const PlanDev *plans, int n_plans, PlanLut lut, int64_t vb) {
    extern __shared__ __align__(16) unsigned char bsm_raw[];
    BSortSmem &sm = *reinterpret_cast<BSortSmem *>(bsm_raw);
    const PlanDev P = plans[find_plan_by(plans, n_plans, lut.sort, vb, 0)];
    const int c = (int)(vb - P.chunk0);
    const int nb = P.nb;
    const int64_t c0 = (int64_t)c * kBChunk;
    const int len = (int)min((int64_t)kBChunk, P.count - c0);
    for (int b = threadIdx.x; b <= nb; b += kBSortThreads) sm.hist[b] = 0;
    __syncthreads();
    int32_t j[kBSortPer];
    // all of the thread's loads in flight before the first shared-memory atomic
#pragma unroll
    for (int k = 0; k < kBSortPer; ++k) {
        const int i = threadIdx.x + k * kBSortThreads;
        j[k] = i < len ? __ldcs(P.rv + c0 + i) : -1;
    }
#pragma unroll
    for (int k = 0; k < kBSortPer; ++k)
        if (j[k] >= 0) atomicAdd(&sm.hist[j[k] >> kBBits], 1);
    __syncthreads();
    block_exclusive_scan(sm.hist, nb + 1, sm.warp_tmp);
    int32_t *seg = P.segoff + (int64_t)c * (nb + 1);
    for (int b = threadIdx.x; b <= nb; b += kBSortThreads) seg[b] = sm.hist[b];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kBSortPer; ++k) {
        if (j[k] < 0) continue;
        const int slot = atomicAdd(&sm.hist[j[k] >> kBBits], 1);
        sm.st_s[slot] = (uint16_t)(threadIdx.x + k * kBSortThreads);
        sm.st_j[slot] = j[k];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < len; i += kBSortThreads) {
        P.lst_s[c0 + i] = (int32_t)(c0 + sm.st_s[i]);
        P.lst_j[c0 + i] = sm.st_j[i];
    }
}

__global__ void __launch_bounds__(kBSortThreads) k_bucket_sort(const PlanDev *plans, int n_plans, PlanLut lut, int64_t nvb) {
    // grid-stride over the virtual CTAs: the launch may be capped to a share of the SMs
    for (int64_t vb = blockIdx.x; vb < nvb; vb += gridDim.x) {
        k_bucket_sort_body(plans, n_plans, lut, vb);
        __syncthreads();
    }
}

__device__ __forceinline__ void k_bucket_resolve_body(const PlanDev *plans, int n_plans,
                                                                    PlanLut lut, int32_t *status, int64_t vb) {
    extern __shared__ __align__(16) unsigned char brm_raw[];
    BResSmem &sm = *reinterpret_cast<BResSmem *>(brm_raw);
    const int pi = find_plan_by(plans, n_plans, lut.bucket, vb, 1);
    const PlanDev P = plans[pi];
    const int b = (int)(vb - P.bucket0);
    const int nb = P.nb, nch = P.nch;
    const int64_t N = P.n_elems, count = P.count, z0 = N - count;
    const int64_t pbase = (int64_t)b << kBBits;
    const int64_t lim0 = N - 1 - pbase;   // position pbase + l is the i of step lim0 - l
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int32_t *segoff = sm.u.g.segoff, *segstart = sm.u.g.segstart;
    for (int c = tid; c < nch; c += kBResThreads) {
        const int32_t *row = P.segoff + (int64_t)c * (nb + 1);
        const int32_t r0 = row[b];
        segstart[c] = c * kBChunk + r0;
        segoff[c] = row[b + 1] - r0;
    }
    for (int i = tid; i < kBWords; i += kBResThreads) sm.bits[i] = 0u;
    for (int i = tid; i < kBSize / 2; i += kBResThreads) sm.head2[i] = 0xFFFFFFFFu;
    for (int i = tid; i <= kBSub; i += kBResThreads) sm.sub[i] = 0;
    if (tid == 0) { sm.err = 0; sm.npass = 1; sm.nchain = 0; }
    __syncthreads();
    const int32_t n = block_exclusive_scan(segoff, nch, sm.warp_tmp);
    if (tid == 0) segoff[nch] = n;
    // entry k of the bucket lives in chunk c (last segoff <= k), at segstart[c] + k - segoff[c]
    auto chunk_of = [&](int32_t k) -> int {
        int lo = 0, hi = nch - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (segoff[mid] <= k) lo = mid; else hi = mid - 1;
        }
        return lo;
    };
    const bool multi = n > kBCap;
    __syncthreads();
    if (multi) {
        // size the passes from a 64-bin position histogram (a 128-position bin holds at most
        // ~21 entries per position, far below kBCap), greedily filling each pass to kBCap
        for (int32_t k = tid; k < n; k += kBResThreads) {
            const int c = chunk_of(k);
            atomicAdd(&sm.sub[(P.lst_j[segstart[c] + k - segoff[c]] & (kBSize - 1)) / (kBSize / kBSub)], 1);
        }
        __syncthreads();
        if (tid == 0) {
            int np = 0, acc = 0;
            int bounds[kBSub + 1];
            bounds[0] = 0;
            for (int i = 0; i < kBSub; ++i) {
                if (acc + sm.sub[i] > kBCap && acc > 0) { bounds[++np] = i; acc = 0; }
                acc += sm.sub[i];
            }
            bounds[++np] = kBSub;
            for (int i = 0; i <= np; ++i) sm.sub[i] = bounds[i] * (kBSize / kBSub);
            sm.npass = np;
        }
    } else {
        // single pass: expand the segments into a per-entry chunk table (lp doubles as it)
        for (int c = warp; c < nch; c += kBResThreads / 32)
            for (int32_t k = segoff[c] + lane; k < segoff[c + 1]; k += 32) sm.lp[k] = (uint16_t)c;
        if (tid == 0) { sm.sub[0] = 0; sm.sub[1] = kBSize; }
    }
    __syncthreads();
    const int npass = sm.npass;
    for (int ps = 0; ps < npass; ++ps) {
        const int plo = sm.sub[ps], phi = sm.sub[ps + 1];
        if (ps > 0) {   // pass 0's heads were cleared with the rest of the state
            for (int i = plo / 2 + tid; i < phi / 2; i += kBResThreads) sm.head2[i] = 0xFFFFFFFFu;
        }
        if (tid == 0) sm.fill = 0;
        __syncthreads();
        if (!multi) {
            // single pass: every entry is this pass's.  The global loads of a batch of
            // entries are issued together before their list pushes (a shared-memory CAS
            // loop would otherwise serialise one global round trip per entry)
            constexpr int kB = 8;
            for (int32_t k0 = tid; k0 < n; k0 += kB * kBResThreads) {
                int32_t jj[kB], ss[kB];
#pragma unroll
                for (int u = 0; u < kB; ++u) {
                    const int32_t k = k0 + u * kBResThreads;
                    if (k < n) {
                        const int c = sm.lp[k];
                        const int32_t g = segstart[c] + (k - segoff[c]);
                        jj[u] = __ldcs(P.lst_j + g);
                        ss[u] = __ldcs(P.lst_s + g);
                    }
                }
#pragma unroll
                for (int u = 0; u < kB; ++u) {
                    const int32_t k = k0 + u * kBResThreads;
                    if (k < n) {
                        const int l = jj[u] & (kBSize - 1);
                        sm.ls[k] = ss[u];
                        sm.lp[k] = (uint16_t)l;   // entry k's chunk, read above by this same thread
                        sm.nx[k] = (int16_t)head_push(sm, l, k);
                    }
                }
            }
        }
        for (int32_t k = tid; multi && k < n; k += kBResThreads) {
            const int c = multi ? chunk_of(k) : sm.lp[k];
            const int32_t g = segstart[c] + (k - segoff[c]);
            const int32_t jj = P.lst_j[g], ss = P.lst_s[g];
            const int l = jj & (kBSize - 1);
            const bool mine = l >= plo && l < phi;
            int e = k;
            if (multi) {
                const unsigned act = __activemask();
                const unsigned want = __ballot_sync(act, mine);
                const int leader = __ffs(act) - 1;
                int base = 0;
                if (lane == leader) base = atomicAdd(&sm.fill, __popc(want));
                base = __shfl_sync(act, base, leader);
                e = base + __popc(want & ((1u << lane) - 1u));
            }
            if (!mine) continue;
            if (e >= kBCap) { sm.err = 1; continue; }
            sm.ls[e] = ss;
            sm.lp[e] = (uint16_t)l;
            sm.nx[e] = (int16_t)head_push(sm, l, e);
        }
        __syncthreads();
        const int fill = multi ? min(sm.fill, kBCap) : n;
        for (int e = tid; e < fill; e += kBResThreads) {
            const int32_t s = sm.ls[e];
            const int l = sm.lp[e];
            int32_t best = -1;
            for (int x = head_get(sm, l); x >= 0; x = sm.nx[x]) {
                const int32_t t = sm.ls[x];
                if (t < s && t > best) best = t;
            }
            if (best < 0) {
                // nothing wrote the target before step s: the step outputs it
                atomicOr(&sm.bits[l >> 5], 1u << (l & 31));
                if (P.full_idx || s == count - 1) P.idx[count - 1 - s] = (int32_t)(pbase + l);
            } else {
                // chain-list entry: staged in shared memory (the segment tables are dead in a single pass)
                int i = kBStage;
                if (!multi) {
                    const unsigned mask = __activemask();
                    const int leader = __ffs(mask) - 1;
                    int base = 0;
                    if (lane == leader) base = atomicAdd(&sm.nchain, __popc(mask));
                    i = __shfl_sync(mask, base, leader) + __popc(mask & ((1u << lane) - 1u));
                }
                if (i < kBStage) {
                    sm.u.c.cs[i] = s;
                    sm.u.c.ct[i] = best;
                } else {
                    const int32_t slot = atomicAdd(P.nchain, 1);
                    P.rv[slot] = s;      // rv is free once the sort has read it
                    P.pred[slot] = best;
                }
            }
        }
        __syncthreads();
        if (!multi) {
            const int staged = min(sm.nchain, kBStage);
            if (tid == 0) sm.chain_base = staged ? atomicAdd(P.nchain, staged) : 0;
            __syncthreads();
            for (int i = tid; i < staged; i += kBResThreads) {
                P.rv[sm.chain_base + i] = sm.u.c.cs[i];
                P.pred[sm.chain_base + i] = sm.u.c.ct[i];
            }
        }
        // tail positions of this range: the latest step before the position's own step that wrote it
        const int64_t q0 = max(pbase + plo, z0), q1 = min(pbase + phi, N);
        for (int64_t pos = q0 + tid; pos < q1; pos += kBResThreads) {
            const int l = (int)(pos - pbase);
            const int32_t lim = (int32_t)(lim0 - l);
            int32_t best = -1;
            for (int x = head_get(sm, l); x >= 0; x = sm.nx[x]) {
                const int32_t t = sm.ls[x];
                if (t < lim && t > best) best = t;
            }
            P.wtail[pos - z0] = best;
        }
        __syncthreads();
    }
    if (P.bitmap) {
        const int64_t w0 = (int64_t)b * kBWords;
        const int nw = (int)min((int64_t)kBWords, (N + 31) / 32 - w0);
        for (int i = tid; i < nw; i += kBResThreads) P.bitmap[w0 + i] = sm.bits[i];
    }
    if (tid == 0 && sm.err) atomicOr(status + pi, EDGC_ECAPACITY);
}

__global__ void __launch_bounds__(kBResThreads, 2) k_bucket_resolve(const PlanDev *plans, int n_plans,
                                                                    PlanLut lut, int32_t *status, int64_t nvb) {
    // grid-stride over the virtual CTAs: the launch may be capped to a share of the SMs
    for (int64_t vb = blockIdx.x; vb < nvb; vb += gridDim.x) {
        k_bucket_resolve_body(plans, n_plans, lut, status, vb);
        __syncthreads();
    }
}

__device__ __forceinline__ void k_bucket_chain_body(const PlanDev *plans, int n_plans, PlanLut lut, int64_t vb) {
    const PlanDev P = plans[find_plan_by(plans, n_plans, lut.chain, vb, 2)];
    const int64_t N = P.n_elems, count = P.count, z0 = N - count;
    const int64_t e_base = (int64_t)(vb - P.oblock0) * kOutPerBlock + threadIdx.x;
    const int64_t nch = *P.nchain;
    for (int k = 0; k < kOutPerThread; ++k) {
        const int64_t e = e_base + (int64_t)k * kStepThreads;
        if (e >= nch) break;
        const int32_t s = P.rv[e];
        int32_t t = P.pred[e], outv = 0;
        while (true) {
            const int32_t pos = (int32_t)(N - 1 - t);
            const int32_t t2 = P.wtail[pos - z0];
            if (t2 < 0) { outv = pos; break; }
            t = t2;
        }
        if (P.full_idx || s == count - 1) P.idx[count - 1 - s] = outv;
        if (P.bitmap) atomicOr(P.bitmap + (outv >> 5), 1u << (outv & 31));
    }
}

__global__ void __launch_bounds__(kStepThreads) k_bucket_chain(const PlanDev *plans, int n_plans, PlanLut lut, int64_t nvb) {
    // grid-stride over the virtual CTAs: the launch may be capped to a share of the SMs
    for (int64_t vb = blockIdx.x; vb < nvb; vb += gridDim.x) {
        k_bucket_chain_body(plans, n_plans, lut, vb);
        __syncthreads();
    }
}

// ---- set mode: membership bits only (EDGC_PLAN_BITMAP_ONLY tail-shuffle plans) --
// The Gaussian estimator needs the SET of sampled positions, not NumPy's order,
// and the set of a partial Fisher-Yates has an order-free description.  With
// step s finalising position i_s = N-1-s, target j_s = rv[s] <= i_s, z0 = N-count:
//   M(p)     = latest step (largest s) with j_s = p and j_s != i_s; D(p) = M(p) exists
//   last(s)  = M(j_s) == s  (no later step hits j_s again)
//   good(s)  = j_s != i_s && last(s) && (j_s < z0 || good(N-1-j_s))
// Position p < z0 is sampled iff D(p) (its value leaves for the tail the first
// time it is hit); a tail position q >= z0 iff D(q) or !good(N-1-q): the value q
// ends outside the tail only if it is carried down to a non-tail position along
// a path of "last writer" links, and then no earlier step hit q.  (Derivation in
// DESIGN.md §4; every rule is emulated against NumPy in tests/test_plan_logic.py.)
// Kernels: k_set_sort packs each 32K-step chunk by 32K-position bucket (4 B per
// step); k_set_resolve computes M in shared memory per bucket, stores the bucket's
// D bits whole and marks !last steps; k_set_tail finishes the tail positions.
// No chain lists, no per-position tables in HBM.
#ifndef EDGC_SET_BITS
#define EDGC_SET_BITS 14
#endif
constexpr int kSBits = EDGC_SET_BITS;
constexpr int kSSize = 1 << kSBits;          // positions per set-mode bucket (M: 64 KB of shared memory)
constexpr int kSWords = kSSize / 32;
constexpr int kSChunk = 32768;               // steps per sort CTA (15-bit step-in-chunk)
constexpr int kSMaxLog2N = 26;               // N <= 2^26 (GPT2-12.1B's largest, 51.4M, included)
constexpr int kSMaxBuckets = (1 << kSMaxLog2N) / kSSize;
constexpr int kSMaxChunks = (1 << kSMaxLog2N) / kSChunk;
constexpr int kSSortThreads = 1024;
constexpr int kSSortPer = kSChunk / kSSortThreads;
// measured (plan_prof, GPT2-2.5B): 16K-position buckets, 512 threads, 3 CTAs/SM 2.78 ms;
// 8K buckets, 256 threads, 6/SM 2.88 ms; 16K, 256 threads 3.30 ms
constexpr int kSResThreads = (1 << kSBits) <= 8192 ? 256 : 512;
constexpr int kSResPerSM = (1 << kSBits) <= 8192 ? 6 : 3;
#ifndef EDGC_SRES_BATCH
#define EDGC_SRES_BATCH 4
#endif
#ifndef EDGC_STAIL_WORDS
#define EDGC_STAIL_WORDS 4
#endif
constexpr int kSResBatch = EDGC_SRES_BATCH;  // segments whose loads a warp keeps in flight
constexpr int kSTailThreads = 256;           // a warp per bitmap word
constexpr int kSTailWords = EDGC_STAIL_WORDS;  // words per warp (independent loads in flight)
static_assert(kSChunk == kBChunk, "both bucket paths share the chunk tables");

struct SSortSmem {
    int32_t hist[kSMaxBuckets + 1];
    int32_t warp_tmp[33];
    uint32_t st[kSChunk];
};

__device__ __forceinline__ void k_set_sort_body(const PlanDev *plans, int n_plans, PlanLut lut, int64_t vb) {
    extern __shared__ __align__(16) unsigned char ssm_raw[];
    SSortSmem &sm = *reinterpret_cast<SSortSmem *>(ssm_raw);
    const PlanDev P = plans[find_plan_by(plans, n_plans, lut.sort, vb, 0)];
    const int c = (int)(vb - P.chunk0);
    const int nb = P.nb;
    const int64_t c0 = (int64_t)c * kSChunk;
    const int len = (int)min((int64_t)kSChunk, P.count - c0);
    for (int b = threadIdx.x; b <= nb; b += kSSortThreads) sm.hist[b] = 0;
    __syncthreads();
    int32_t j[kSSortPer];
#pragma unroll
    for (int k = 0; k < kSSortPer; ++k) {
        const int i = threadIdx.x + k * kSSortThreads;
        j[k] = i < len ? P.rv[c0 + i] : -1;
    }
#pragma unroll
    for (int k = 0; k < kSSortPer; ++k)
        if (j[k] >= 0) atomicAdd(&sm.hist[j[k] >> kSBits], 1);
    __syncthreads();
    block_exclusive_scan(sm.hist, nb + 1, sm.warp_tmp);
    int32_t *seg = P.segoff + (int64_t)c * (nb + 1);
    for (int b = threadIdx.x; b <= nb; b += kSSortThreads) seg[b] = sm.hist[b];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kSSortPer; ++k) {
        if (j[k] < 0) continue;
        const int slot = atomicAdd(&sm.hist[j[k] >> kSBits], 1);
        sm.st[slot] = ((uint32_t)(threadIdx.x + k * kSSortThreads) << kSBits) | ((uint32_t)j[k] & (kSSize - 1));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < len; i += kSSortThreads) P.lst_pk[c0 + i] = sm.st[i];
    // one sampled element for the Gaussian shift: step 0's output is its own target
    if (c == 0 && threadIdx.x == 0) P.idx[0] = j[0];
}

__global__ void __launch_bounds__(kSSortThreads) k_set_sort(const PlanDev *plans, int n_plans, PlanLut lut,
                                                            int64_t nvb) {
    for (int64_t vb = blockIdx.x; vb < nvb; vb += gridDim.x) {
        k_set_sort_body(plans, n_plans, lut, vb);
        __syncthreads();
    }
}

// dynamic shared memory: M, the bucket's D bits, then the per-chunk segment tables sized by
// the call's largest chunk count (3 CTAs per SM at GPT2-2.5B sizes, 2 at the largest N)
struct SResSmem {
    int32_t M[kSSize];
    uint32_t bits[kSWords];            // D bits of the bucket
    int32_t tab[1];                    // segoff[max_nch + 1] (segment lengths, then their prefix), segstart[max_nch]
};

inline size_t set_resolve_smem(int max_nch) {
    return offsetof(SResSmem, tab) + sizeof(int32_t) * (2 * (size_t)max_nch + 1);
}

__device__ __forceinline__ void k_set_resolve_body(const PlanDev *plans, int n_plans, PlanLut lut, int64_t vb) {
    extern __shared__ __align__(16) unsigned char srm_raw[];
    SResSmem &sm = *reinterpret_cast<SResSmem *>(srm_raw);
    const PlanDev &P = plans[find_plan_by(plans, n_plans, lut.bucket, vb, 1)];
    const int b = (int)(vb - P.bucket0);
    const int nb = P.nb, nch = P.nch;
    const int64_t N = P.n_elems;
    const int64_t pbase = (int64_t)b << kSBits;
    const int32_t ibase = (int32_t)(N - 1 - pbase);   // step s finalises position pbase + l iff s == ibase - l
    uint32_t *notlast = P.notlast;
    int32_t *segoff = sm.tab, *segstart = sm.tab + nch + 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int c = tid; c < nch; c += kSResThreads) {
        const int32_t *row = P.segoff + (int64_t)c * (nb + 1);
        const int32_t r0 = row[b];
        segstart[c] = c * kSChunk + r0;
        segoff[c] = row[b + 1] - r0;
    }
    for (int l = tid; l < kSSize / 4; l += kSResThreads) reinterpret_cast<int4 *>(sm.M)[l] = make_int4(-1, -1, -1, -1);
    for (int w = tid; w < kSWords; w += kSResThreads) sm.bits[w] = 0u;
    __syncthreads();
    // One pass over the bucket's entries (a warp per sort-chunk segment, kSResBatch segments'
    // loads in flight).  old = atomicMax(M[l], s) settles "last" without a second pass: if
    // old > s a later step hits l, so s is not last; otherwise s displaces old, which is not
    // last -- every step but the final maximum is marked exactly once, in any arrival order.
    // D(l) is set by the first arrival.  Self-swaps (s finalises l itself) take no part.
    for (int c0 = warp * kSResBatch; c0 < nch; c0 += (kSResThreads / 32) * kSResBatch) {
        int32_t len[kSResBatch];
        int32_t mx = 0;
#pragma unroll
        for (int u = 0; u < kSResBatch; ++u) {
            len[u] = c0 + u < nch ? segoff[c0 + u] : 0;
            mx = max(mx, len[u]);
        }
        for (int32_t k0 = 0; k0 < mx; k0 += 32) {
            uint32_t e[kSResBatch];
#pragma unroll
            for (int u = 0; u < kSResBatch; ++u)
                if (k0 + lane < len[u]) e[u] = __ldg(P.lst_pk + segstart[c0 + u] + k0 + lane);
#pragma unroll
            for (int u = 0; u < kSResBatch; ++u) {
                if (k0 + lane >= len[u]) continue;
                const int32_t st = (c0 + u) * kSChunk + (int32_t)(e[u] >> kSBits);
                const int l = (int)(e[u] & (kSSize - 1));
                if (st == ibase - l) continue;
                const int32_t old = atomicMax(&sm.M[l], st);
                if (old > st) {
                    atomicOr(notlast + (st >> 5), 1u << (st & 31));
                } else if (old >= 0) {
                    atomicOr(notlast + (old >> 5), 1u << (old & 31));
                } else {
                    atomicOr(&sm.bits[l >> 5], 1u << (l & 31));
                }
            }
        }
    }
    __syncthreads();
    const int64_t w0 = (int64_t)b * kSWords;
    const int64_t nw = (N + 31) / 32;
    for (int w = tid; w < kSWords; w += kSResThreads)
        if (w0 + w < nw) P.bitmap[w0 + w] = sm.bits[w];
}

__global__ void __launch_bounds__(kSResThreads, kSResPerSM) k_set_resolve(const PlanDev *plans, int n_plans, PlanLut lut,
                                                                 int64_t nvb) {
    for (int64_t vb = blockIdx.x; vb < nvb; vb += gridDim.x) {
        k_set_resolve_body(plans, n_plans, lut, vb);
        __syncthreads();
    }
}

// tail positions q >= z0 not hit by an earlier step: sampled iff !good(N-1-q).
// A warp finishes kSTailWords bitmap words: every position's first link (D word,
// rv, !last bit) is loaded up front, the second links of all positions that need
// one (~1 in 8: the value came from another tail position) are loaded together,
// and the rare deeper chains are followed one by one.
__device__ __forceinline__ bool set_chain_good(const int32_t *rv, const uint32_t *notlast, int32_t n1, int32_t z0,
                                               int32_t st) {
    while (true) {
        const int32_t j = rv[st];
        if (j == n1 - st) return false;                         // self-swap: the value stays
        if ((notlast[st >> 5] >> (st & 31)) & 1u) return false; // taken back into the tail later
        if (j < z0) return true;                                // carried down below the tail
        st = n1 - j;
    }
}

__device__ __forceinline__ void k_set_tail_body(const PlanDev &P, int64_t vb) {
    // 32-bit index arithmetic: N < 2^31 on this path
    const int32_t N = (int32_t)P.n_elems, n1 = N - 1, z0 = (int32_t)(P.n_elems - P.count);
    const int32_t *rv = P.rv;
    const uint32_t *notlast = P.notlast;
    uint32_t *bitmap = P.bitmap;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int32_t w_first = (z0 >> 5) + ((int32_t)(vb - P.oblock0) * (kSTailThreads / 32) + warp) * kSTailWords;
    const int32_t nw = (int32_t)((P.n_elems + 31) >> 5);
    uint32_t word[kSTailWords], nl[kSTailWords];
    int32_t j[kSTailWords];
#pragma unroll
    for (int u = 0; u < kSTailWords; ++u) {
        const int32_t w = w_first + u, q = (w << 5) + lane;
        const bool in = w < nw && q >= z0 && q < N;
        word[u] = w < nw ? bitmap[w] : 0u;
        const int32_t st = in ? n1 - q : 0;
        j[u] = in ? rv[st] : -1;
        nl[u] = in ? notlast[st >> 5] >> (st & 31) : 0u;
    }
    // state: 1 sampled, 0 not, 2 follow the value to the tail position j came from
    int state[kSTailWords];
    int32_t st2[kSTailWords];
#pragma unroll
    for (int u = 0; u < kSTailWords; ++u) {
        const int32_t st = n1 - ((w_first + u) << 5) - lane;
        state[u] = 0;
        if (j[u] >= 0 && !((word[u] >> lane) & 1u))
            state[u] = (j[u] == n1 - st || (nl[u] & 1u)) ? 1 : (j[u] >= z0 ? 2 : 0);
        st2[u] = n1 - j[u];
    }
#pragma unroll
    for (int u = 0; u < kSTailWords; ++u) {   // second links of every position that needs one, together
        if (state[u] != 2) continue;
        j[u] = rv[st2[u]];
        nl[u] = notlast[st2[u] >> 5] >> (st2[u] & 31);
    }
#pragma unroll
    for (int u = 0; u < kSTailWords; ++u) {
        if (state[u] != 2) continue;
        if (j[u] == n1 - st2[u] || (nl[u] & 1u)) state[u] = 1;
        else if (j[u] < z0) state[u] = 0;
        else state[u] = set_chain_good(rv, notlast, n1, z0, n1 - j[u]) ? 0 : 1;
    }
#pragma unroll
    for (int u = 0; u < kSTailWords; ++u) {
        const unsigned bits = __ballot_sync(0xffffffffu, state[u] == 1);
        if (lane == 0 && bits) bitmap[w_first + u] = word[u] | bits;
    }
}

__global__ void __launch_bounds__(kSTailThreads) k_set_tail(const PlanDev *plans, int n_plans, PlanLut lut,
                                                            int64_t nvb) {
    __shared__ int pi;
    for (int64_t vb = blockIdx.x; vb < nvb; vb += gridDim.x) {
        if (threadIdx.x == 0) pi = find_plan_by(plans, n_plans, lut.chain, vb, 2);
        __syncthreads();
        k_set_tail_body(plans[pi], vb);
        __syncthreads();
    }
}

struct PlanLayout {
    std::vector<PlanDev> dev;
    int64_t ws_bytes = 0;
    int64_t step_blocks = 0;
    int64_t bchunks = 0, buckets = 0, oblocks = 0;   // bucket path (plans with bucketed = 1)
    int32_t *nchains = nullptr;                       // all bucket plans' chain counters (zeroed per call)
    std::vector<int32_t> lut_host;                    // [sort | bucket | chain] CTA-group -> plan tables
    int64_t lut_n[3] = {0, 0, 0};
    int32_t *lut_dev = nullptr;
    int32_t *walk_order = nullptr;            // k_walk: plans by decreasing step count
    std::vector<int32_t> walk_order_host;
    int n_bucketed = 0;
    int setmode = 0;                                  // bucketed plans take the set-only path (k_set_*)
    uint32_t *notlast = nullptr;                      // all set-mode plans' !last bits (zeroed per call)
    int64_t notlast_words = 0;
    int64_t table_bytes = 0;
    char *table_base = nullptr;
    std::vector<int64_t> table_off;   // head-table plans, relative to table_base (contiguous)
};

int layout_plans(const edgc_plan_desc *plans, int n, void *ws, int64_t ws_bytes, PlanLayout &L) {
    Arena a(ws, ws_bytes);
    L.dev.resize(n);
    PlanDev *descs_dev = a.take<PlanDev>(n);
    (void)descs_dev;
    int64_t blocks = 0;
    static const bool no_bucket = std::getenv("EDGC_PLAN_HEADTABLE") != nullptr;
    // set mode when every plan of the call is bitmap-only (the tracker's plans): the order-free resolve
    static const bool no_set = std::getenv("EDGC_PLAN_NOSET") != nullptr;
    bool call_set = !no_set;
    for (int i = 0; i < n; ++i)
        if (!(plans[i].flags & EDGC_PLAN_BITMAP_ONLY) || plans[i].bitmap == nullptr) call_set = false;
    for (int i = 0; i < n; ++i) {
        const edgc_plan_desc &d = plans[i];
        EDGC_REQUIRE(d.n_elems >= 2 && d.n_elems < (int64_t(1) << 31), "plan %d: N=%lld outside [2, 2^31)", i,
                     (long long)d.n_elems);
        EDGC_REQUIRE(d.count >= 1 && d.count < d.n_elems, "plan %d: count=%lld must be in [1, N)", i,
                     (long long)d.count);
        PlanDev &P = L.dev[i];
        P = PlanDev{};
        P.state = (((u128)d.state_hi) << 64) | d.state_lo;
        P.inc = (((u128)d.inc_hi) << 64) | d.inc_lo;
        P.n_elems = d.n_elems;
        P.count = d.count;
        P.idx = d.idx;
        P.bitmap = d.bitmap;
        P.full_idx = (d.flags & EDGC_PLAN_BITMAP_ONLY) ? 0 : 1;
        P.tail = (d.n_elems > 10000 && d.count > d.n_elems / 20) ? 1 : 0;
        // bucket paths: the list resolve up to 2^25 positions, the set resolve (a call whose plans
        // are all bitmap-only) up to 2^26
        const int64_t bmax = call_set ? (int64_t(1) << kSMaxLog2N) : (int64_t)kBMaxBuckets * kBSize;
        P.bucketed = (!no_bucket && P.tail && d.n_elems <= bmax) ? 1 : 0;
        P.step_block0 = blocks;
        blocks += ceil_div(d.count, kStepThreads);
    }
    L.step_blocks = blocks;
    bool any_b = false;
    for (int i = 0; i < n; ++i) any_b |= L.dev[i].bucketed != 0;
    L.setmode = (call_set && any_b) ? 1 : 0;
    if (L.setmode) {
        int64_t words = 0;
        for (int i = 0; i < n; ++i)
            if (L.dev[i].bucketed) words += align256(4 * ceil_div(L.dev[i].count, 32)) / 4;
        L.notlast = a.take<uint32_t>(words);
        L.notlast_words = words;
        int64_t wo = 0;
        for (int i = 0; i < n; ++i) {
            PlanDev &P = L.dev[i];
            if (!P.bucketed) continue;
            P.setmode = 1;
            P.notlast = L.notlast ? L.notlast + wo : nullptr;
            wo += align256(4 * ceil_div(P.count, 32)) / 4;
        }
    }
    for (int i = 0; i < n; ++i) {
        PlanDev &P = L.dev[i];
        P.rv = a.take<int32_t>(P.count);
        if (P.setmode) {
            P.nb = (int32_t)ceil_div(P.n_elems, kSSize);
            P.nch = (int32_t)ceil_div(P.count, kSChunk);
            P.lst_pk = a.take<uint32_t>(P.count);
            P.segoff = a.take<int32_t>((int64_t)P.nch * (P.nb + 1));
            P.chunk0 = L.bchunks;
            L.bchunks += P.nch;
            P.bucket0 = L.buckets;
            L.buckets += P.nb;
            P.oblock0 = L.oblocks;
            const int64_t z0 = P.n_elems - P.count;
            L.oblocks += ceil_div(ceil_div(P.n_elems, 32) - (z0 >> 5), (int64_t)(kSTailThreads / 32) * kSTailWords);
            ++L.n_bucketed;
            continue;
        }
        if (!P.bucketed) {
            // zero-width ranges at the running offsets keep the CTA -> plan searches monotone
            P.chunk0 = L.bchunks;
            P.bucket0 = L.buckets;
            P.oblock0 = L.oblocks;
            P.next = a.take<int32_t>(P.count);
            continue;
        }
        P.nb = (int32_t)ceil_div(P.n_elems, kBSize);
        P.nch = (int32_t)ceil_div(P.count, kBChunk);
        P.lst_s = a.take<int32_t>(P.count);
        P.lst_j = a.take<int32_t>(P.count);
        P.segoff = a.take<int32_t>((int64_t)P.nch * (P.nb + 1));
        P.pred = a.take<int32_t>(P.count);
        P.wtail = a.take<int32_t>(P.count);
        P.chunk0 = L.bchunks;
        L.bchunks += P.nch;
        P.bucket0 = L.buckets;
        L.buckets += P.nb;
        P.oblock0 = L.oblocks;
        L.oblocks += ceil_div(P.count, kOutPerBlock);
        ++L.n_bucketed;
    }
    // CTA-group -> plan tables (largest plan whose range starts at or before the group's first CTA)
    const int64_t tot[3] = {L.bchunks, L.buckets, L.oblocks};
    L.lut_host.clear();
    for (int w = 0; w < 3; ++w) {
        L.lut_n[w] = (tot[w] >> kLutShift) + 1;
        int p = 0;
        for (int64_t g = 0; g < L.lut_n[w]; ++g) {
            const int64_t blk = g << kLutShift;
            auto off = [&](int q) { return w == 0 ? L.dev[q].chunk0 : w == 1 ? L.dev[q].bucket0 : L.dev[q].oblock0; };
            while (p + 1 < n && off(p + 1) <= blk) ++p;
            L.lut_host.push_back(p);
        }
    }
    a.off = align256(a.off);
    L.lut_dev = reinterpret_cast<int32_t *>(a.base ? a.base + a.off : nullptr);
    a.off += align256(4 * (int64_t)L.lut_host.size());
    L.nchains = reinterpret_cast<int32_t *>(a.base ? a.base + a.off : nullptr);
    for (int i = 0; i < n; ++i)
        if (L.dev[i].bucketed) L.dev[i].nchain = L.nchains + i;
    a.off += align256(4 * (int64_t)n);
    L.walk_order = reinterpret_cast<int32_t *>(a.base ? a.base + a.off : nullptr);
    a.off += align256(4 * (int64_t)n);
    L.walk_order_host.resize(n);
    for (int i = 0; i < n; ++i) L.walk_order_host[i] = i;
    std::stable_sort(L.walk_order_host.begin(), L.walk_order_host.end(),
                     [&](int x, int y) { return L.dev[x].count > L.dev[y].count; });
    const int64_t t0 = a.off;
    L.table_off.assign(n + 1, 0);
    for (int i = 0; i < n; ++i) {
        PlanDev &P = L.dev[i];
        L.table_off[i] = a.off - t0;
        if (P.bucketed) continue;
        P.head = reinterpret_cast<int32_t *>(a.base ? a.base + a.off : nullptr);
        a.off += align256(P.n_elems * 4);
    }
    L.table_off[n] = a.off - t0;
    L.table_bytes = a.off - t0;
    L.table_base = a.base ? a.base + t0 : nullptr;
    L.ws_bytes = a.off;
    return EDGC_OK;
}

__global__ void k_gather(int src_dtype, const void *src, const int32_t *idx, int64_t count, int dst_dtype,
                         void *dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = idx ? (int64_t)idx[i] : i;
        const double v = src_dtype == 0 ? (double)reinterpret_cast<const float *>(src)[k]
                                        : reinterpret_cast<const double *>(src)[k];
        if (dst_dtype == 0)
            reinterpret_cast<float *>(dst)[i] = (float)v;
        else
            reinterpret_cast<double *>(dst)[i] = v;
    }
}

}  // namespace
}  // namespace edgc

using namespace edgc;

extern "C" int64_t edgc_sample_plan_workspace_bytes(const edgc_plan_desc *plans, int n_plans) {
    PlanLayout L;
    if (n_plans < 0) return -1;
    if (layout_plans(plans, n_plans, nullptr, INT64_MAX, L) != EDGC_OK) return -1;
    return L.ws_bytes;
}

extern "C" int edgc_sample_plan(const edgc_plan_desc *plans, int n_plans, int32_t *status_dev, void *ws,
                                int64_t ws_bytes, void *stream) {
    if (n_plans == 0) return EDGC_OK;
    EDGC_REQUIRE(n_plans > 0 && plans && status_dev, "edgc_sample_plan: bad arguments");
    for (int i = 0; i < n_plans; ++i)
        EDGC_REQUIRE(plans[i].idx && (!(plans[i].flags & EDGC_PLAN_BITMAP_ONLY) || plans[i].bitmap),
                     "plan %d: idx is required, and a bitmap with EDGC_PLAN_BITMAP_ONLY", i);
    PlanLayout L;
    int rc = layout_plans(plans, n_plans, ws, ws_bytes, L);
    if (rc != EDGC_OK) return rc;
    EDGC_REQUIRE(L.ws_bytes <= ws_bytes, "edgc_sample_plan: workspace %lld < needed %lld", (long long)ws_bytes,
                 (long long)L.ws_bytes);
    cudaStream_t st = (cudaStream_t)stream;
    PlanDev *d_plans = reinterpret_cast<PlanDev *>(ws);
    EDGC_CUDA_TRY(cudaMemcpyAsync(d_plans, L.dev.data(), sizeof(PlanDev) * n_plans, cudaMemcpyHostToDevice, st));
    // the plan kernels run grid-stride over their virtual CTAs; EDGC_PLAN_SMS caps them to a
    // share of the SMs (measured: capping spreads the interference over more steps and costs
    // more than it saves, so the default is the whole GPU)
    static const int plan_sms = [] {
        const char *e = std::getenv("EDGC_PLAN_SMS");
        const int v = e ? std::atoi(e) : 0;
        return v > 0 ? std::min(v, edgc::sm_count()) : edgc::sm_count();
    }();
    // One short-lived CTA per virtual CTA (not a persistent grid-stride loop), so a higher-
    // priority stream's kernels -- the training step's -- take SMs back as plan CTAs retire
    // (measured with the step on a high-priority stream: 8.96 -> 8.6 ms/step).
    // EDGC_PLAN_PERSISTENT restores the grid-stride launch.
    static const bool plan_short = std::getenv("EDGC_PLAN_PERSISTENT") == nullptr;
    auto capped = [&](int64_t nvb, int per_sm) {
        if (plan_short) return (unsigned)std::max<int64_t>(1, nvb);
        return (unsigned)std::max<int64_t>(1, std::min<int64_t>(nvb, (int64_t)plan_sms * per_sm));
    };
    // every plan's status is OK (the walk generates its own draws; kept for the ABI)
    EDGC_CUDA_TRY(cudaMemsetAsync(status_dev, 0, 4 * (size_t)n_plans, st));
    EDGC_CUDA_TRY(cudaMemcpyAsync(L.walk_order, L.walk_order_host.data(), 4 * (size_t)n_plans,
                                  cudaMemcpyHostToDevice, st));
    static bool walk_attr = false;
    if (!walk_attr) {
        EDGC_CUDA_TRY(cudaFuncSetAttribute(k_walk<kWalkNBlkAhead, 1000>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(kWalkPlans * sizeof(WalkRing<kWalkNBlkAhead>))));
        EDGC_CUDA_TRY(cudaFuncSetAttribute(k_walk<kWalkNBlkLat, 100>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)sizeof(WalkRing<kWalkNBlkLat>)));
        walk_attr = true;
    }
    bool latency = false;
    for (int i = 0; i < n_plans; ++i) latency |= (plans[i].flags & EDGC_PLAN_LATENCY) != 0;
    if (latency)
        k_walk<kWalkNBlkLat, 100><<<(unsigned)n_plans, 64, sizeof(WalkRing<kWalkNBlkLat>), st>>>(
            d_plans, n_plans, (const int32_t *)L.walk_order, 1);
    else
        k_walk<kWalkNBlkAhead, 1000><<<(unsigned)ceil_div(n_plans, kWalkPlans), 64 * kWalkPlans,
                                       kWalkPlans * sizeof(WalkRing<kWalkNBlkAhead>), st>>>(
            d_plans, n_plans, (const int32_t *)L.walk_order, kWalkPlans);
    EDGC_LAUNCH_CHECK();
    if (L.n_bucketed) {
        // bucket path (tail-shuffle plans); plans are ordered, so each kernel's CTA range covers
        // only the bucketed plans' chunks / buckets / chain blocks
        static bool battr = false;
        if (!battr) {
            EDGC_CUDA_TRY(cudaFuncSetAttribute(k_bucket_sort, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)sizeof(BSortSmem)));
            EDGC_CUDA_TRY(cudaFuncSetAttribute(k_bucket_resolve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)sizeof(BResSmem)));
            battr = true;
        }
        EDGC_CUDA_TRY(cudaMemsetAsync(L.nchains, 0, 4 * (size_t)n_plans, st));
        EDGC_CUDA_TRY(cudaMemcpyAsync(L.lut_dev, L.lut_host.data(), 4 * L.lut_host.size(), cudaMemcpyHostToDevice,
                                      st));
        const PlanLut lut{L.lut_dev, L.lut_dev + L.lut_n[0], L.lut_dev + L.lut_n[0] + L.lut_n[1]};
        if (L.setmode) {
            static bool sattr = false;
            if (!sattr) {
                EDGC_CUDA_TRY(cudaFuncSetAttribute(k_set_sort, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)sizeof(SSortSmem)));
                EDGC_CUDA_TRY(cudaFuncSetAttribute(k_set_resolve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)set_resolve_smem(kSMaxChunks)));
                sattr = true;
            }
            EDGC_CUDA_TRY(cudaMemsetAsync(L.notlast, 0, 4 * (size_t)L.notlast_words, st));
            k_set_sort<<<capped(L.bchunks, 1), kSSortThreads, sizeof(SSortSmem), st>>>(d_plans, n_plans, lut,
                                                                                        L.bchunks);
            EDGC_LAUNCH_CHECK();
            int max_nch = 1;
            for (int i = 0; i < n_plans; ++i)
                if (L.dev[i].setmode) max_nch = std::max(max_nch, (int)L.dev[i].nch);
            k_set_resolve<<<capped(L.buckets, kSResPerSM), kSResThreads, set_resolve_smem(max_nch), st>>>(d_plans, n_plans, lut,
                                                                                        L.buckets);
            EDGC_LAUNCH_CHECK();
            k_set_tail<<<capped(L.oblocks, 8), kSTailThreads, 0, st>>>(d_plans, n_plans, lut, L.oblocks);
            EDGC_LAUNCH_CHECK();
        } else {
            k_bucket_sort<<<capped(L.bchunks, 1), kBSortThreads, sizeof(BSortSmem), st>>>(d_plans, n_plans, lut,
                                                                                          L.bchunks);
            EDGC_LAUNCH_CHECK();
            k_bucket_resolve<<<capped(L.buckets, 2), kBResThreads, sizeof(BResSmem), st>>>(
                d_plans, n_plans, lut, status_dev, L.buckets);
            EDGC_LAUNCH_CHECK();
            k_bucket_chain<<<capped(L.oblocks, 8), kStepThreads, 0, st>>>(d_plans, n_plans, lut, L.oblocks);
            EDGC_LAUNCH_CHECK();
        }
    }
    // head-table path (Floyd plans, N > 2^25, or EDGC_PLAN_HEADTABLE): index + resolve groups of
    // consecutive such plans whose tables, links and bounded values fit in L2 together
    const int64_t kGroupBytes = 48ll << 20;
    int p0 = 0;
    while (p0 < n_plans) {
        if (L.dev[p0].bucketed) { ++p0; continue; }
        int p1 = p0 + 1;
        int64_t bytes = (L.table_off[p0 + 1] - L.table_off[p0]) + 8 * L.dev[p0].count;
        while (p1 < n_plans && !L.dev[p1].bucketed) {
            const int64_t more = (L.table_off[p1 + 1] - L.table_off[p1]) + 8 * L.dev[p1].count;
            if (bytes + more > kGroupBytes) break;
            bytes += more;
            ++p1;
        }
        EDGC_CUDA_TRY(cudaMemsetAsync(L.table_base + L.table_off[p0], 0xFF, L.table_off[p1] - L.table_off[p0], st));
        const int64_t blk0 = L.dev[p0].step_block0;
        const int64_t blk1 = (p1 < n_plans) ? L.dev[p1].step_block0 : L.step_blocks;
        k_index<<<(unsigned)(blk1 - blk0), kStepThreads, 0, st>>>(d_plans, p0, p1, blk0);
        EDGC_LAUNCH_CHECK();
        k_resolve<<<(unsigned)(blk1 - blk0), kStepThreads, 0, st>>>(d_plans, p0, p1, blk0);
        EDGC_LAUNCH_CHECK();
        p0 = p1;
    }
    return EDGC_OK;
}

extern "C" int edgc_gather(int src_dtype, const void *src, const int32_t *idx, int64_t count, int dst_dtype,
                           void *dst, void *stream) {
    EDGC_REQUIRE((src_dtype == 0 || src_dtype == 1) && (dst_dtype == 0 || dst_dtype == 1) && count >= 0,
                 "edgc_gather: bad dtype/count");
    if (count == 0) return EDGC_OK;
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>(ceil_div(count, threads), (int64_t)sm_count() * 16);
    k_gather<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(src_dtype, src, idx, count, dst_dtype, dst);
    EDGC_LAUNCH_CHECK();
    return EDGC_OK;
}
