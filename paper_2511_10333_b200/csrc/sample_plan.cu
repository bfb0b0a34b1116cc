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
    uint32_t *draws;   // [n_draws]
    int64_t n_draws;   // even
    int32_t *rv;       // [count] bounded values
    int32_t *next;     // [count]
    int32_t *head;     // [n_elems] latest step targeting each position (-1: none)
    int32_t tail;      // 1 = tail shuffle, 0 = Floyd
    int64_t draw_chunk0;  // first P1 chunk index of this plan
    int64_t step_block0;  // first P3/P4 block index of this plan
};

constexpr int kDrawsPerThread = 64;  // 64-bit outputs per P1 thread
constexpr int kP1Threads = 256;
constexpr int64_t kDrawsPerBlock = (int64_t)kDrawsPerThread * kP1Threads;
constexpr int kWalkThreads = 1024;
constexpr int kStepThreads = 256;

__device__ __forceinline__ int find_plan(const PlanDev *plans, int n, int64_t blk, bool by_draw) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        int64_t b0 = by_draw ? plans[mid].draw_chunk0 : plans[mid].step_block0;
        if (b0 <= blk) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// ---- P1: u32 draw stream ---------------------------------------------------
// Block b of a plan owns 64-bit outputs [b*64*256, (b+1)*64*256); thread t
// produces outputs t, t+256, t+512, ... of that range (one jump-ahead, then a
// 256-step affine LCG map per output), so every warp store is coalesced.
__global__ void __launch_bounds__(kP1Threads) k_draws(const PlanDev *plans, int n_plans) {
    const PlanDev &P = plans[find_plan(plans, n_plans, blockIdx.x, true)];
    const int64_t o_base = (int64_t)(blockIdx.x - P.draw_chunk0) * kDrawsPerBlock;
    const int64_t n64 = P.n_draws / 2;
    if (o_base >= n64) return;
    u128 s = pcg_jump(P.state, P.inc, (uint64_t)(o_base + threadIdx.x));
    u128 a_t, c_t;
    pcg_affine(P.inc, kP1Threads, a_t, c_t);
    uint2 *out = reinterpret_cast<uint2 *>(P.draws);
    const u128 m1 = pcg_mult();
    for (int k = 0; k < kDrawsPerThread; ++k) {
        const int64_t o = o_base + threadIdx.x + (int64_t)k * kP1Threads;
        if (o >= n64) break;
        const uint64_t v = pcg_output(s * m1 + P.inc);   // output o = XSL-RR(state after o+1 steps)
        out[o] = make_uint2((uint32_t)v, (uint32_t)(v >> 32));
        s = a_t * s + c_t;
    }
}

// Lemire 32-bit bounded draw check (NumPy bounded_lemire_uint32).
__device__ __forceinline__ bool lemire_accept(uint32_t x, uint32_t rng, uint32_t &val) {
    const uint32_t excl = rng + 1u;
    const uint64_t m = (uint64_t)x * excl;
    val = (uint32_t)(m >> 32);
    const uint32_t left = (uint32_t)m;
    if (left >= excl) return true;
    const uint32_t thr = (0xFFFFFFFFu - rng) % excl;
    return left >= thr;
}

__device__ __forceinline__ uint32_t step_rng(const PlanDev &P, int64_t s) {
    // tail: i = N-1-s (bounded(0..i)); Floyd: j = N-count+s (bounded(0..j))
    return P.tail ? (uint32_t)(P.n_elems - 1 - s) : (uint32_t)(P.n_elems - P.count + s);
}

// ---- P2: assign draws to steps --------------------------------------------
// One CTA per plan walks windows of kWT steps.  Lane l tests its step against
// the draws at shifts 0..kWK-1 (draw u+l+j): a Lemire rejection at lane f and
// shift d moves every later step one draw further, so the window resolves by
// scanning rejection events in lane order (warp 0, ballots) and accepting each
// lane at shift #events at lanes <= l.  Up to kWK-1 rejections fit in one
// window; rarer bursts end the window early.  The draw window lives in shared
// memory and the next one is prefetched while the current one resolves.
constexpr int kWT = 256;                  // threads per walk CTA
constexpr int kWQ = 4;                    // consecutive steps per thread
constexpr int kWW = kWT * kWQ;            // steps per window
constexpr int kWK = 4;                    // speculative shifts
constexpr int kRingBlk = 1024;            // draws per ring block (4 KB bulk copy)
constexpr int kRingN = 8;                 // blocks in flight
constexpr int kRing = kRingBlk * kRingN;  // ring size (draws), power of two

__global__ void __launch_bounds__(kWT) k_walk(const PlanDev *plans, int32_t *status) {
    const PlanDev &P = plans[blockIdx.x];
    extern __shared__ __align__(128) uint32_t s_ring[];   // kRing draws (dynamic: 32 KB)
    __shared__ uint32_t s_mask[kWK][kWW / 32];
    __shared__ int s_ev[kWK];
    __shared__ int s_ne, s_len, s_err;
    __shared__ __align__(8) uint64_t s_full[kRingN];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t count = P.count, nd = P.n_draws;
    const int64_t nblocks = (nd + kRingBlk - 1) / kRingBlk;
    const uint32_t tail = (uint32_t)P.tail;
    const uint32_t rng_hi = tail ? (uint32_t)(P.n_elems - 1) : (uint32_t)(P.n_elems - P.count);
    int32_t *rv = P.rv;
    const uint32_t *draws = P.draws;
    int64_t next_blk = 0;   // first block not yet requested (thread 0)
    auto request = [&](int64_t upto) {
        while (next_blk < upto && next_blk < nblocks) {
            const int slot = (int)(next_blk % kRingN);
            const int64_t first = next_blk * kRingBlk;
            const uint32_t bytes = (uint32_t)(min((int64_t)kRingBlk, nd - first) * 4);
            ptx::mbar_arrive_expect_tx(&s_full[slot], bytes);
            ptx::bulk_g2s(&s_ring[slot * kRingBlk], draws + first, bytes, &s_full[slot]);
            ++next_blk;
        }
    };
    if (tid == 0) {
        for (int i = 0; i < kRingN; ++i) ptx::mbar_init(&s_full[i], 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        s_err = 0;
    }
    __syncthreads();
    if (tid == 0) request(kRingN);
    int64_t s = 0, u = 0;
    while (s < count) {
        const int64_t b0 = u / kRingBlk;
        for (int64_t bb = b0; bb <= b0 + 1 && bb < nblocks; ++bb)
            ptx::mbar_wait(&s_full[bb % kRingN], (uint32_t)((bb / kRingN) & 1));
        // this thread's steps s + 4 tid + q use draws u + 4 tid + q + j
        const int nvalid = (int)min((int64_t)kWW, count - s);
        const uint32_t ubase = (uint32_t)(u & (kRing - 1)) + 4u * tid;
        const int64_t dleft = nd - u - 4 * tid;   // draws generated from this thread's first one on
        uint32_t d[kWQ + kWK - 1];
#pragma unroll
        for (int e = 0; e < kWQ + kWK - 1; ++e) d[e] = s_ring[(ubase + e) & (kRing - 1)];
        uint32_t val[kWQ][kWK];
        uint32_t nib[kWK] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int q = 0; q < kWQ; ++q) {
            const int step = 4 * tid + q;
            // rng of step s + step: tail i = N-1-(s+step); Floyd j = N-count+(s+step)
            const uint32_t off = (uint32_t)s + (uint32_t)step;
            const uint32_t rng = tail ? rng_hi - off : rng_hi + off;
            const uint32_t excl = rng + 1u;
#pragma unroll
            for (int j = 0; j < kWK; ++j) {
                const uint64_t m = (uint64_t)d[q + j] * excl;
                val[q][j] = (uint32_t)(m >> 32);
                bool rej = false;
                const uint32_t left = (uint32_t)m;
                if (left < excl) rej = left < (0xFFFFFFFFu - rng) % excl;
                if ((int64_t)(q + j) >= dleft) rej = true;   // past the generated stream
                if (step < nvalid && rej) nib[j] |= 1u << q;
            }
        }
        // assemble per-shift 32-bit words: word (8 warp + lane/8) holds steps 32 w .. 32 w + 31
#pragma unroll
        for (int j = 0; j < kWK; ++j) {
            uint32_t wv = nib[j] << (4 * (lane & 7));
            wv |= __shfl_xor_sync(0xffffffffu, wv, 1);
            wv |= __shfl_xor_sync(0xffffffffu, wv, 2);
            wv |= __shfl_xor_sync(0xffffffffu, wv, 4);
            if ((lane & 7) == 0) s_mask[j][warp * 4 + (lane >> 3)] = wv;
        }
        __syncthreads();
        if (warp == 0) {
            int cur = 0, dd = 0, ne = 0, len = nvalid;
            while (true) {
                uint32_t bits = s_mask[dd][lane];
                const int lo = lane * 32;
                if (lo + 32 <= cur) bits = 0u;
                else if (lo < cur) bits &= ~((1u << (cur - lo)) - 1u);
                const unsigned any = __ballot_sync(0xffffffffu, bits != 0u);
                if (!any) break;
                const int wi = __ffs(any) - 1;
                const uint32_t wbits = __shfl_sync(0xffffffffu, bits, wi);
                const int f = wi * 32 + __ffs(wbits) - 1;
                if (lane == 0) s_ev[ne] = f;
                ++ne;
                ++dd;
                if (dd == kWK) { len = f; break; }
                cur = f;
            }
            if (lane == 0) { s_ne = ne; s_len = len; }
        }
        __syncthreads();
        const int ne = s_ne, len = s_len;
        int ev[kWK];
#pragma unroll
        for (int e = 0; e < kWK; ++e) ev[e] = (e < ne) ? s_ev[e] : 0x7fffffff;
        uint32_t out[kWQ];
#pragma unroll
        for (int q = 0; q < kWQ; ++q) {
            const int step = 4 * tid + q;
            int sh = 0;
#pragma unroll
            for (int e = 0; e < kWK; ++e) sh += (ev[e] <= step);
            uint32_t v = val[q][0];
#pragma unroll
            for (int j = 1; j < kWK; ++j) v = (sh == j) ? val[q][j] : v;
            out[q] = v;
        }
        const int first = 4 * tid;
        if (first + kWQ <= len && ((s & 3) == 0)) {
            *reinterpret_cast<int4 *>(rv + s + first) = make_int4(out[0], out[1], out[2], out[3]);
        } else {
#pragma unroll
            for (int q = 0; q < kWQ; ++q)
                if (first + q < len) rv[s + first + q] = (int32_t)out[q];
        }
        if (tid == 0 && u + len + ne > nd) s_err = 1;
        s += len;
        u += len + ne;
        __syncthreads();   // every read of ring blocks below u / kRingBlk is done
        if (tid == 0) request(u / kRingBlk + kRingN);
        if (s_err || (len == 0 && ne == 0)) break;
    }
    if (tid == 0) status[blockIdx.x] = (s_err || s < count) ? EDGC_EDRAWS : EDGC_OK;
}

__device__ __forceinline__ int find_plan_steps(const PlanDev *plans, int n, int64_t blk) {
    return find_plan(plans, n, blk, false);
}

// ---- P3: per-position lists of the steps whose bounded value is that position
// (direct-mapped heads: one atomic exchange per step, no probing)
__global__ void __launch_bounds__(kStepThreads) k_index(const PlanDev *plans, int p0, int p1, int64_t blk0) {
    const int p = p0 + find_plan_steps(plans + p0, p1 - p0, blk0 + blockIdx.x);
    const PlanDev &P = plans[p];
    const int64_t s = (int64_t)(blk0 + blockIdx.x - P.step_block0) * kStepThreads + threadIdx.x;
    if (s >= P.count) return;
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
    const PlanDev &P = plans[p];
    const int64_t s64 = (int64_t)(blk0 + blockIdx.x - P.step_block0) * kStepThreads + threadIdx.x;
    if (s64 >= P.count) return;
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
        P.idx[count - 1 - s] = (int32_t)val;
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
        P.idx[s] = outv;
        if (P.bitmap) atomicOr(P.bitmap + (outv >> 5), 1u << (outv & 31));
    }
}

struct PlanLayout {
    std::vector<PlanDev> dev;
    int64_t ws_bytes = 0;
    int64_t draw_chunks = 0, step_blocks = 0;
    int64_t table_bytes = 0;
    char *table_base = nullptr;
    std::vector<int64_t> table_off;   // per plan, relative to table_base (plan tables are contiguous)
};

int layout_plans(const edgc_plan_desc *plans, int n, void *ws, int64_t ws_bytes, PlanLayout &L) {
    Arena a(ws, ws_bytes);
    L.dev.resize(n);
    PlanDev *descs_dev = a.take<PlanDev>(n);
    (void)descs_dev;
    int64_t chunk = 0, blocks = 0;

    for (int i = 0; i < n; ++i) {
        const edgc_plan_desc &d = plans[i];
        EDGC_REQUIRE(d.n_elems >= 2 && d.n_elems < (int64_t(1) << 31), "plan %d: N=%lld outside [2, 2^31)", i,
                     (long long)d.n_elems);
        EDGC_REQUIRE(d.count >= 1 && d.count < d.n_elems, "plan %d: count=%lld must be in [1, N)", i,
                     (long long)d.count);
        PlanDev &P = L.dev[i];
        P.state = (((u128)d.state_hi) << 64) | d.state_lo;
        P.inc = (((u128)d.inc_hi) << 64) | d.inc_lo;
        P.n_elems = d.n_elems;
        P.count = d.count;
        P.idx = d.idx;
        P.bitmap = d.bitmap;
        P.tail = (d.n_elems > 10000 && d.count > d.n_elems / 20) ? 1 : 0;
        // expected rejections ~ count * N / 2^33 (threshold ~ uniform below rng+1)
        const double lam = (double)d.count * (double)d.n_elems / 4294967296.0;
        int64_t slack = (int64_t)(2.0 * lam + 16.0 * std::sqrt(lam + 1.0)) + 4096;
        int64_t nd = d.count + slack;
        nd = (nd + 3) & ~int64_t(3);
        P.n_draws = nd;
        P.draw_chunk0 = chunk;
        chunk += ceil_div(nd / 2, kDrawsPerBlock);
        P.step_block0 = blocks;
        blocks += ceil_div(d.count, kStepThreads);

    }
    // round the P1 chunk index up so blocks never straddle more than needed
    L.draw_chunks = chunk;
    L.step_blocks = blocks;
    for (int i = 0; i < n; ++i) {
        PlanDev &P = L.dev[i];
        P.draws = a.take<uint32_t>(P.n_draws);
        P.rv = a.take<int32_t>(P.count);
        P.next = a.take<int32_t>(P.count);
    }
    a.off = align256(a.off);
    const int64_t t0 = a.off;
    L.table_off.assign(n + 1, 0);
    for (int i = 0; i < n; ++i) {
        PlanDev &P = L.dev[i];
        L.table_off[i] = a.off - t0;
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
    PlanLayout L;
    int rc = layout_plans(plans, n_plans, ws, ws_bytes, L);
    if (rc != EDGC_OK) return rc;
    EDGC_REQUIRE(L.ws_bytes <= ws_bytes, "edgc_sample_plan: workspace %lld < needed %lld", (long long)ws_bytes,
                 (long long)L.ws_bytes);
    cudaStream_t st = (cudaStream_t)stream;
    PlanDev *d_plans = reinterpret_cast<PlanDev *>(ws);
    EDGC_CUDA_TRY(cudaMemcpyAsync(d_plans, L.dev.data(), sizeof(PlanDev) * n_plans, cudaMemcpyHostToDevice, st));
    k_draws<<<(unsigned)L.draw_chunks, kP1Threads, 0, st>>>(d_plans, n_plans);
    EDGC_LAUNCH_CHECK();
    static bool walk_attr = false;
    if (!walk_attr) {
        EDGC_CUDA_TRY(cudaFuncSetAttribute(k_walk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(kRing * sizeof(uint32_t))));
        walk_attr = true;
    }
    k_walk<<<n_plans, kWT, kRing * sizeof(uint32_t), st>>>(d_plans, status_dev);
    EDGC_LAUNCH_CHECK();
    // index + resolve plan groups whose hash tables, links and bounded values
    // fit in L2 together, so the random table traffic stays on chip
    const int64_t kGroupBytes = 48ll << 20;
    int p0 = 0;
    while (p0 < n_plans) {
        int p1 = p0 + 1;
        int64_t bytes = (L.table_off[p0 + 1] - L.table_off[p0]) + 8 * L.dev[p0].count;
        while (p1 < n_plans) {
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
