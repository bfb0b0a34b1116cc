// Low-rank compression with error feedback (compressor.py:94-151), batched
// over a bucket set of gradient matrices, plus the (rank-averaged)
// reconstruction (compressor.py:126-133, grad_source.py:404-408).
//
// One step for every matrix k (all matrices in one launch per phase):
//   pass 1   w <- g + (w - p_res q_res^T)            (error feedback, in place)
//            P_raw = w q_warm                         (row dots, fp64 partials
//                                                      per column chunk)
//   factor   P_raw = sum of chunk partials (fixed order), Gram = P_raw^T P_raw,
//            Cholesky with MGS dead-column semantics -> T, twice (CholQR2);
//            P = P_raw T  (== MGS(P_raw), compressor.py:74-91)
//   pass 2   Q = w^T P                                (column sums, fp64
//                                                      partials per row block)
//   finalize Q = sum of row-block partials; dead columns <- fresh basis
//            (compressor.py:113-114); q_warm <- Q
// HBM traffic per element: pass 1 reads g, w and writes w (12 B); pass 2
// reads w (4 B); the reconstruction writes out (4 B).
//
// Z path (r <= 4, n <= 8192, float4-aligned): pass 1 runs as thread-block
// clusters, one cluster per row strip, one CTA per 1024-column chunk.  Row
// dots are exchanged through distributed shared memory each 8-row round, so
// every CTA knows P_raw rows while their w values are still in registers and
// accumulates Z = w^T P_raw in the same sweep.  Then Q = w^T P = Z T with the
// CholQR transform T, and pass 2 is skipped: 16 B/elem for the whole step.
// The warm start is preconditioned by the previous step's transform (any
// upper-triangular right factor leaves MGS(P) unchanged), which keeps T well
// conditioned; if cond(R) still exceeds kappa_max the matrix falls back to
// the re-read pass 2 on the device (status bit 1).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstring>
#include <cmath>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "ptx.cuh"
#include "tc_gemm.cuh"

namespace edgc {
namespace {

struct MatDev {
    const float *g;
    float *w;
    const float *p_res;
    const float *q_res;
    float *q_warm;
    const float *basis;
    float *p_out;
    float *q_out;
    int64_t m, n, ld_g;
    int32_t r, r_res, ld_q, vec;
    // scratch (workspace)
    double *p_part;   // [nchunk1][m][r]
    double *p_raw;    // [m][r]
    double *q_part;   // [nblk2][n][r]
    double *tmat;     // [r][r] combined T (column j at tmat[j*r .. j*r+r))
    int32_t *dead;    // [r]
    int32_t nchunk1, nblk2;
    double *precond;  // state: r_cap x r_cap upper-triangular warm-start preconditioner (or NULL)
    double *zpart;    // [nitems][n][r] Z partials (Z path)
    int32_t ld_s, zmode, nitems, zc;   // zc = cluster size (column chunks) on the Z path
    double *fwork;    // 5 r^2 factor scratch
    double *p_tmp;    // [m][r] CholQR intermediate
    int32_t wide;     // wide = 1: tiled GEMM path (r > 8 or unaligned)
    int32_t zw;       // Z path: columns per CTA of the cluster (multiple of 4, <= kTCW)
    int32_t al4;      // g and w rows float4-aligned (n, ld_g multiples of 4, 16-byte bases)
    int32_t tc;       // wide path on the tensor cores (P_raw and Q with one K split each)
    int32_t fx;       // factorisation by the multi-CTA kernels (wide ranks): k_factor skips it
    int32_t gks;      // rows per Gram K split (fx)
    int32_t gsplit;   // Gram K splits (fx)
    double *gpart;    // [gsplit][r][r] Gram partials (fx; aliases q_part when it fits)
    int32_t *fmode;   // fx: 1 = single CholQR, 2 = CholQR2 (set by k_fx_chol1)
};

// fused sampled-iteration statistics of one matrix (edgc_compress_plan_set_sampling)
struct SampDev {
    const uint32_t *bitmap;   // membership bits, NULL = not sampled
    const int32_t *first;     // flat index of the first sample (shift)
    double *part;             // [slots][2] shifted sums of this matrix
};

// Z-path work item: one row strip of one matrix, processed by one cluster
struct ZTile {
    int32_t mat, item;
    int64_t row0, row1;
};

// pass-1 / pass-2 tiles
struct Tile {
    int32_t mat;
    int32_t chunk;   // column chunk index (pass 1) / row block index (pass 2)
    int64_t slot0, slot1;  // [slot0, slot1) column slots (VEC columns each)
    int64_t row0, row1;
};

constexpr int kP1Threads = 256;
constexpr int kP1Rows = 64;     // rows per pass-1 tile
constexpr int kP2Threads = 256;
constexpr int kP2Rows = 256;    // rows per pass-2 tile (one fp64 partial per block)
constexpr int kFactorThreads = 256;
constexpr int kMaxRank = 1024;     // device limit (TMEM-free fp32 path)
constexpr int kNarrow = 8;         // register kernels up to this rank
constexpr int64_t kWideSplitK = 2048;
constexpr int kZRows = 512;    // rows per cluster work item
constexpr double kKappaMax = 64.0;

template <int VEC> struct VecT;
template <> struct VecT<4> {
    typedef float4 T;
    __device__ static float4 ld(const float *p) { return __ldg(reinterpret_cast<const float4 *>(p)); }
    __device__ static float4 ld_cs(const float *p) { return __ldcs(reinterpret_cast<const float4 *>(p)); }
    __device__ static void st(float *p, const float (&v)[4]) {
        *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
    }
    __device__ static void unpack(const float4 &x, float (&v)[4]) { v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w; }
};
template <> struct VecT<2> {
    typedef float2 T;
    __device__ static float2 ld(const float *p) { return __ldg(reinterpret_cast<const float2 *>(p)); }
    __device__ static float2 ld_cs(const float *p) { return __ldcs(reinterpret_cast<const float2 *>(p)); }
    __device__ static void st(float *p, const float (&v)[2]) { *reinterpret_cast<float2 *>(p) = make_float2(v[0], v[1]); }
    __device__ static void unpack(const float2 &x, float (&v)[2]) { v[0] = x.x; v[1] = x.y; }
};
template <> struct VecT<1> {
    typedef float T;
    __device__ static float ld(const float *p) { return __ldg(p); }
    __device__ static float ld_cs(const float *p) { return __ldcs(p); }
    __device__ static void st(float *p, const float (&v)[1]) { *p = v[0]; }
    __device__ static void unpack(const float &x, float (&v)[1]) { v[0] = x; }
};

// ------------------------------------------------------------------ pass 1
// RB rows at a time; per row the thread's VEC columns give RMAX partial dots,
// reduced across the CTA in fp64 (butterfly within warps, fixed-order sum
// across warps) and written as this column chunk's partial of P_raw.
template <int VEC, int RMAX, int RB>
__global__ void __launch_bounds__(kP1Threads) k_pass1(const MatDev *mats, const Tile *tiles, int32_t *status) {
    constexpr int V = RB * RMAX;               // values reduced per row block
    constexpr int VW = V < 32 ? V : 32;        // values per butterfly
    constexpr int NB = V / VW;                 // butterflies per row block
    constexpr int NWARP = kP1Threads / 32;
    const Tile t = tiles[blockIdx.x];
    const MatDev &M = mats[t.mat];
    const int r = M.r, rr_res = M.r_res;
    const int64_t n = M.n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t slot = t.slot0 + tid;
    const bool active = slot < t.slot1;
    const int64_t col0 = slot * VEC;

    __shared__ float s_pres[RB][RMAX];
    __shared__ double s_red[NWARP][V];

    float qw[VEC][RMAX], qr[VEC][RMAX];
#pragma unroll
    for (int v = 0; v < VEC; ++v)
#pragma unroll
        for (int k = 0; k < RMAX; ++k) {
            qw[v][k] = (active && k < r) ? M.q_warm[(col0 + v) * M.ld_q + k] : 0.f;
            qr[v][k] = (active && k < rr_res) ? M.q_res[(col0 + v) * rr_res + k] : 0.f;
        }
    bool bad = false;
    for (int64_t row = t.row0; row < t.row1; row += RB) {
        __syncthreads();
        if (tid < RB * RMAX) {
            const int rr = tid / RMAX, k = tid % RMAX;
            const int64_t i = row + rr;
            s_pres[rr][k] = (k < rr_res && i < t.row1) ? M.p_res[i * rr_res + k] : 0.f;
        }
        __syncthreads();
        double acc[V];
#pragma unroll
        for (int rr = 0; rr < RB; ++rr) {
            const int64_t i = row + rr;
            float pk[RMAX];
#pragma unroll
            for (int k = 0; k < RMAX; ++k) pk[k] = 0.f;
            if (active && i < t.row1) {
                float gv[VEC], wv[VEC];
                VecT<VEC>::unpack(VecT<VEC>::ld_cs(M.g + i * M.ld_g + col0), gv);
                VecT<VEC>::unpack(VecT<VEC>::ld_cs(M.w + i * n + col0), wv);
#pragma unroll
                for (int v = 0; v < VEC; ++v) {
                    // residual = w - p_res q_res^T (compressor.py:112), then work = g + residual (:106)
                    float dot = 0.f;
#pragma unroll
                    for (int k = 0; k < RMAX; ++k) dot = fmaf(s_pres[rr][k], qr[v][k], dot);
                    const float x = gv[v] + (wv[v] - dot);
                    bad |= !isfinite(x);
                    wv[v] = x;
#pragma unroll
                    for (int k = 0; k < RMAX; ++k) pk[k] = fmaf(x, qw[v][k], pk[k]);
                }
                VecT<VEC>::st(M.w + i * n + col0, wv);
            }
#pragma unroll
            for (int k = 0; k < RMAX; ++k) acc[rr * RMAX + k] = (double)pk[k];
        }
        // reduce acc across the CTA
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            double part[VW];
#pragma unroll
            for (int q = 0; q < VW; ++q) part[q] = acc[b * VW + q];
            const double s = warp_reduce_scatter<VW>(part, lane);
            const int owner = scatter_owner_index<VW>(lane);
            if ((lane & ((32 / VW) - 1)) == 0) s_red[warp][b * VW + owner] = s;
        }
        __syncthreads();
        if (tid < V) {
            const int rr = tid / RMAX, k = tid % RMAX;
            const int64_t i = row + rr;
            if (i < t.row1 && k < r) {
                double s = 0.0;
#pragma unroll
                for (int w = 0; w < NWARP; ++w) s += s_red[w][tid];
                M.p_part[((int64_t)t.chunk * M.m + i) * r + k] = s;
            }
        }
    }
    if (__syncthreads_or(bad) && tid == 0) atomicOr(status + t.mat, 1);
}

// ------------------------------------------- pass 1 (Z, TMA-pipelined)
// Warp-specialised for bandwidth.  Per CTA (one per <= 1280-column chunk of a
// cluster's row strip; clusters of 1, 2, 3 or 6 CTAs pack the 18-20 SM GPCs,
// 7-8 only for n > 7680):
//   producer warp  streams [4 rows x chunk] tiles of g and w into a 3-stage
//                  shared-memory ring with 1-D bulk async copies (TMA
//                  engine, mbarrier complete_tx);
//   10 consumer warps  error feedback, w write-back, fp64 row dots (exact
//                  fp32 x fp32 products), per-warp butterfly -> red[] ring;
//                  then, kTLag rounds later, Z += x * P_raw with that round's
//                  rows -- they never wait on the cluster;
//   exchange warp  sums the 8 warp partials, pushes them into every peer's
//                  shared memory (st.shared::cluster) and release-arrives on
//                  the peer's mbarrier; it completes round b - kTD (waits for
//                  all peers, publishes the P_raw rows) only after pushing
//                  round b, so one cluster round trip is always in flight.
// All hand-offs are mbarriers / named barriers; no block-wide barrier in the
// steady state.  Non-finite work is detected on the exchanged row sums: a
// fp64 sum of exact fp32 x fp32 products is non-finite iff one of the x is.
#ifndef EDGC_TLAG
#define EDGC_TLAG 3
#endif
constexpr int kTCons = 320;
constexpr int kTThreads = kTCons + 64;   // + producer warp + exchange warp
constexpr int kTRB = 4;
#ifndef EDGC_P1_STASYNC
#define EDGC_P1_STASYNC 1   // peer pushes by st.async + complete_tx (0: st.shared::cluster + release arrive)
#endif
#ifndef EDGC_P1_EARLYZ
#define EDGC_P1_EARLYZ 1    // 1: the lagged Z update runs right after the stage wait (interleaves with the round)
#endif
#ifndef EDGC_P1_MEMONLY
#define EDGC_P1_MEMONLY 0   // diagnostics: stream g, w -> w only (no row dots, exchange or Z)
#endif
#ifndef EDGC_P1_NOEXCH
#define EDGC_P1_NOEXCH 0    // diagnostics: row dots + warp reductions, no cluster exchange / Z
#endif
#ifndef EDGC_P1_NOZ
#define EDGC_P1_NOZ 0       // diagnostics: full exchange, Z update skipped
#endif
#ifndef EDGC_TCEF_PFD
#define EDGC_TCEF_PFD 3
#endif
#ifndef EDGC_TCEF_STAGES
#define EDGC_TCEF_STAGES 1
#endif
#ifndef EDGC_PROD_SLEEP
#define EDGC_PROD_SLEEP 64
#endif
#ifndef EDGC_CONS_SLEEP
#define EDGC_CONS_SLEEP 0
#endif
#ifndef EDGC_TSTAGES
#define EDGC_TSTAGES 3
#endif
constexpr int kTStages = EDGC_TSTAGES;   // 32 KB TMA stages (pure prefetch: x lives in its own ring)
constexpr int kTCW = 4 * kTCons;
constexpr int kTLag = EDGC_TLAG;         // consumer Z update lags its round by this many rounds
#ifndef EDGC_TD
#define EDGC_TD 1
#endif
#ifndef EDGC_STCS
#define EDGC_STCS 1
#endif
#ifndef EDGC_CONS_FINITE
#define EDGC_CONS_FINITE 0
#endif
constexpr int kTD = EDGC_TD;             // exchange completes round b - kTD after pushing round b
static_assert(kTLag >= kTD, "consumers must not wait for a round the exchange has not completed");
constexpr int kTRing = kTLag + 1;        // red / prow / named-barrier ring depth
constexpr int kTSlots = 2 * kTD + 2;     // DSMEM receive slots (a peer refills slot b only after my round b)
constexpr int kTV = kTRB * 4;            // row-dot values per round (RMAX = 4)

struct TSmem {
    float g[kTStages][kTRB][kTCW];
    float w[kTStages][kTRB][kTCW];
    float xs[kTRing][kTRB][kTCW];        // x (new w) of the last kTRing rounds (each thread its own columns)
    float prowf[kTRing][kTV];            // P_raw rows of the round, as float, for the Z update
    double recv[kTSlots][8][kTV];
    double red[kTRing][kTCons / 32][kTV];
    double S[16];
    alignas(8) uint64_t full[kTStages];
    alignas(8) uint64_t empty[kTStages];
    alignas(8) uint64_t xfull[kTSlots];
    alignas(8) uint64_t prowready[kTRing];
};

template <bool SAMPLE>
__global__ void __launch_bounds__(kTThreads, 1) k_pass1t(const MatDev *mats, const ZTile *tiles, int32_t *status,
                                                         const SampDev *samp) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    TSmem &sm = *reinterpret_cast<TSmem *>(smem_raw);
    const uint32_t C = ptx::cluster_nctarank();
    const uint32_t me = ptx::cluster_ctarank();
    const ZTile t = tiles[blockIdx.x / C];
    const MatDev &M = mats[t.mat];
    // descriptor fields in registers: the asm memory clobbers below would
    // otherwise force a global reload of every field each round
    const int r = M.r, rr_res = M.r_res;
    const int64_t n = M.n, ld_g = M.ld_g, ld_q = M.ld_q;
    const float *__restrict__ gptr = M.g;
    float *wptr = M.w;
    const float *__restrict__ pres_ptr = M.p_res;
    const float *__restrict__ qres_ptr = M.q_res;
    const float *__restrict__ qwarm_ptr = M.q_warm;
    double *praw_ptr = M.p_raw;
    double *zpart_ptr = M.zpart;
    const double *precond_ptr = M.precond;
    const int ld_s = M.ld_s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t col_base = (int64_t)me * M.zw;
    const int64_t chunk_cols = max((int64_t)0, min((int64_t)M.zw, n - col_base));
    const int nrounds = (int)((t.row1 - t.row0 + kTRB - 1) / kTRB);
    constexpr int kProducer = kTCons / 32, kExchange = kTCons / 32 + 1;

    if (tid == 0) {
        for (int s = 0; s < kTStages; ++s) {
            ptx::mbar_init(&sm.full[s], 1);
            ptx::mbar_init(&sm.empty[s], kTCons / 32);
        }
        for (int s = 0; s < kTSlots; ++s) ptx::mbar_init(&sm.xfull[s], EDGC_P1_STASYNC ? 1 : C);
        for (int s = 0; s < kTRing; ++s) ptx::mbar_init(&sm.prowready[s], 1);
        ptx::fence_mbar_init();
    }
    if (tid < 16) {
        const int i = tid / 4, k = tid % 4;
        double v = (i == k) ? 1.0 : 0.0;
        if (precond_ptr && i < r && k < r) v = precond_ptr[(int64_t)i * ld_s + k];
        sm.S[tid] = v;
    }
    ptx::cluster_sync();

    if (warp == kProducer) {
        if (lane == 0 && chunk_cols > 0) {
            const uint32_t bytes = (uint32_t)(chunk_cols * 4);
            for (int b = 0; b < nrounds; ++b) {
                const int s = b % kTStages;
                const int64_t i0 = t.row0 + (int64_t)b * kTRB;
                const int rows = (int)min((int64_t)kTRB, t.row1 - i0);
                if (b >= kTStages) ptx::mbar_wait_sleep<EDGC_PROD_SLEEP>(&sm.empty[s], ((b / kTStages) - 1) & 1);
                ptx::mbar_arrive_expect_tx(&sm.full[s], 2u * bytes * (uint32_t)rows);
                for (int rr = 0; rr < rows; ++rr) {
                    ptx::bulk_g2s(&sm.g[s][rr][0], gptr + (i0 + rr) * ld_g + col_base, bytes, &sm.full[s]);
                    ptx::bulk_g2s(&sm.w[s][rr][0], wptr + (i0 + rr) * n + col_base, bytes, &sm.full[s]);
                }
            }
        }
    } else if (warp == kExchange) {
        if (EDGC_P1_MEMONLY) goto done;
        if (EDGC_P1_NOEXCH) {
            for (int b = 0; b < nrounds; ++b) ptx::named_bar_sync(2 + b % kTRing, kTCons + 32);
            goto done;
        }
        bool bad = false;
        auto push = [&](int b) {
            const int q = b % kTRing, slot = b % kTSlots;
            ptx::named_bar_sync(2 + q, kTCons + 32);   // the consumer warps wrote red[q]
            {
                // all 32 lanes: lane l sums half of the warps' partials of value l % 16, fixed order
                constexpr int kHalf = kTCons / 64;
                const int v = lane & (kTV - 1), w0 = (lane >> 4) * kHalf;
                double a = 0.0;
#pragma unroll
                for (int w = 0; w < kHalf; ++w) a += sm.red[q][w0 + w][v];
                a += __shfl_xor_sync(0xffffffffu, a, 16);
                if (lane < kTV) sm.recv[slot][me][lane] = a;            // my own contribution, in place
            }
            __syncwarp();
#if EDGC_P1_STASYNC
            // my barrier expects the C-1 peers' vectors as transaction bytes; my own arrive
            // (release) publishes my own slot; the peers' st.async complete the transaction
            if (lane == 0) ptx::mbar_arrive_expect_tx(&sm.xfull[slot], (C - 1u) * kTV * 8u);
            if ((uint32_t)lane < C && (uint32_t)lane != me) {
                // lane cc streams the whole row-dot vector into peer cc's slot for me
                const uint32_t cc = (uint32_t)lane;
                const uint32_t dst = ptx::mapa(ptx::smem_addr(&sm.recv[slot][me][0]), cc);
                const uint32_t bar = ptx::mapa(ptx::smem_addr(&sm.xfull[slot]), cc);
#pragma unroll
                for (int e = 0; e < kTV; e += 2)
                    ptx::st_async_v2_f64(dst + 8u * e, sm.recv[slot][me][e], sm.recv[slot][me][e + 1], bar);
            }
#else
            if ((uint32_t)lane < C && (uint32_t)lane != me) {
                // lane cc pushes the whole row-dot vector to peer cc, then release-arrives
                // there: the C pushes and releases proceed in parallel
                const uint32_t cc = (uint32_t)lane;
                const uint32_t dst = ptx::mapa(ptx::smem_addr(&sm.recv[slot][me][0]), cc);
#pragma unroll
                for (int e = 0; e < kTV; e += 2)
                    ptx::st_cluster_v2_f64(dst + 8u * e, sm.recv[slot][me][e], sm.recv[slot][me][e + 1]);
                ptx::mbar_arrive_remote(ptx::mapa(ptx::smem_addr(&sm.xfull[slot]), cc));
            }
            if ((uint32_t)lane == me) ptx::mbar_arrive_cta(&sm.xfull[slot]);
#endif
        };
        auto complete = [&](int b) {
            const int q = b % kTRing, slot = b % kTSlots;
            ptx::mbar_wait_cluster(&sm.xfull[slot], (b / kTSlots) & 1);
            if (lane < kTV) {
                double a = 0.0;
                for (uint32_t cc = 0; cc < C; ++cc) a += sm.recv[slot][cc][lane];
                if (!EDGC_CONS_FINITE) bad |= !isfinite(a);
                sm.prowf[q][lane] = (float)a;
                const int64_t i = t.row0 + (int64_t)b * kTRB + (lane >> 2);
                const int k = lane & 3;
                if (me == 0 && i < t.row1 && k < r) praw_ptr[i * r + k] = a;
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cta(&sm.prowready[q]);
        };
        for (int b = 0; b < nrounds; ++b) {
            push(b);
            if (b >= kTD) complete(b - kTD);
        }
        for (int bb = max(0, nrounds - kTD); bb < nrounds; ++bb) complete(bb);
        if (__any_sync(0xffffffffu, bad) && lane == 0 && me == 0) atomicOr(status + t.mat, 1);
    } else {
        // ---------------- consumer warps
        // Lane-permuted partials: lane L computes output (row, k) = slot i ^ f(L) into slot i,
        // f(L) = bits (16, 8, 4, 2) of L.  Partner lanes at every butterfly level then hold their
        // halves in opposite order, so the fp64 reduce-scatter is shuffle + add only (no selects):
        // rows are processed in order rr ^ f/4 and the q_warm columns are pre-permuted by f%4.
        const int f = (((lane >> 4) & 1) << 3) | (((lane >> 3) & 1) << 2) | (((lane >> 2) & 1) << 1) |
                      ((lane >> 1) & 1);
        const int fr = f >> 2, fk = f & 3;
        const int64_t col0 = col_base + 4 * tid;
        const bool active = 4 * tid < chunk_cols;
        double qw[4][4];
        float qr[4][4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            double raw[4], nat[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) raw[k] = (active && k < r) ? (double)qwarm_ptr[(col0 + v) * ld_q + k] : 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                double a = 0.0;
#pragma unroll
                for (int i = 0; i <= k; ++i) a += raw[i] * sm.S[i * 4 + k];
                nat[k] = a;
                qr[v][k] = (active && k < rr_res) ? qres_ptr[(col0 + v) * rr_res + k] : 0.f;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
                qw[v][k] = fk == 0 ? nat[k] : fk == 1 ? nat[k ^ 1] : fk == 2 ? nat[k ^ 2] : nat[k ^ 3];
        }
        float zacc[4][4];
#pragma unroll
        for (int v = 0; v < 4; ++v)
#pragma unroll
            for (int k = 0; k < 4; ++k) zacc[v][k] = 0.f;
        bool bad = false;
        // sampled iteration: shifted sums of the raw gradient over the membership bits
        double gs1 = 0.0, gs2 = 0.0, gK = 0.0;
        const uint32_t *sbits = nullptr;
        if (SAMPLE) {
            sbits = samp[t.mat].bitmap;
            if (sbits) {
                const int64_t f = __ldg(samp[t.mat].first);
                gK = (double)__ldg(gptr + (f / n) * ld_g + f % n);
            }
        }
        // round bb's x values wait in xs[bb % kTRing] (this thread's columns only) for the lagged Z update
        auto consume = [&](int bb) {
            const int q = bb % kTRing;
            ptx::mbar_wait_sleep<EDGC_CONS_SLEEP>(&sm.prowready[q], (bb / kTRing) & 1);
            if (EDGC_P1_NOZ) return;
#pragma unroll
            for (int rr = 0; rr < kTRB; ++rr) {
                const float4 pv = *reinterpret_cast<const float4 *>(&sm.prowf[q][rr * 4]);
                const float4 xv = *reinterpret_cast<const float4 *>(&sm.xs[q][rr][4 * tid]);
                const float xx[4] = {xv.x, xv.y, xv.z, xv.w}, pp[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
                for (int k = 0; k < 4; ++k)
#pragma unroll
                    for (int v = 0; v < 4; ++v) zacc[v][k] = fmaf(xx[v], pp[k], zacc[v][k]);
            }
        };
        // p_res rows of a round in this lane's row order, one round ahead (broadcast loads)
        const bool pres_v4 = rr_res == 4 && ((uintptr_t)pres_ptr & 15) == 0;
        auto load_pres = [&](int bb, float4 (&pr)[kTRB]) {
            const int64_t r0 = t.row0 + (int64_t)bb * kTRB;
            const int nrow = (int)min((int64_t)kTRB, t.row1 - r0);   // <= 0 past the strip
            if (pres_v4) {
                const float4 *base = reinterpret_cast<const float4 *>(pres_ptr) + r0;
#pragma unroll
                for (int rr = 0; rr < kTRB; ++rr)
                    pr[rr] = (rr ^ fr) < nrow ? __ldg(base + (rr ^ fr)) : make_float4(0.f, 0.f, 0.f, 0.f);
            } else {
#pragma unroll
                for (int rr = 0; rr < kTRB; ++rr) {
                    float pq[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        pq[k] = ((rr ^ fr) < nrow && k < rr_res) ? __ldg(pres_ptr + (r0 + (rr ^ fr)) * rr_res + k) : 0.f;
                    pr[rr] = make_float4(pq[0], pq[1], pq[2], pq[3]);
                }
            }
        };
        float4 pcur[kTRB];
        load_pres(0, pcur);
        // membership bits of a round's 4 x 4 elements, loaded a round ahead (like p_res): a load
        // consumed in its own round would stall every round on a global round trip
        auto load_bits = [&](int bb, uint32_t (&sw)[kTRB]) {
            const int64_t r0 = t.row0 + (int64_t)bb * kTRB;
            const int nrow = (int)min((int64_t)kTRB, t.row1 - r0);   // <= 0 past the strip
#pragma unroll
            for (int rr = 0; rr < kTRB; ++rr) {
                const int lr = rr ^ fr;
                const int64_t e = (r0 + lr) * n + col0;   // 4-aligned: the 4 bits share a word
                sw[rr] = (active && lr < nrow) ? (__ldg(sbits + (e >> 5)) >> (e & 31)) & 0xFu : 0u;
            }
        };
        uint32_t swcur[kTRB] = {0u, 0u, 0u, 0u};
        if (SAMPLE && sbits) load_bits(0, swcur);
#pragma unroll 1
        for (int b = 0; b < nrounds; ++b) {
            const int s = b % kTStages, q = b % kTRing;
            const int64_t i0 = t.row0 + (int64_t)b * kTRB;
            const int rows = (int)min((int64_t)kTRB, t.row1 - i0);
            float4 pnext[kTRB];
            load_pres(b + 1, pnext);
            uint32_t swnext[kTRB] = {0u, 0u, 0u, 0u};
            if (SAMPLE && sbits) load_bits(b + 1, swnext);
            if (chunk_cols > 0) ptx::mbar_wait_sleep<EDGC_CONS_SLEEP>(&sm.full[s], (b / kTStages) & 1);
            if (EDGC_P1_EARLYZ && !EDGC_P1_NOEXCH && b >= kTLag) consume(b - kTLag);
            uint32_t sw[kTRB];
#pragma unroll
            for (int rr = 0; rr < kTRB; ++rr) sw[rr] = swcur[rr];
            double acc[kTV];
#pragma unroll
            for (int rr = 0; rr < kTRB; ++rr) {
                const int lr = rr ^ fr;   // the logical row of this slot
                const float4 gv = *reinterpret_cast<const float4 *>(&sm.g[s][lr][4 * tid]);
                const float4 wv = *reinterpret_cast<const float4 *>(&sm.w[s][lr][4 * tid]);
                const bool live = active && lr < rows;
                const float pp[4] = {pcur[rr].x, pcur[rr].y, pcur[rr].z, pcur[rr].w};
                const float gg[4] = {gv.x, gv.y, gv.z, gv.w};
                const float ww[4] = {wv.x, wv.y, wv.z, wv.w};
                if (SAMPLE && sbits) {
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        if ((sw[rr] >> v) & 1u) {
                            const double d = (double)gg[v] - gK;
                            gs1 += d;
                            gs2 = fma(d, d, gs2);
                        }
                }
                float xx[4];
                double pk[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    float dot = 0.f;
#pragma unroll
                    for (int k = 0; k < 4; ++k) dot = fmaf(pp[k], qr[v][k], dot);
                    xx[v] = live ? gg[v] + (ww[v] - dot) : 0.f;
#if EDGC_CONS_FINITE
                    bad |= !isfinite(xx[v]);
#endif
                    const double xd = (double)xx[v];
#pragma unroll
                    for (int k = 0; k < 4; ++k) pk[k] = fma(xd, qw[v][k], pk[k]);
                }
                if (live) {
#if EDGC_STCS
                    __stcs(reinterpret_cast<float4 *>(wptr + (i0 + lr) * n + col0), make_float4(xx[0], xx[1], xx[2], xx[3]));
#else
                    ptx::st_global_v4(wptr + (i0 + lr) * n + col0, xx[0], xx[1], xx[2], xx[3]);
#endif
                }
                *reinterpret_cast<float4 *>(&sm.xs[q][lr][4 * tid]) = make_float4(xx[0], xx[1], xx[2], xx[3]);
#pragma unroll
                for (int k = 0; k < 4; ++k) acc[rr * 4 + k] = pk[k];
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_relaxed(&sm.empty[s]);   // stage s read: refill it
            if (EDGC_P1_MEMONLY) continue;
            // select-free reduce-scatter (offsets 16, 8, 4, 2 halve the slots; 1 finishes)
#pragma unroll
            for (int h = kTV / 2; h >= 1; h >>= 1)
#pragma unroll
                for (int i = 0; i < h; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i + h], 2 * h);
            acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
            if ((lane & 1) == 0) sm.red[q][warp][f] = acc[0];
            ptx::named_bar_arrive(2 + q, kTCons + 32);   // hand red[q] to the exchange warp
            if (!EDGC_P1_EARLYZ && !EDGC_P1_NOEXCH && b >= kTLag) consume(b - kTLag);
#pragma unroll
            for (int rr = 0; rr < kTRB; ++rr) {
                pcur[rr] = pnext[rr];
                swcur[rr] = swnext[rr];
            }
        }
        if (EDGC_P1_MEMONLY || EDGC_P1_NOEXCH) goto done;
        for (int bb = max(0, nrounds - kTLag); bb < nrounds; ++bb) consume(bb);
        if (active) {
#pragma unroll
            for (int v = 0; v < 4; ++v)
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (k < r) zpart_ptr[((int64_t)t.item * n + col0 + v) * r + k] = (double)zacc[v][k];
        }
        if (EDGC_CONS_FINITE && bad) atomicOr(status + t.mat, 1);
        if (SAMPLE && sbits) {
            // this CTA's slot: fixed-order sum over the consumer warps
            __shared__ double s_gs[kTCons / 32][2];
            gs1 = warp_sum(gs1);
            gs2 = warp_sum(gs2);
            if (lane == 0) { s_gs[warp][0] = gs1; s_gs[warp][1] = gs2; }
            ptx::named_bar_sync(7, kTCons);
            if (tid == 0) {
                double a = 0.0, c = 0.0;
                for (int w = 0; w < kTCons / 32; ++w) { a += s_gs[w][0]; c += s_gs[w][1]; }
                double *dst = samp[t.mat].part + 2 * ((int64_t)t.item * C + me);
                dst[0] = a;
                dst[1] = c;
            }
        }
    }
done:
    ptx::cluster_sync();  // no CTA leaves while a peer may still push into it
}

// ------------------------------------------------------------------ factor
// One CTA per matrix; r x r work matrices live in the matrix's workspace slice
// (L1/L2 resident).  Gram by (entry, row-group) partial sums reduced in fixed
// order; right-looking Cholesky with the MGS dead-column rule (a column whose
// projected norm -- the Schur-complement diagonal -- is <= tol is zeroed and
// drops out of later projections, compressor.py:80-90); triangular inverse by
// independent column back-substitutions; everything fp64 and deterministic.
// r <= 4: each thread owns whole rows (stride kFactorThreads) and accumulates
// all r(r+1)/2 products in registers; then per-warp butterflies and a
// fixed-order sum over warps (deterministic).
template <int R>
__device__ void gram_rows(const double *P, int64_t m, double *gram) {
    constexpr int E = R * (R + 1) / 2;
    __shared__ double s_part[kFactorThreads / 32][10];
    double acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = 0.0;
#pragma unroll 4
    for (int64_t i = threadIdx.x; i < m; i += kFactorThreads) {
        double x[R];
#pragma unroll
        for (int a = 0; a < R; ++a) x[a] = P[i * R + a];
        int e = 0;
#pragma unroll
        for (int a = 0; a < R; ++a)
#pragma unroll
            for (int b = a; b < R; ++b, ++e) acc[e] = fma(x[a], x[b], acc[e]);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int e = 0; e < E; ++e)
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
    if (lane == 0) {
#pragma unroll
        for (int e = 0; e < E; ++e) s_part[warp][e] = acc[e];
    }
    __syncthreads();
    if (threadIdx.x < E) {
        int a = 0, rem = threadIdx.x;
        while (rem >= R - a) { rem -= R - a; ++a; }
        const int b = a + rem;
        double sum = 0.0;
        for (int w = 0; w < kFactorThreads / 32; ++w) sum += s_part[w][threadIdx.x];
        gram[a * R + b] = sum;
        gram[b * R + a] = sum;
    }
    __syncthreads();
}

// r > 4: 4x4 register blocks of the Gram's upper block triangle, rows split over
// row groups when there are fewer blocks than threads; fixed-order group sums.
__device__ void gram_pass(const double *P, int64_t m, int r, double *gram, double *s_tmp) {
    switch (r) {
        case 1: gram_rows<1>(P, m, gram); return;
        case 2: gram_rows<2>(P, m, gram); return;
        case 3: gram_rows<3>(P, m, gram); return;
        case 4: gram_rows<4>(P, m, gram); return;
        default: break;
    }
    (void)s_tmp;
    __shared__ double s_blk[kFactorThreads][16];
    const int tid = threadIdx.x;
    const int nbk = (r + 3) / 4, nblocks = nbk * (nbk + 1) / 2;
    const int ng = max(1, kFactorThreads / nblocks);      // row groups
    const int per = kFactorThreads / ng;                   // block slots per row group (>= nblocks or all)
    const int g = tid / per < ng ? tid / per : -1;
    for (int blk0 = 0; blk0 < nblocks; blk0 += kFactorThreads / ng) {
        const int slots = min(nblocks - blk0, kFactorThreads / ng);
        const int blk = blk0 + tid % (kFactorThreads / ng);
        const bool mine = g >= 0 && (tid % (kFactorThreads / ng)) < slots;
        double acc[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
        int A = 0, B = 0;
        if (mine) {
            int rem = blk;
            while (rem >= nbk - A) { rem -= nbk - A; ++A; }
            B = A + rem;
#pragma unroll 2
            for (int64_t i = g; i < m; i += ng) {
                const double *row = P + i * r;
                double pa[4], pb[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    pa[u] = 4 * A + u < r ? row[4 * A + u] : 0.0;
                    pb[u] = 4 * B + u < r ? row[4 * B + u] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[u][v] = fma(pa[u], pb[v], acc[u][v]);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) s_blk[tid][u * 4 + v] = acc[u][v];
        __syncthreads();
        // thread (slot, entry) sums its block entry over the row groups in order
        for (int e = tid; e < slots * 16; e += kFactorThreads) {
            const int sl = e / 16, uv = e % 16;
            double sum = 0.0;
            for (int gg = 0; gg < ng; ++gg) sum += s_blk[gg * (kFactorThreads / ng) + sl][uv];
            int rem = blk0 + sl, AA = 0;
            while (rem >= nbk - AA) { rem -= nbk - AA; ++AA; }
            const int BB = AA + rem;
            const int a = 4 * AA + uv / 4, bb = 4 * BB + uv % 4;
            if (a < r && bb < r && (AA != BB || bb >= a)) {
                gram[a * r + bb] = sum;
                gram[bb * r + a] = sum;
            }
        }
        __syncthreads();
    }
}

// A (r x r, destroyed) -> R (upper, row-major R[i*r+j]); dead[] updated when detect.
// tol_k = tol * scale[k] (scale = NULL -> 1).
template <int NT = kFactorThreads>
__device__ void chol_dead(double *A, int r, double tol, const double *scale, int32_t *dead, double *R, bool detect) {
    const int tid = threadIdx.x;
    for (int e = tid; e < r * r; e += NT) R[e] = 0.0;
    __syncthreads();
    for (int k = 0; k < r; ++k) {
        if (tid == 0) {
            const double nrm = sqrt(fmax(A[k * r + k], 0.0));
            if (detect) dead[k] = !(nrm > tol * (scale ? scale[k] : 1.0));
            R[k * r + k] = dead[k] ? 0.0 : nrm;
        }
        __syncthreads();
        if (!dead[k]) {
            const double piv = R[k * r + k];
            for (int j = k + 1 + tid; j < r; j += NT) R[k * r + j] = A[k * r + j] / piv;
            __syncthreads();
            // trailing upper triangle, one warp per row i, lanes along j (coalesced, no div/mod)
            const double *rk = R + k * r;
            for (int i = k + 1 + tid / 32; i < r; i += NT / 32) {
                const double ri = rk[i];
                double *Ai = A + i * r;
                int j = i + tid % 32;
                // four elements per lane in flight (loads first: A and R share the workspace)
                for (; j + 96 < r; j += 128) {
                    double a0 = Ai[j], a1 = Ai[j + 32], a2 = Ai[j + 64], a3 = Ai[j + 96];
                    const double b0 = rk[j], b1 = rk[j + 32], b2 = rk[j + 64], b3 = rk[j + 96];
                    a0 -= ri * b0;
                    a1 -= ri * b1;
                    a2 -= ri * b2;
                    a3 -= ri * b3;
                    Ai[j] = a0;
                    Ai[j + 32] = a1;
                    Ai[j + 64] = a2;
                    Ai[j + 96] = a3;
                }
                for (; j < r; j += 32) Ai[j] -= ri * rk[j];
            }
        }
        __syncthreads();
    }
}

// T = R^{-1} over the live columns (dead rows/columns zero); T column j at T[j*r + i].
// One warp per column (columns dealt round-robin, so the O(j^2) costs balance): the
// back substitution is sequential in i, each step a lane-strided dot product of row i
// of R with the column so far, summed by a fixed-order butterfly (deterministic).
template <int NT = kFactorThreads>
__device__ void tri_inverse(const double *R, const int32_t *dead, int r, double *T) {
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    constexpr int kW = NT / 32;
    for (int j = warp; j < r; j += kW) {
        double *x = T + (int64_t)j * r;
        for (int i = lane; i < r; i += 32) x[i] = 0.0;
        __syncwarp();
        if (dead[j]) continue;
        if (lane == 0) x[j] = 1.0 / R[j * r + j];
        __syncwarp();
        for (int i = j - 1; i >= 0; --i) {
            if (dead[i]) continue;
            double acc = 0.0;
            for (int l = i + 1 + lane; l <= j; l += 32) acc += R[i * r + l] * x[l];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) x[i] = -acc / R[i * r + i];
            __syncwarp();
        }
    }
    __syncthreads();
}

// dst (m x r) = src (m x r) * T (upper, column-major by column)
template <int R>
__device__ void right_mul_rows(const double *src, const double *T, int64_t m, double *dst, float *dst_f) {
    double t[R][R];
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
        for (int l = 0; l <= j; ++l) t[j][l] = T[j * R + l];
#pragma unroll 4
    for (int64_t i = threadIdx.x; i < m; i += kFactorThreads) {
        double x[R];
#pragma unroll
        for (int l = 0; l < R; ++l) x[l] = src[i * R + l];
#pragma unroll
        for (int j = 0; j < R; ++j) {
            double acc = 0.0;
#pragma unroll
            for (int l = 0; l <= j; ++l) acc += x[l] * t[j][l];
            if (dst) dst[i * R + j] = acc;
            if (dst_f) dst_f[i * R + j] = (float)acc;
        }
    }
    __syncthreads();
}

__device__ void right_mul(const double *src, const double *T, int64_t m, int r, double *dst, float *dst_f) {
    switch (r) {
        case 1: right_mul_rows<1>(src, T, m, dst, dst_f); return;
        case 2: right_mul_rows<2>(src, T, m, dst, dst_f); return;
        case 3: right_mul_rows<3>(src, T, m, dst, dst_f); return;
        case 4: right_mul_rows<4>(src, T, m, dst, dst_f); return;
        default: break;
    }
    // dst[i][j] = sum_{l <= j} src[i][l] T[j][l]: 4 rows x 4 columns per thread per item
    const int ncb = (r + 3) / 4;
    const int64_t nrb = (m + 3) / 4;
    for (int64_t item = threadIdx.x; item < nrb * ncb; item += kFactorThreads) {
        const int64_t i0 = (item / ncb) * 4;
        const int j0 = (int)(item % ncb) * 4;
        double acc[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
        const int lmax = min(r, j0 + 4);
        for (int l = 0; l < lmax; ++l) {
            double a[4], t[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) a[u] = i0 + u < m ? src[(i0 + u) * r + l] : 0.0;
#pragma unroll
            for (int v = 0; v < 4; ++v) t[v] = (j0 + v < r && l <= j0 + v) ? T[(int64_t)(j0 + v) * r + l] : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], t[v], acc[u][v]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                if (i0 + u >= m || j0 + v >= r) continue;
                const int64_t e = (i0 + u) * r + j0 + v;
                if (dst) dst[e] = acc[u][v];
                if (dst_f) dst_f[e] = (float)acc[u][v];
            }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kFactorThreads) k_factor(const MatDev *mats, int32_t *status, double col_tol,
                                                           int32_t *any_fb, int32_t epoch) {
    const MatDev &M = mats[blockIdx.x];
    if ((status[blockIdx.x] & 1) || M.fx) return;
    const int r = M.r;
    const int64_t m = M.m;
    const int tid = threadIdx.x;
    double *gram = M.fwork, *R = gram + r * r, *T1 = R + r * r, *T2 = T1 + r * r, *S = T2 + r * r;
    __shared__ double s_tmp[kFactorThreads];
    __shared__ double s_tol;
    int32_t *dead = M.dead;
    const bool pre = M.zmode && M.precond;
    if (!M.zmode && M.p_raw != M.p_part) {
        // P_raw = sum over column chunks, fixed order (a single chunk is P_raw itself)
        for (int64_t e = tid; e < m * r; e += kFactorThreads) {
            double acc = 0.0;
            for (int c = 0; c < M.nchunk1; ++c) acc += M.p_part[(int64_t)c * m * r + e];
            M.p_raw[e] = acc;
        }
    }
    for (int e = tid; e < r * r; e += kFactorThreads) {
        const int i = e / r, k = e % r;
        S[e] = pre ? M.precond[(int64_t)i * M.ld_s + k] : (i == k ? 1.0 : 0.0);
    }
    for (int j = tid; j < r; j += kFactorThreads) dead[j] = 0;
    __syncthreads();
    gram_pass(M.p_raw, m, r, gram, s_tmp);
    if (tid == 0) {
        // tolerance relative to ||P_orig||_F with P_raw = P_orig S (compressor.py:79)
        double fro2 = 0.0;
        if (pre) {
            for (int j = 0; j < r; ++j) {          // Sinv column j into T2 (scratch)
                for (int l = 0; l < r; ++l) T2[j * r + l] = 0.0;
                for (int l = j; l >= 0; --l) {
                    double v = (l == j) ? 1.0 : 0.0;
                    for (int q = l + 1; q <= j; ++q) v -= S[l * r + q] * T2[j * r + q];
                    T2[j * r + l] = v / S[l * r + l];
                }
            }
            for (int j = 0; j < r; ++j)
                for (int u = 0; u <= j; ++u)
                    for (int v = 0; v <= j; ++v) fro2 += T2[j * r + u] * gram[u * r + v] * T2[j * r + v];
        } else {
            for (int j = 0; j < r; ++j) fro2 += gram[j * r + j];
        }
        s_tol = col_tol * sqrt(fro2);
        for (int j = 0; j < r; ++j) T1[j] = S[j * r + j];   // column scales (P_orig norms = R_jj / S_jj)
    }
    __syncthreads();
    // scales must survive chol_dead (which uses R); copy to the tail of T2's region is not needed:
    // chol_dead reads scale[k] only at step k before R row k is written.
    double *scale = T2;  // reuse: T2 is free again
    for (int j = tid; j < r; j += kFactorThreads) scale[j] = T1[j];
    __syncthreads();
    chol_dead(gram, r, s_tol, scale, dead, R, true);
    // ||R||_F^2 and, after the inverse, ||R^{-1}||_F^2 by block reductions (R, T1 are zero
    // outside their triangles)
    auto block_sumsq = [&](const double *X) -> double {
        double a = 0.0;
        for (int e = tid; e < r * r; e += kFactorThreads) a += X[e] * X[e];
        a = warp_sum(a);
        if ((tid & 31) == 0) s_tmp[tid >> 5] = a;
        __syncthreads();
        double tot = 0.0;
        for (int w = 0; w < kFactorThreads / 32; ++w) tot += s_tmp[w];
        __syncthreads();
        return tot;
    };
    const double rn2 = block_sumsq(R);
    tri_inverse(R, dead, r, T1);
    const double tn2 = block_sumsq(T1);
    // one fp64 CholQR pass leaves P orthonormal to ~cond^2 * m * eps64: enough when cond(R) is
    // small (Z path: <= 64, which the Z trick needs anyway; otherwise <= 1000 -> < 1e-6)
    const double kappa = sqrt(rn2 * tn2);
    const bool single = kappa <= (M.zmode ? kKappaMax : 1000.0);
    if (M.zmode && !single && tid == 0) {
        atomicOr(status + blockIdx.x, 2);
        *any_fb = epoch;   // k_pass2 runs its tiles only if some matrix needs it this run
    }
    if (single) {
        right_mul(M.p_raw, T1, m, r, nullptr, M.p_out);
        for (int e = tid; e < r * r; e += kFactorThreads) M.tmat[e] = T1[e];
        __syncthreads();
    } else {
    // P1 = P_raw T1, then a second CholQR pass restores orthogonality to fp64 level
    right_mul(M.p_raw, T1, m, r, M.p_tmp, nullptr);
    gram_pass(M.p_tmp, m, r, gram, s_tmp);
    chol_dead(gram, r, 0.0, nullptr, dead, R, false);
    tri_inverse(R, dead, r, T2);
    right_mul(M.p_tmp, T2, m, r, nullptr, M.p_out);
    // T = T1 T2: P = P_raw T, and on the Z path Q = Z T
    for (int e = tid; e < r * r; e += kFactorThreads) {
        const int j = e / r, l = e % r;
        double a = 0.0;
        for (int i = l; i <= j; ++i) a += T1[(int64_t)i * r + l] * T2[(int64_t)j * r + i];
        M.tmat[(int64_t)j * r + l] = a;
    }
    __syncthreads();
    }
    if (pre) {
        // next preconditioner A = S T (dead columns restart from e_j)
        for (int e = tid; e < r * r; e += kFactorThreads) {
            const int i = e / r, j = e % r;
            double a = 0.0;
            if (dead[j]) {
                a = (i == j) ? 1.0 : 0.0;
            } else {
                for (int l = i; l <= j; ++l) a += S[i * r + l] * M.tmat[(int64_t)j * r + l];
            }
            M.precond[(int64_t)i * M.ld_s + j] = a;
        }
    }
}

// ------------------------------------------- multi-CTA factorisation (r >= 32)
// At wide ranks the O(m r^2) parts of CholQR(2) -- the Gram matrices and the
// right multiplications by the triangular transforms -- dominate, and one CTA
// per matrix leaves most SMs idle.  They run here as tiled fp64 GEMMs over many
// CTAs (64x64 output tiles, 4x4 per thread, fixed-order K-split reduction);
// the r x r work (Cholesky with dead-column detection, triangular inverse,
// conditioning) stays one CTA per matrix and reuses k_factor's routines.
//   k_fx_gram(pass)   Gram partials of P_raw (pass 1) or P_raw T1 (pass 2)
//   k_fx_chol1        gram -> R, T1 = R^-1, kappa -> fmode (1: single, 2: CholQR2)
//   k_fx_rmul(pass)   pass 1: P = P_raw T1 (fp32 p_out) or p_tmp = P_raw T1 (fp64)
//                     pass 2: P = p_tmp T2
//   k_fx_chol2        fmode 2: second Cholesky -> T2, tmat = T1 T2
struct FxTile {
    int32_t mat, split;
    int32_t i0, j0;        // Gram: output block origins; rmul: column block j0, row block in r0
    int64_t r0, r1;        // Gram: K (row) range; rmul: output row range
};

constexpr int kFxT = 64, kFxK = 16, kFxThreads = 256;
constexpr int kFxBig = 128;   // tile edge of the fp64 factorisation GEMMs at r >= 128

__device__ __forceinline__ bool fx_active(const MatDev &M, const int32_t *status, int mat, int pass) {
    if (status[mat] & 1) return false;
    return pass == 1 || *M.fmode == 2;
}

// fp64 register-blocked tile GEMMs of the multi-CTA factorisation: a TT x TT output tile
// per CTA (TT = 64 below rank 128, 128 above), 256 threads as 16 x 16, each thread
// RB x RB outputs at rows 2 ty + 32 u' + {0,1}, columns 2 tx + 32 v' + {0,1} (double2
// shared loads, conflict-free across the 16 tx lanes).  Every output's K sum runs in
// ascending k, so the result does not depend on TT.
template <int TT>
struct FxBlk {
    static constexpr int RB = TT / 16, RP = RB / 2;
};

// gpart[split][i][j] = sum_{k in split} X[k][i] X[k][j] for the upper tile (i0 <= j0)
template <int TT>
__global__ void __launch_bounds__(kFxThreads) k_fx_gram(const MatDev *mats, const FxTile *tiles, const int32_t *status,
                                                        int pass) {
    constexpr int RB = FxBlk<TT>::RB, RP = FxBlk<TT>::RP;
    const FxTile t = tiles[blockIdx.x];
    const MatDev &M = mats[t.mat];
    if (!fx_active(M, status, t.mat, pass)) return;
    const int r = M.r;
    const double *X = pass == 1 ? M.p_raw : M.p_tmp;
    __shared__ __align__(16) double As[kFxK][TT], Bs[kFxK][TT];
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    double acc[RB][RB] = {};
    for (int64_t k0 = t.r0; k0 < t.r1; k0 += kFxK) {
        for (int e = tid; e < kFxK * TT; e += kFxThreads) {
            const int kk = e / TT, c = e % TT;
            const int64_t k = k0 + kk;
            const bool kin = k < t.r1;
            As[kk][c] = (kin && t.i0 + c < r) ? X[k * r + t.i0 + c] : 0.0;
            Bs[kk][c] = (kin && t.j0 + c < r) ? X[k * r + t.j0 + c] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kFxK; ++kk) {
            double a[RB], b[RB];
#pragma unroll
            for (int u = 0; u < RP; ++u) {
                const double2 x = *reinterpret_cast<const double2 *>(&As[kk][2 * ty + 32 * u]);
                const double2 y = *reinterpret_cast<const double2 *>(&Bs[kk][2 * tx + 32 * u]);
                a[2 * u] = x.x; a[2 * u + 1] = x.y;
                b[2 * u] = y.x; b[2 * u + 1] = y.y;
            }
#pragma unroll
            for (int u = 0; u < RB; ++u)
#pragma unroll
                for (int v = 0; v < RB; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
        }
        __syncthreads();
    }
    double *G = M.gpart + (int64_t)t.split * r * r;
#pragma unroll
    for (int u = 0; u < RB; ++u)
#pragma unroll
        for (int v = 0; v < RB; ++v) {
            const int i = t.i0 + 2 * ty + 32 * (u / 2) + (u & 1), j = t.j0 + 2 * tx + 32 * (v / 2) + (v & 1);
            if (i < r && j < r) G[i * r + j] = acc[u][v];
        }
}

// gram (upper, mirrored) = fixed-order sum of the split partials
template <int NT>
__device__ void fx_gram_sum(const MatDev &M, double *gram) {
    const int r = M.r;
    for (int e = threadIdx.x; e < r * r; e += NT) {
        const int i = e / r, j = e % r;
        if (j < i) continue;
        // the tile holding (i, j) is upper by block: (i/64 <= j/64); entries below the
        // diagonal inside a diagonal block are computed too, use the upper one
        double a = 0.0;
        for (int c = 0; c < M.gsplit; ++c) a += M.gpart[(int64_t)c * r * r + e];
        gram[i * r + j] = a;
        gram[j * r + i] = a;
    }
    __syncthreads();
}

// the r x r work of the wide-rank factorisation: 16 warps per matrix (latency-bound chains)
constexpr int kCholThreads = 512;

__global__ void __launch_bounds__(kCholThreads) k_fx_chol1(const MatDev *mats, int32_t *status, double col_tol) {
    const MatDev &M = mats[blockIdx.x];
    if (!M.fx || (status[blockIdx.x] & 1)) return;
    const int r = M.r, tid = threadIdx.x;
    double *gram = M.fwork, *R = gram + r * r, *T1 = R + r * r;
    __shared__ double s_tmp[kCholThreads / 32];
    __shared__ double s_tol;
    int32_t *dead = M.dead;
    for (int j = tid; j < r; j += kCholThreads) dead[j] = 0;
    fx_gram_sum<kCholThreads>(M, gram);
    if (tid == 0) {
        double fro2 = 0.0;   // ||P_raw||_F^2 (compressor.py:79)
        for (int j = 0; j < r; ++j) fro2 += gram[j * r + j];
        s_tol = col_tol * sqrt(fro2);
    }
    __syncthreads();
    chol_dead<kCholThreads>(gram, r, s_tol, nullptr, dead, R, true);
    auto block_sumsq = [&](const double *X) -> double {
        double a = 0.0;
        for (int e = tid; e < r * r; e += kCholThreads) a += X[e] * X[e];
        a = warp_sum(a);
        if ((tid & 31) == 0) s_tmp[tid >> 5] = a;
        __syncthreads();
        double tot = 0.0;
        for (int w = 0; w < kCholThreads / 32; ++w) tot += s_tmp[w];
        __syncthreads();
        return tot;
    };
    const double rn2 = block_sumsq(R);
    tri_inverse<kCholThreads>(R, dead, r, T1);
    const double tn2 = block_sumsq(T1);
    const bool single = sqrt(rn2 * tn2) <= 1000.0;   // as k_factor (non-Z)
    if (single)
        for (int e = tid; e < r * r; e += kCholThreads) M.tmat[e] = T1[e];
    if (tid == 0) *M.fmode = single ? 1 : 2;
}

__global__ void __launch_bounds__(kCholThreads) k_fx_chol2(const MatDev *mats, const int32_t *status) {
    const MatDev &M = mats[blockIdx.x];
    if (!M.fx || (status[blockIdx.x] & 1) || *M.fmode != 2) return;
    const int r = M.r, tid = threadIdx.x;
    double *gram = M.fwork, *R = gram + r * r, *T1 = R + r * r, *T2 = T1 + r * r;
    fx_gram_sum<kCholThreads>(M, gram);
    chol_dead<kCholThreads>(gram, r, 0.0, nullptr, M.dead, R, false);
    tri_inverse<kCholThreads>(R, M.dead, r, T2);
    // T = T1 T2 (P = P_raw T)
    for (int e = tid; e < r * r; e += kCholThreads) {
        const int j = e / r, l = e % r;
        double a = 0.0;
        for (int i = l; i <= j; ++i) a += T1[(int64_t)i * r + l] * T2[(int64_t)j * r + i];
        M.tmat[(int64_t)j * r + l] = a;
    }
}

// Y[i][j] = sum_{l <= j} X[i][l] T(l, j), T column j at T[j*r + l] (upper triangular)
template <int TT>
__global__ void __launch_bounds__(kFxThreads) k_fx_rmul(const MatDev *mats, const FxTile *tiles, const int32_t *status,
                                                        int pass) {
    constexpr int RB = FxBlk<TT>::RB, RP = FxBlk<TT>::RP;
    const FxTile t = tiles[blockIdx.x];
    const MatDev &M = mats[t.mat];
    if (!fx_active(M, status, t.mat, pass)) return;
    const int r = M.r;
    const bool single = *M.fmode == 1;
    const double *X = pass == 1 ? M.p_raw : M.p_tmp;
    const double *T = M.fwork + (int64_t)(pass == 1 ? 2 : 3) * r * r;   // T1 or T2
    __shared__ __align__(16) double As[kFxK][TT], Bs[kFxK][TT];
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    double acc[RB][RB] = {};
    const int kend = min(r, t.j0 + TT);   // T upper: l <= j < j0 + TT
    for (int k0 = 0; k0 < kend; k0 += kFxK) {
        for (int e = tid; e < kFxK * TT; e += kFxThreads) {
            // A: rows r0.. x K (coalesced along K); B: K x columns j0..
            const int c = e / kFxK, kk = e % kFxK;
            const int k = k0 + kk;
            const int64_t i = t.r0 + c;
            As[kk][c] = (i < t.r1 && k < kend) ? X[i * r + k] : 0.0;
            const int j = t.j0 + c;
            Bs[kk][c] = (j < r && k <= j) ? T[(int64_t)j * r + k] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kFxK; ++kk) {
            double a[RB], b[RB];
#pragma unroll
            for (int u = 0; u < RP; ++u) {
                const double2 x = *reinterpret_cast<const double2 *>(&As[kk][2 * ty + 32 * u]);
                const double2 y = *reinterpret_cast<const double2 *>(&Bs[kk][2 * tx + 32 * u]);
                a[2 * u] = x.x; a[2 * u + 1] = x.y;
                b[2 * u] = y.x; b[2 * u + 1] = y.y;
            }
#pragma unroll
            for (int u = 0; u < RB; ++u)
#pragma unroll
                for (int v = 0; v < RB; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < RB; ++u)
#pragma unroll
        for (int v = 0; v < RB; ++v) {
            const int64_t i = t.r0 + 2 * ty + 32 * (u / 2) + (u & 1);
            const int j = t.j0 + 2 * tx + 32 * (v / 2) + (v & 1);
            if (i >= t.r1 || j >= r) continue;
            const double y = acc[u][v];
            if (pass == 1 && !single) M.p_tmp[i * r + j] = y;
            else M.p_out[i * r + j] = (float)y;
        }
}

// --------------------------------------------------------- wide-rank path
// r > 8 (and unaligned shapes): a 64x64x16 smem-tiled fp32 GEMM with strided
// operands and fp64 split-K partials, used for P_raw = w q_warm and
// Q = w^T P, plus a tiled error-feedback update w <- g + (w - p_res q_res^T).
struct GemmTile {
    int32_t mat, split;
    int64_t i0, j0;        // output tile origin
    int64_t k0, k1;        // K range of this split
};

constexpr int kGT = 64, kGK = 16, kGThreads = 256;

// op 0: P_raw partial (M = m, N = r, K = n):  A(i,k) = w[i*n + k], B(k,j) = q_warm[k*ld_q + j]
// op 1: Q partial     (M = n, N = r, K = m):  A(i,k) = w[k*n + i], B(k,j) = p_out[k*r + j]
// op 2: EF update     (M = m, N = n, K = r_res): C = p_res q_res^T; w <- g + (w - C)
template <int OP>
__global__ void __launch_bounds__(kGThreads) k_gemm(const MatDev *mats, const GemmTile *tiles, int32_t *status) {
    const GemmTile t = tiles[blockIdx.x];
    const MatDev &M = mats[t.mat];
    if (OP == 1) {
        const int st = status[t.mat];
        if ((st & 1) || (M.zmode && !(st & 2))) return;
    }
    const int64_t n = M.n, m = M.m;
    const int r = M.r, rres = M.r_res;
    const int64_t MM = OP == 0 ? m : (OP == 1 ? n : m);
    const int64_t NN = OP == 2 ? n : r;
    // P_raw and Q partials accumulate exact fp32 products in fp64: at high rank
    // P_raw can be ill-conditioned and its rounding is amplified by cond(R)
    typedef typename std::conditional<OP == 2, float, double>::type AccT;
    __shared__ float As[kGK][kGT + 4];
    __shared__ float Bs[kGK][kGT + 4];
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    AccT acc[4][4] = {};
    for (int64_t k0 = t.k0; k0 < t.k1; k0 += kGK) {
        // A tile: kGT rows x kGK cols
        for (int e = tid; e < kGT * kGK; e += kGThreads) {
            int ii, kk;
            if (OP == 1) { ii = e % kGT; kk = e / kGT; } else { kk = e % kGK; ii = e / kGK; }
            const int64_t gi = t.i0 + ii, gk = k0 + kk;
            float v = 0.f;
            if (gi < MM && gk < t.k1) {
                if (OP == 0) v = M.w[gi * n + gk];
                else if (OP == 1) v = M.w[gk * n + gi];
                else v = M.p_res[gi * rres + gk];
            }
            As[kk][ii] = v;
        }
        for (int e = tid; e < kGT * kGK; e += kGThreads) {
            const int jj = e % kGT, kk = e / kGT;
            const int64_t gj = t.j0 + jj, gk = k0 + kk;
            float v = 0.f;
            if (gj < NN && gk < t.k1) {
                if (OP == 0) v = M.q_warm[gk * M.ld_q + gj];
                else if (OP == 1) v = M.p_out[gk * r + gj];
                else v = M.q_res[gj * rres + gk];
            }
            Bs[kk][jj] = v;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kGK; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) { a[u] = As[kk][ty * 4 + u]; b[u] = Bs[kk][tx * 4 + u]; }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = (AccT)a[u] * (AccT)b[v] + acc[u][v];
        }
        __syncthreads();
    }
    bool bad = false;
    if (OP == 2 && M.al4) {
        // error-feedback epilogue, float4 rows: each thread's 4 columns are adjacent (n % 4 == 0)
        const int64_t gj = t.j0 + tx * 4;
        if (gj < NN) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t gi = t.i0 + ty * 4 + u;
                if (gi >= MM) continue;
                const float4 g4 = __ldcs(reinterpret_cast<const float4 *>(M.g + gi * M.ld_g + gj));
                float4 *wp = reinterpret_cast<float4 *>(M.w + gi * n + gj);
                const float4 w4 = __ldcs(wp);
                const float x0 = g4.x + (w4.x - (float)acc[u][0]), x1 = g4.y + (w4.y - (float)acc[u][1]);
                const float x2 = g4.z + (w4.z - (float)acc[u][2]), x3 = g4.w + (w4.w - (float)acc[u][3]);
                bad |= !(isfinite(x0) && isfinite(x1) && isfinite(x2) && isfinite(x3));
                __stcs(wp, make_float4(x0, x1, x2, x3));
            }
        }
        if (__syncthreads_or(bad) && tid == 0) atomicOr(status + t.mat, 1);
        return;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int64_t gi = t.i0 + ty * 4 + u, gj = t.j0 + tx * 4 + v;
            if (gi >= MM || gj >= NN) continue;
            if (OP == 0) {
                M.p_part[((int64_t)t.split * m + gi) * r + gj] = (double)acc[u][v];
            } else if (OP == 1) {
                M.q_part[((int64_t)t.split * n + gi) * r + gj] = (double)acc[u][v];
            } else {
                const float x = M.g[gi * M.ld_g + gj] + (M.w[gi * n + gj] - (float)acc[u][v]);
                bad |= !isfinite(x);
                M.w[gi * n + gj] = x;
            }
        }
    if (OP == 2 && __syncthreads_or(bad) && tid == 0) atomicOr(status + t.mat, 1);
}

// Skinny fp64-accumulating GEMMs of the wide path with the output tile matched
// to the rank: OP 0 P_raw partial = W[:, K-chunk] q_warm[K-chunk, :], OP 1 Q
// partial = W[K-chunk, :]^T P[K-chunk, :].  BM x BN outputs per CTA (BM * BN =
// 4096, 4x4 per thread); A staged as fp32, the small B tile pre-converted to fp64.
// EF update of the wide path on CUDA cores, w <- g + (w - p_res q_res^T), r_res <= RK: one
// 64 x 64 tile per CTA, 4 x 4 per thread.  The thread's g and w are requested first (float4,
// streaming), so their HBM latency overlaps the factor loads and the FMAs (k_gemm<2> loaded
// them after the products); the products are summed in the same order, so w is bit-identical.
template <int RK>
__global__ void __launch_bounds__(kGThreads) k_ef(const MatDev *mats, const GemmTile *tiles, int32_t *status) {
    constexpr int FV = kGT * RK / kGThreads;   // factor elements per thread and operand
    const GemmTile t = tiles[blockIdx.x];
    const MatDev &M = mats[t.mat];
    const int64_t n = M.n, m = M.m;
    const int rres = M.r_res;
    __shared__ __align__(16) float As[RK][kGT + 4];
    __shared__ __align__(16) float Bs[RK][kGT + 4];
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    // factor rows first (L2-resident, needed before the FMAs), then the streaming g and w
    float fa[FV], fb[FV];
#pragma unroll
    for (int u = 0; u < FV; ++u) {
        const int e = tid + u * kGThreads;
        const int ii = e / RK, k = e % RK;   // consecutive threads read one contiguous factor row
        const int64_t gi = t.i0 + ii, gjj = t.j0 + ii;
        fa[u] = (k < rres && gi < m) ? M.p_res[gi * rres + k] : 0.f;
        fb[u] = (k < rres && gjj < n) ? M.q_res[gjj * rres + k] : 0.f;
    }
    const int64_t gj = t.j0 + tx * 4;
    const bool v4 = M.al4 && gj < n;   // al4: n % 4 == 0, so the thread's 4 columns are in range
    float4 g4[4], w4[4];
    if (v4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t gi = t.i0 + ty * 4 + u;
            if (gi < m) {
                g4[u] = __ldcs(reinterpret_cast<const float4 *>(M.g + gi * M.ld_g + gj));
                w4[u] = __ldcs(reinterpret_cast<const float4 *>(M.w + gi * n + gj));
            }
        }
    }
#pragma unroll
    for (int u = 0; u < FV; ++u) {
        const int e = tid + u * kGThreads;
        As[e % RK][e / RK] = fa[u];
        Bs[e % RK][e / RK] = fb[u];
    }
    __syncthreads();
    float acc[4][4] = {};
#pragma unroll
    for (int k = 0; k < RK; ++k) {
        const float4 a4 = *reinterpret_cast<const float4 *>(&As[k][ty * 4]);
        const float4 b4 = *reinterpret_cast<const float4 *>(&Bs[k][tx * 4]);
        const float a[4] = {a4.x, a4.y, a4.z, a4.w}, b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] = a[u] * b[v] + acc[u][v];
    }
    bool bad = false;
    if (v4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t gi = t.i0 + ty * 4 + u;
            if (gi >= m) continue;
            const float x0 = g4[u].x + (w4[u].x - acc[u][0]), x1 = g4[u].y + (w4[u].y - acc[u][1]);
            const float x2 = g4[u].z + (w4[u].z - acc[u][2]), x3 = g4[u].w + (w4[u].w - acc[u][3]);
            bad |= !(isfinite(x0) && isfinite(x1) && isfinite(x2) && isfinite(x3));
            __stcs(reinterpret_cast<float4 *>(M.w + gi * n + gj), make_float4(x0, x1, x2, x3));
        }
    } else if (!M.al4) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int64_t gi = t.i0 + ty * 4 + u, gc = gj + v;
                if (gi >= m || gc >= n) continue;
                const float x = M.g[gi * M.ld_g + gc] + (M.w[gi * n + gc] - acc[u][v]);
                bad |= !isfinite(x);
                M.w[gi * n + gc] = x;
            }
    }
    if (__syncthreads_or(bad) && tid == 0) atomicOr(status + t.mat, 1);
}

// Skinny GEMMs of the 8 < r <= 32 path: P_raw partial (OP 0: M = m, N = r, K = n) and Q partial
// (OP 1: M = n, N = r, K = m).  BM x BN outputs per CTA, 4 x 4 per thread; K in 32-wide steps
// with the next step's w tile loaded into registers (float4, coalesced along the contiguous
// dimension) while the current one is multiplied from shared memory.  fp32 products are summed
// in fp32 over one K step and folded into fp64 accumulators (the tensor-core path accumulates
// 128-wide K chunks in fp32 the same way).
constexpr int kSkK = 32;
template <int OP, int BM>
constexpr int skinny_smem() { return 2 * (OP == 0 ? BM * (kSkK + 4) : kSkK * (BM + 4)) * (int)sizeof(float); }
// 4 x 4 register tile update acc[u][v] += a[u][c] b[v] (fp32 FMA per element, fixed order): on
// FFMA2 the columns go in pairs with a[u][c] as the broadcast scalar operand (same rounding per
// lane, half the FMA instructions)
#ifndef EDGC_SKINNY_FFMA2
#define EDGC_SKINNY_FFMA2 1
#endif
template <bool F2 = EDGC_SKINNY_FFMA2 != 0>
__device__ __forceinline__ void skinny_fma4x4(float (&acc)[4][4], const float (&a)[4][4], int c, const float4 b4) {
    if constexpr (F2) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const float2 lo = __ffma2_rn(make_float2(a[u][c], a[u][c]), make_float2(b4.x, b4.y),
                                     make_float2(acc[u][0], acc[u][1]));
        const float2 hi = __ffma2_rn(make_float2(a[u][c], a[u][c]), make_float2(b4.z, b4.w),
                                     make_float2(acc[u][2], acc[u][3]));
        acc[u][0] = lo.x; acc[u][1] = lo.y; acc[u][2] = hi.x; acc[u][3] = hi.y;
    }
    } else {
    const float b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(a[u][c], b[v], acc[u][v]);
    }
}

template <int OP, int BM, int BN>
__global__ void __launch_bounds__((BM / 4) * (BN / 4), 512 / ((BM / 4) * (BN / 4)))
k_skinny(const MatDev *mats, const GemmTile *tiles, int32_t *status) {
    constexpr int TX = BN / 4, NT = (BM / 4) * TX;   // 4 x 4 outputs per thread
    constexpr int kAV = BM * kSkK / 4 / NT;          // float4 of the w tile per thread
    const GemmTile t = tiles[blockIdx.x];
    const MatDev &M = mats[t.mat];
    if (OP == 1) {
        const int st = status[t.mat];
        if ((st & 1) || (M.zmode && !(st & 2))) return;
    }
    const int64_t n = M.n, m = M.m;
    const int r = M.r;
    const int64_t MM = OP == 0 ? m : n;
    const float *__restrict__ w = M.w;
    const float *__restrict__ bsrc = OP == 0 ? M.q_warm : M.p_out;
    const int64_t ldb = OP == 0 ? M.ld_q : r;
    // OP 0 keeps the w tile row-major (rows i, 32 k + 4 pad: float4 stores and loads conflict-free),
    // OP 1 k-major (rows k, BM i + 4 pad)
    constexpr int AR = OP == 0 ? BM : kSkK, AC = OP == 0 ? kSkK + 4 : BM + 4;
    constexpr int kBV = BN * kSkK / NT;        // q / P elements of one K step per thread
    extern __shared__ __align__(16) float sk_smem[];
    float (*As)[AR][AC] = reinterpret_cast<float (*)[AR][AC]>(sk_smem);   // two stages
    __shared__ __align__(16) float Bs[kSkK][BN + 4];
    const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
    // float4 e of the w tile: OP 0 rows i (contiguous along k): e -> (row e / 8, k quad e % 8);
    // OP 1 rows k (contiguous along i): e -> (k e / (BM/4), i quad e % (BM/4)).  Copied with
    // cp.async into the stage not being multiplied (no registers held across the multiply).
    const bool vec = (n % 4 == 0) && ((uintptr_t)w % 16 == 0);
    auto issue_a = [&](int64_t k0, int buf) {
#pragma unroll
        for (int u = 0; u < kAV; ++u) {
            const int e = tid + u * NT;
            int ii, kk;
            int64_t gi, gk;
            if (OP == 0) { ii = e / (kSkK / 4); kk = 4 * (e % (kSkK / 4)); }
            else { kk = e / (BM / 4); ii = 4 * (e % (BM / 4)); }
            gi = t.i0 + ii; gk = k0 + kk;
            float *dst = OP == 0 ? &As[buf][ii][kk] : &As[buf][kk][ii];
            const bool in = OP == 0 ? gi < MM : gk < t.k1;
            const int64_t lim = OP == 0 ? t.k1 - gk : MM - gi;   // valid of the 4 contiguous
            const float *src = OP == 0 ? w + gi * n + gk : w + gk * n + gi;
            if (vec && in && lim >= 4) {
                tc::cp_async16(dst, src);
            } else {
#pragma unroll
                for (int c = 0; c < 4; ++c) dst[c] = (in && c < lim) ? src[c] : 0.f;
            }
        }
        tc::cp_async_commit();
    };
    auto load_b = [&](int64_t k0, float (&b)[kBV]) {
#pragma unroll
        for (int u = 0; u < kBV; ++u) {
            const int e = tid + u * NT;
            const int64_t gj = t.j0 + e % BN, gk = k0 + e / BN;
            b[u] = (gj < r && gk < t.k1) ? bsrc[gk * ldb + gj] : 0.f;
        }
    };
    double acc[4][4] = {};
    float b_next[kBV];
    issue_a(t.k0, 0);
    load_b(t.k0, b_next);
    int buf = 0;
    for (int64_t k0 = t.k0; k0 < t.k1; k0 += kSkK, buf ^= 1) {
        const bool more = k0 + kSkK < t.k1;
        if (more) issue_a(k0 + kSkK, buf ^ 1);   // next step's tile in flight during the multiply
#pragma unroll
        for (int u = 0; u < kBV; ++u) {
            const int e = tid + u * NT;
            Bs[e / BN][e % BN] = b_next[u];
        }
        if (more) tc::cp_async_wait<1>();
        else tc::cp_async_wait<0>();
        __syncthreads();
        if (more) load_b(k0 + kSkK, b_next);
        float accf[4][4] = {};
#pragma unroll
        for (int k4 = 0; k4 < kSkK; k4 += 4) {
            float a[4][4];   // a[u][c]: row ty*4+u, k k4+c
            if (OP == 0) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {   // rows ty + u BM/4: 8 rows of a warp on distinct banks
                    const float4 x = *reinterpret_cast<const float4 *>(&As[buf][ty + u * (BM / 4)][k4]);
                    a[u][0] = x.x; a[u][1] = x.y; a[u][2] = x.z; a[u][3] = x.w;
                }
            } else {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float4 x = *reinterpret_cast<const float4 *>(&As[buf][k4 + c][ty * 4]);
                    a[0][c] = x.x; a[1][c] = x.y; a[2][c] = x.z; a[3][c] = x.w;
                }
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float4 b4 = *reinterpret_cast<const float4 *>(&Bs[k4 + c][tx * 4]);
                skinny_fma4x4(accf, a, c, b4);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] += (double)accf[u][v];
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int64_t gi = t.i0 + (OP == 0 ? ty + u * (BM / 4) : ty * 4 + u), gj = t.j0 + tx * 4 + v;
            if (gi >= MM || gj >= r) continue;
            if (OP == 0) M.p_part[((int64_t)t.split * m + gi) * r + gj] = acc[u][v];
            else M.q_part[((int64_t)t.split * n + gi) * r + gj] = acc[u][v];
        }
}

// P_raw partials with the EF update fused in (4 < r <= 16, r_res <= BN, float4-aligned rows):
// the K step's g and w tiles arrive together by cp.async, the step first applies
// w <- g + (w - p_res q_resᵀ) in shared memory -- each thread 4-row x 4-column blocks,
// products summed over s ascending exactly as k_ef, so w is bit-identical -- streams the
// new w back to HBM, and then multiplies it into the P_raw partials as k_skinny<0> does.
// One pass over w instead of two (12 B/elem for EF + P_raw instead of 16).
// rows per fused CTA: 64, the product split over KS thread groups (KS = 4 for 8-rank blocks,
// 2 for 16: 128 threads, 128 registers, 4 CTAs per SM).  Measured (GPT2-2.5B, pass 1 per step):
// r = 8 7.2 -> 5.6 ms (785 -> 901 GB/s; KS = 1 / 2 / 4: 9.4 / 5.9 / 5.6 ms, 96 registers at
// 5 CTAs per SM 8.1 ms), r = 16 7.6 -> 7.1 ms (128 rows: KS = 1 / 2 7.6 / 7.4 ms).
#ifndef EDGC_SKEF_ROWS16
#define EDGC_SKEF_ROWS16 64
#endif
constexpr int kSkEfRows8 = 64, kSkEfRows16 = EDGC_SKEF_ROWS16;
#ifndef EDGC_SKEF_KS8
#define EDGC_SKEF_KS8 4
#endif
#ifndef EDGC_SKEF_KS16
#define EDGC_SKEF_KS16 2
#endif
#ifndef EDGC_SKEF_KS32
#define EDGC_SKEF_KS32 1
#endif
constexpr int kSkEfKS8 = EDGC_SKEF_KS8, kSkEfKS16 = EDGC_SKEF_KS16;   // product K-split (k_skinny_ef)
constexpr int kSkEfKS32 = EDGC_SKEF_KS32, kSkEfRows32 = 64;
#ifndef EDGC_SKEF32_DEFAULT
#define EDGC_SKEF32_DEFAULT 1
#endif
constexpr bool kSkEf32Default = EDGC_SKEF32_DEFAULT != 0;
// Q partials (k_skinny<1>) rows (columns j of w) per CTA
#ifndef EDGC_SKQ_ROWS8
#define EDGC_SKQ_ROWS8 256
#endif
#ifndef EDGC_SKQ_ROWS16
#define EDGC_SKQ_ROWS16 128   // measured r = 16: 128 / 256 / 512 rows 656 / 647 / 619 GB/s; r = 8 best at 256
#endif
#ifndef EDGC_SKQ_ROWS32
#define EDGC_SKQ_ROWS32 128   // measured r = 32 pass 2: 64 / 128 / 256 rows 4.50 / 4.53 / 5.42 ms
#endif
constexpr int kSkQRows8 = EDGC_SKQ_ROWS8, kSkQRows16 = EDGC_SKQ_ROWS16, kSkQRows32 = EDGC_SKQ_ROWS32;
#ifndef EDGC_SKQ_K
#define EDGC_SKQ_K 1024
#endif
// K (rows of w) per skinny Q tile = one fp64 partial [n][r] per block: 256 / 512 / 1024 / 2048 rows
// measured (GPT2-2.5B, pass 2 + finalize): r = 8 2.16 / 1.92 / 1.86 / 1.87 ms, r = 16 3.03 / 2.74 /
// 2.61 / 2.57, r = 32 5.70 / 5.10 / 4.81 / 4.69 (fewer fp64 partials to write and sum)
constexpr int kSkQK = EDGC_SKQ_K;
template <int BM, int BN>
struct SkEfSmem {
    float a[2][BM][kSkK + 4];   // w -> x (new w) per stage
    float g[2][BM][kSkK + 4];
    float pt[BN][BM + 4];       // p_res rows of the CTA, transposed
    float qt[BN][kSkK + 4];     // q_res rows of the K step, transposed
    float b[kSkK][BN + 4];      // q_warm rows of the K step
};
// KS: K-split of the product -- KS thread groups each multiply kSkK / KS columns of the step
// into their own 4 x 4 register tiles (fp32 per step, folded into fp64), summed group by group
// in fixed order at the end.  KS = 4 at 8-rank blocks: 128 threads per 64-row CTA instead of 32
// (measured: 255 registers and 1.25 warps per scheduler at KS = 1, DRAM 50% -- latency bound).
#ifndef EDGC_SKEF_THREADS_SM
#define EDGC_SKEF_THREADS_SM 512   // K-split CTAs: registers capped for this many threads per SM (128 each)
#endif
// 16-rank blocks: 4 CTAs per SM on FFMA measured best (3 CTAs at 168 registers, with or without
// FFMA2: r = 16 pass 1 7.12 -> 7.45 ms; tools/probe_skef16.sh)
#ifndef EDGC_SKEF16_THREADS_SM
#define EDGC_SKEF16_THREADS_SM 512
#endif
// FFMA2 at 16-rank blocks: bit 0 the product tiles (they spill at the 128-register cap: pass 1
// 7.2 -> 7.6 ms), bit 1 the EF blocks (7.2 -> 7.1 ms at r = 16, 6.80 -> 6.73 at r = 12)
#ifndef EDGC_SKEF16_FFMA2
#define EDGC_SKEF16_FFMA2 2
#endif
#ifndef EDGC_SKEF32_THREADS_SM
#define EDGC_SKEF32_THREADS_SM 384   // 64 x 32 tiles: 3 CTAs per SM at 168 registers (4 at 128 spill: 14.97 vs 11.65 ms at r = 32)
#endif
template <int BM, int BN, int KS>
__global__ void __launch_bounds__((BM / 4) * (BN / 4) * KS,
                                  BN > 16 ? EDGC_SKEF32_THREADS_SM / ((BM / 4) * (BN / 4) * KS)
                                  : BN == 16 ? EDGC_SKEF16_THREADS_SM / ((BM / 4) * (BN / 4) * KS)
                                  : KS > 1 ? EDGC_SKEF_THREADS_SM / ((BM / 4) * (BN / 4) * KS) : 1)
k_skinny_ef(const MatDev *mats, const GemmTile *tiles, int32_t *status) {
    constexpr int TX = BN / 4, NG = (BM / 4) * TX, NT = NG * KS;
    constexpr int kAV = BM * kSkK / 4 / NT;          // float4 of one tile per thread
    constexpr int kBV = BN * kSkK / NT;               // q_warm / q_res elements of one K step per thread
    constexpr int kCB = kSkK / 4;                     // 4-column EF blocks per row block
    constexpr int kEB = (BM / 4) * kCB / NT;          // 4 x 4 EF blocks per thread
    constexpr int kKG = kSkK / KS;                    // product columns per group and step
    static_assert(kAV >= 1 && kBV >= 1 && kEB >= 1 && kKG % 4 == 0, "skinny EF thread layout");
    // FFMA2 tiles except at 16-rank blocks (there they spill at the 128-register cap: measured
    // r = 16 pass 1 7.05 -> 8.19 ms; r = 8 / 32 gain 2%)
    constexpr bool kF2 = EDGC_SKINNY_FFMA2 != 0 && (BN != 16 || (EDGC_SKEF16_FFMA2 & 1) != 0);   // product tiles
    constexpr bool kF2E = EDGC_SKINNY_FFMA2 != 0 && (BN != 16 || (EDGC_SKEF16_FFMA2 & 2) != 0);  // EF blocks
    static_assert(KS * BM * BN * (int)sizeof(double) <= (int)sizeof(float) * 2 * BM * (kSkK + 4),
                  "K-split partials reuse the w stages");
    extern __shared__ __align__(16) unsigned char skef_raw[];
    SkEfSmem<BM, BN> &S = *reinterpret_cast<SkEfSmem<BM, BN> *>(skef_raw);
    const GemmTile t = tiles[blockIdx.x];
    const MatDev &M = mats[t.mat];
    const int64_t n = M.n, m = M.m, ldg = M.ld_g;
    const int r = M.r, rres = M.r_res;
    float *__restrict__ w = M.w;
    const float *__restrict__ g = M.g;
    const int tid = threadIdx.x, kg = tid / NG, tx = (tid % NG) % TX, ty = (tid % NG) / TX;
    for (int e = tid; e < BN * BM; e += NT) {
        const int s = e / BM, ii = e % BM;
        const int64_t gi = t.i0 + ii;
        S.pt[s][ii] = (s < rres && gi < m) ? M.p_res[gi * rres + s] : 0.f;
    }
    auto issue = [&](int64_t k0, int buf) {
#pragma unroll
        for (int u = 0; u < kAV; ++u) {
            const int e = tid + u * NT;
            const int ii = e / (kSkK / 4), kk = 4 * (e % (kSkK / 4));
            const int64_t gi = t.i0 + ii, gk = k0 + kk;
            if (gi < m && gk + 4 <= t.k1) {   // rows are float4-aligned and K chunks multiples of 4
                tc::cp_async16(&S.a[buf][ii][kk], w + gi * n + gk);
                tc::cp_async16(&S.g[buf][ii][kk], g + gi * ldg + gk);
            } else {
                *reinterpret_cast<float4 *>(&S.a[buf][ii][kk]) = make_float4(0.f, 0.f, 0.f, 0.f);
                *reinterpret_cast<float4 *>(&S.g[buf][ii][kk]) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        tc::cp_async_commit();
    };
    auto load_b = [&](int64_t k0, float (&b)[kBV], float (&q)[kBV]) {
#pragma unroll
        for (int u = 0; u < kBV; ++u) {
            const int e = tid + u * NT;
            const int64_t gj = t.j0 + e % BN, gk = k0 + e / BN;
            b[u] = (gj < r && gk < t.k1) ? M.q_warm[gk * M.ld_q + gj] : 0.f;
            const int s = e % BN;
            q[u] = (s < rres && gk < t.k1) ? M.q_res[gk * rres + s] : 0.f;
        }
    };
    double acc[4][4] = {};
    float b_next[kBV], q_next[kBV];
    issue(t.k0, 0);
    load_b(t.k0, b_next, q_next);
    bool bad = false;
    int buf = 0;
    for (int64_t k0 = t.k0; k0 < t.k1; k0 += kSkK, buf ^= 1) {
        const bool more = k0 + kSkK < t.k1;
        if (more) issue(k0 + kSkK, buf ^ 1);
#pragma unroll
        for (int u = 0; u < kBV; ++u) {
            const int e = tid + u * NT;
            S.b[e / BN][e % BN] = b_next[u];
            S.qt[e % BN][e / BN] = q_next[u];
        }
        if (more) tc::cp_async_wait<1>();
        else tc::cp_async_wait<0>();
        __syncthreads();
        if (more) load_b(k0 + kSkK, b_next, q_next);
        // EF on the tile: block (rows 4 rb .. +3, columns 4 cb .. +3); a quarter warp covers
        // one row's 8 blocks (128 contiguous bytes)
#pragma unroll
        for (int eb = 0; eb < kEB; ++eb) {
            const int bid = tid + eb * NT, rb = bid / kCB, cb = bid % kCB;
            float c[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) c[u][v] = 0.f;
            for (int s2 = 0; s2 < rres; ++s2) {
                const float4 a4 = *reinterpret_cast<const float4 *>(&S.pt[s2][rb * 4]);
                const float4 q4 = *reinterpret_cast<const float4 *>(&S.qt[s2][cb * 4]);
                const float a[4] = {a4.x, a4.y, a4.z, a4.w};
                if constexpr (kF2E) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float2 lo = __ffma2_rn(make_float2(a[u], a[u]), make_float2(q4.x, q4.y),
                                                 make_float2(c[u][0], c[u][1]));
                    const float2 hi = __ffma2_rn(make_float2(a[u], a[u]), make_float2(q4.z, q4.w),
                                                 make_float2(c[u][2], c[u][3]));
                    c[u][0] = lo.x; c[u][1] = lo.y; c[u][2] = hi.x; c[u][3] = hi.y;
                }
                } else {
                const float q[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) c[u][v] = a[u] * q[v] + c[u][v];
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int ii = rb * 4 + u;
                const int64_t gi = t.i0 + ii, gk = k0 + cb * 4;
                float4 *ap = reinterpret_cast<float4 *>(&S.a[buf][ii][cb * 4]);
                const float4 w4 = *ap;
                const float4 g4 = *reinterpret_cast<const float4 *>(&S.g[buf][ii][cb * 4]);
                const float x0 = g4.x + (w4.x - c[u][0]), x1 = g4.y + (w4.y - c[u][1]);
                const float x2 = g4.z + (w4.z - c[u][2]), x3 = g4.w + (w4.w - c[u][3]);
                const float4 x = make_float4(x0, x1, x2, x3);
                *ap = x;
                if (gi < m && gk + 4 <= t.k1) {
                    bad |= !(isfinite(x0) && isfinite(x1) && isfinite(x2) && isfinite(x3));
                    __stcs(reinterpret_cast<float4 *>(w + gi * n + gk), x);
                }
            }
        }
        __syncthreads();
        float accf[4][4] = {};
#pragma unroll
        for (int k4 = kg * kKG; k4 < (kg + 1) * kKG; k4 += 4) {
            float a[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {   // rows ty + u BM/4: 8 rows of a warp on distinct banks
                const float4 x = *reinterpret_cast<const float4 *>(&S.a[buf][ty + u * (BM / 4)][k4]);
                a[u][0] = x.x; a[u][1] = x.y; a[u][2] = x.z; a[u][3] = x.w;
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float4 b4 = *reinterpret_cast<const float4 *>(&S.b[k4 + c][tx * 4]);
                skinny_fma4x4<kF2>(accf, a, c, b4);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] += (double)accf[u][v];
        __syncthreads();
    }
    if (KS > 1) {
        // group partials through the (now idle) w stages, summed in group order
        double *red = reinterpret_cast<double *>(&S.a[0][0][0]);   // [KS][BM][BN]
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) red[((int64_t)kg * BM + ty + u * (BM / 4)) * BN + tx * 4 + v] = acc[u][v];
        __syncthreads();
        if (kg == 0) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    double sum = 0.0;
#pragma unroll
                    for (int h = 0; h < KS; ++h) sum += red[((int64_t)h * BM + ty + u * (BM / 4)) * BN + tx * 4 + v];
                    acc[u][v] = sum;
                }
        }
    }
    if (kg == 0) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int64_t gi = t.i0 + ty + u * (BM / 4), gj = t.j0 + tx * 4 + v;
                if (gi >= m || gj >= r) continue;
                M.p_part[((int64_t)t.split * m + gi) * r + gj] = acc[u][v];
            }
    }
    if (__syncthreads_or(bad) && tid == 0) atomicOr(status + t.mat, 1);
}

// cudaFuncSetAttribute applies to the current device: remember which devices have it
template <typename K>
int smem_attr_once(K kernel, int bytes, uint64_t &done_mask) {
    int dev = 0;
    EDGC_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 64 && (done_mask >> dev & 1)) return EDGC_OK;
    EDGC_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    if (dev < 64) done_mask |= 1ull << dev;
    return EDGC_OK;
}

template <int OP, int BM, int BN>
int launch_skinny(unsigned grid, cudaStream_t st, const MatDev *mats, const GemmTile *tiles, int32_t *status) {
    static uint64_t attr = 0;
    const int rc = smem_attr_once(k_skinny<OP, BM, BN>, skinny_smem<OP, BM>(), attr);
    if (rc != EDGC_OK) return rc;
    k_skinny<OP, BM, BN><<<grid, (BM / 4) * (BN / 4), skinny_smem<OP, BM>(), st>>>(mats, tiles, status);
    return EDGC_OK;
}

template <int BM, int BN, int KS>
int launch_skinny_ef(unsigned grid, cudaStream_t st, const MatDev *mats, const GemmTile *tiles, int32_t *status) {
    static uint64_t attr = 0;
    const int rc = smem_attr_once(k_skinny_ef<BM, BN, KS>, (int)sizeof(SkEfSmem<BM, BN>), attr);
    if (rc != EDGC_OK) return rc;
    k_skinny_ef<BM, BN, KS><<<grid, (BM / 4) * (BN / 4) * KS, sizeof(SkEfSmem<BM, BN>), st>>>(mats, tiles, status);
    return EDGC_OK;
}

// ------------------------------------------------- wide path on tcgen05
// Above kTcMinRank the wide-path contractions run on the tensor cores
// (tc_gemm.cuh: 3xTF32 operands, fp32 accumulation in 128-K chunks folded
// round-to-nearest; ~1e-6 relative error against an exact product):
//   TcPraw  P_raw = w q_warm      (M = m, N = r, K = n; one fp64 partial)
//   TcQ     Q = w^T P             (M = n, N = r, K = m; one fp64 partial)
//   TcEF    w <- g + (w - p_res q_res^T)   (M = m, N = n, K = r_res)
// The fp64 partial layouts are the CUDA-core path's with a single K split, so
// the factorisation and finalize kernels are shared.
// number of epilogue items u (rows row0 + 4u) inside the problem, rem = rows left from row0
__device__ __forceinline__ int tc_rows4(int64_t rem) { return rem <= 0 ? 0 : rem >= 29 ? 8 : (int)((rem + 3) / 4); }

struct TcPraw {
    static constexpr bool kAMN = false, kBMN = true;
    static constexpr int kPF = 0, kPFDepth = 2, kStages = 0;
    using Tile = GemmTile;
    const MatDev *mats;
    const GemmTile *tiles;
    int ntiles;
    __device__ Tile tile(int i) const { return tiles[i]; }
    __device__ int64_t tile_k(const Tile &t) const { return t.k1 - t.k0; }
    __device__ void views(const Tile &t, tc::View &a, tc::View &b) const {
        const MatDev &M = mats[t.mat];
        a = tc::View{M.w + t.i0 * M.n + t.k0, M.n, M.m - t.i0, t.k1 - t.k0, 0, 0};
        b = tc::View{M.q_warm + t.k0 * M.ld_q + t.j0, M.ld_q, M.r - t.j0, t.k1 - t.k0, 0, 0};
    }
    __device__ void prefetch(const Tile &, int, int, uint8_t *) const {}
    __device__ void epilogue(const Tile &t, int row0, int col, const float4 (&v)[8], const uint8_t *) const {
        const MatDev &M = mats[t.mat];
        const int nc = M.r - (int)t.j0 - col;
        if (nc <= 0) return;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t gi = t.i0 + row0 + 4 * u;
            if (gi >= M.m) break;
            double *dst = M.p_part + ((int64_t)t.split * M.m + gi) * M.r + t.j0 + col;
            dst[0] = v[u].x;
            if (nc > 1) dst[1] = v[u].y;
            if (nc > 2) dst[2] = v[u].z;
            if (nc > 3) dst[3] = v[u].w;
        }
    }
};

struct TcQ {
    static constexpr bool kAMN = true, kBMN = true;
    static constexpr int kPF = 0, kPFDepth = 2, kStages = 0;
    using Tile = GemmTile;
    const MatDev *mats;
    const GemmTile *tiles;
    const int32_t *status;
    int ntiles;
    __device__ Tile tile(int i) const { return tiles[i]; }
    __device__ int64_t tile_k(const Tile &t) const {
        const int st = status[t.mat];
        if ((st & 1) || (mats[t.mat].zmode && !(st & 2))) return 0;   // diverged / Z path done
        return t.k1 - t.k0;
    }
    __device__ void views(const Tile &t, tc::View &a, tc::View &b) const {
        const MatDev &M = mats[t.mat];
        a = tc::View{M.w + t.k0 * M.n + t.i0, M.n, M.n - t.i0, t.k1 - t.k0, 0, 0};
        b = tc::View{M.p_out + t.k0 * M.r + t.j0, M.r, M.r - t.j0, t.k1 - t.k0, 0, 0};
    }
    __device__ void prefetch(const Tile &, int, int, uint8_t *) const {}
    __device__ void epilogue(const Tile &t, int row0, int col, const float4 (&v)[8], const uint8_t *) const {
        const MatDev &M = mats[t.mat];
        const int nc = M.r - (int)t.j0 - col;
        if (nc <= 0) return;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t gi = t.i0 + row0 + 4 * u;
            if (gi >= M.n) break;
            double *dst = M.q_part + ((int64_t)t.split * M.n + gi) * M.r + t.j0 + col;
            dst[0] = v[u].x;
            if (nc > 1) dst[1] = v[u].y;
            if (nc > 2) dst[2] = v[u].z;
            if (nc > 3) dst[3] = v[u].w;
        }
    }
};

#ifndef EDGC_EF_DIAG
#define EDGC_EF_DIAG 0   // diagnostics (wrong results): 1 = no g / w loads, 2 = no w stores
#endif
// TcEF tile width (measured: 64 columns with a 3-slice g / w prefetch ring is slower,
// 13.6 vs 11.0 ms at r = 128)
constexpr int kTcEFN = 128;

// PFD - 1 slices of g and w prefetched ahead; STAGES operand stages.  Up to r_res = 128 (K of at
// most four 32-wide blocks) one stage and three slot buffers (the operands p_res, q_res are small);
// above, the earlier two stages and two buffers (measured: r = 32 375 -> 388 GB/s with the first,
// GPT2-12.1B at r = 256 166 vs 162 GB/s with the second)
template <int PFD, int STAGES>
struct TcEFT {
    static constexpr bool kAMN = false, kBMN = false;
    static constexpr int kPF = 16, kPFDepth = PFD, kStages = STAGES;
    using Tile = GemmTile;
    const MatDev *mats;
    const GemmTile *tiles;
    int32_t *status;
    int ntiles;
    __device__ Tile tile(int i) const { return tiles[i]; }
    __device__ int64_t tile_k(const Tile &t) const { return t.k1 - t.k0; }
    __device__ void views(const Tile &t, tc::View &a, tc::View &b) const {
        const MatDev &M = mats[t.mat];
        const int rr = M.r_res;
        a = tc::View{M.p_res + t.i0 * rr, rr, M.m - t.i0, rr, 0, 0};
        b = tc::View{M.q_res + t.j0 * rr, rr, M.n - t.j0, rr, 0, 0};
    }
    __device__ void prefetch(const Tile &t, int row0, int col, uint8_t *dst) const {
        const MatDev &M = mats[t.mat];
        const int64_t j = t.j0 + col;
        if (!M.al4 || j >= M.n || EDGC_EF_DIAG == 1) return;
        const int nu = tc_rows4(M.m - t.i0 - row0);
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (u < nu) {
                const int64_t gi = t.i0 + row0 + 4 * u;
                tc::cp_async16(dst + u * 2048, M.g + gi * M.ld_g + j);
                tc::cp_async16(dst + (8 + u) * 2048, M.w + gi * M.n + j);
            }
    }
    __device__ void epilogue(const Tile &t, int row0, int col, const float4 (&v)[8], const uint8_t *pf) const {
        const MatDev &M = mats[t.mat];
        const int64_t j = t.j0 + col;
        if (j >= M.n) return;
        const int nu = tc_rows4(M.m - t.i0 - row0);   // rows row0 + 4u < m
        bool bad = false;
        if (M.al4) {
            // g and w arrived through the prefetch slots
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (u < nu) {
                    const int64_t gi = t.i0 + row0 + 4 * u;
                    const float4 g4 = ptx::ld_shared_v4(pf + u * 2048), w4 = ptx::ld_shared_v4(pf + (8 + u) * 2048);
                    const float x0 = g4.x + (w4.x - v[u].x), x1 = g4.y + (w4.y - v[u].y);
                    const float x2 = g4.z + (w4.z - v[u].z), x3 = g4.w + (w4.w - v[u].w);
                    bad |= !(isfinite(x0) && isfinite(x1) && isfinite(x2) && isfinite(x3));
                    if (EDGC_EF_DIAG != 2)
                        __stcs(reinterpret_cast<float4 *>(M.w + gi * M.n + j), make_float4(x0, x1, x2, x3));
                }
        } else {
            const int nc = M.n - j < 4 ? (int)(M.n - j) : 4;
            // static u: a dynamic index into v[] would put the slice in local memory
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (u >= nu) break;
                const int64_t gi = t.i0 + row0 + 4 * u;
                const float *g = M.g + gi * M.ld_g + j;
                float *w = M.w + gi * M.n + j;
                for (int c = 0; c < nc; ++c) {
                    const float a = c == 0 ? v[u].x : c == 1 ? v[u].y : c == 2 ? v[u].z : v[u].w;
                    const float x = g[c] + (w[c] - a);
                    bad |= !isfinite(x);
                    w[c] = x;
                }
            }
        }
        if (bad) atomicOr(status + t.mat, 1);
    }
};
using TcEF = TcEFT<EDGC_TCEF_PFD, EDGC_TCEF_STAGES>;   // r_res <= 128
using TcEFWide = TcEFT<2, 0>;

// EDGC_TC_MIN_RANK (default 16): wide-path ranks above it use the tensor cores;
// EDGC_NO_TC disables them (A/B runs)
// averaged reconstruction on the tensor cores from this W r on (EDGC_TC_RECON_MIN)
int tc_recon_min() {
    static const int v = [] {
        if (std::getenv("EDGC_NO_TC")) return 1 << 30;
        const char *e = std::getenv("EDGC_TC_RECON_MIN");
        return e ? std::atoi(e) : 33;
    }();
    return v;
}

// EDGC_NARROW_MAX (4..kNarrow, default 4): largest rank on the register-tiled passes.  Ranks 5..8
// measured faster on the skinny GEMMs (GPT2-2.5B set, r = 6: 548 -> 629 GB/s, r = 8: 481 -> 604
// with 256 x 16 tiles): the narrow pass 1 holds 8 ranks per thread at 25% occupancy
int narrow_max() {
    static const int v = [] {
        const char *e = std::getenv("EDGC_NARROW_MAX");
        return e ? std::max(4, std::min(kNarrow, std::atoi(e))) : 4;
    }();
    return v;
}

// EDGC_TC_EF_MIN_RANK (default EDGC_TC_MIN_RANK): the EF update uses the tensor cores above it
int tc_ef_min_rank();

// EDGC_SKINNY_EF_OFF: keep the EF update of 4 < r <= 16 as its own pass (k_ef) instead of fused
// into the P_raw partials
bool skef_off() {
    static const bool v = std::getenv("EDGC_SKINNY_EF_OFF") != nullptr;
    return v;
}

// Ranks 16 < r <= 32 also take the fused CUDA-core EF + P_raw pass (64 x 32 tiles) instead of
// the tcgen05 TcEF + TcPraw pair, with the multi-CTA factorisation (EDGC_SKEF32=0: tensor cores).
// Measured on the GPT2-2.5B set: pass 1 at r = 24 12.3 -> 10.5 ms (410 -> 439 GB/s), r = 32
// 12.4 -> 11.6 ms (393 -> 403 GB/s)
bool skef32() {
    static const bool v = [] {
        const char *e = std::getenv("EDGC_SKEF32");
        return e ? std::atoi(e) != 0 : kSkEf32Default;
    }();
    return v && !skef_off();
}

int tc_min_rank() {
    static const int v = [] {
        if (std::getenv("EDGC_NO_TC")) return 1 << 30;
        const char *e = std::getenv("EDGC_TC_MIN_RANK");
        return e ? std::atoi(e) : 16;
    }();
    return v;
}

int tc_ef_min_rank() {
    static const int v = [] {
        if (std::getenv("EDGC_NO_TC")) return 1 << 30;
        const char *e = std::getenv("EDGC_TC_EF_MIN_RANK");
        return e ? std::atoi(e) : tc_min_rank();
    }();
    return v;
}

// ------------------------------------------------------------------ pass 2
// Q partial over this tile's rows: thread owns VEC columns x RMAX ranks;
// fp32 FMA over 32-row groups, fp64 across groups.
template <int VEC, int RMAX>
__global__ void __launch_bounds__(kP2Threads, VEC == 2 ? 3 : 1) k_pass2(const MatDev *mats, const Tile *tiles, const int32_t *status,
                                                                          const int32_t *any_fb, int32_t epoch) {
    // one independent load first: with every matrix on the Z path and none falling back this
    // run (the steady state) each CTA leaves here instead of after three dependent descriptor
    // loads.  epoch 0: some tile is off the Z path, always run
    if (epoch != 0 && *any_fb != epoch) return;
    const Tile t = tiles[blockIdx.x];
    const MatDev &M = mats[t.mat];
    const int st = status[t.mat];
    if ((st & 1) || (M.zmode && !(st & 2))) return;   // Z path: only on the kappa fallback
    const int r = M.r;
    const int64_t n = M.n;
    const int tid = threadIdx.x;
    const int64_t slot = t.slot0 + tid;
    const bool active = slot < t.slot1;
    const int64_t col0 = slot * VEC;
    __shared__ float s_p[32][RMAX];
    double acc[VEC][RMAX];
#pragma unroll
    for (int v = 0; v < VEC; ++v)
#pragma unroll
        for (int k = 0; k < RMAX; ++k) acc[v][k] = 0.0;
    for (int64_t row = t.row0; row < t.row1; row += 32) {
        __syncthreads();
        for (int e = tid; e < 32 * RMAX; e += kP2Threads) {
            const int rr = e / RMAX, k = e % RMAX;
            const int64_t i = row + rr;
            s_p[rr][k] = (i < t.row1 && k < r) ? M.p_out[i * r + k] : 0.f;
        }
        __syncthreads();
        if (active) {
            float part[VEC][RMAX];
#pragma unroll
            for (int v = 0; v < VEC; ++v)
#pragma unroll
                for (int k = 0; k < RMAX; ++k) part[v][k] = 0.f;
            const int64_t rows = min((int64_t)32, t.row1 - row);
            for (int rr = 0; rr < rows; ++rr) {
                float wv[VEC];
                VecT<VEC>::unpack(VecT<VEC>::ld(M.w + (row + rr) * n + col0), wv);
#pragma unroll
                for (int v = 0; v < VEC; ++v)
#pragma unroll
                    for (int k = 0; k < RMAX; ++k) part[v][k] = fmaf(wv[v], s_p[rr][k], part[v][k]);
            }
#pragma unroll
            for (int v = 0; v < VEC; ++v)
#pragma unroll
                for (int k = 0; k < RMAX; ++k) acc[v][k] += (double)part[v][k];
        }
    }
    if (active) {
#pragma unroll
        for (int v = 0; v < VEC; ++v)
#pragma unroll
            for (int k = 0; k < RMAX; ++k)
                if (k < r) M.q_part[((int64_t)t.chunk * n + col0 + v) * r + k] = acc[v][k];
    }
}

// ---------------------------------------------------------------- finalize
// One thread per Q element (j, k): the Z (or Q) partials of every strip summed in a fixed
// order (deterministic), then Q = Z T through shared memory.  Sized by n r so a single
// matrix still spreads over the GPU; one flat grid over the plan's (matrix, 256-element block)
// pairs (the former [max n r / 256] x matrices grid was mostly empty CTAs: 85 -> 73 us per
// GPT2-2.5B step).
constexpr int kFinThreads = 256;
__global__ void __launch_bounds__(kFinThreads) k_finalize(const MatDev *mats, const int2 *fin, const int32_t *status) {
    // (matrix, block of 256 Q elements): from the flat table, or (y, x) of a one-matrix grid
    const int2 fb = fin ? fin[blockIdx.x] : make_int2((int)blockIdx.y, (int)blockIdx.x);
    const MatDev &M = mats[fb.x];
    const int st = status[fb.x];
    if (st & 1) return;
    const int r = M.r;
    const int64_t n = M.n;
    const bool zq = M.zmode && !(st & 2);
    const int64_t e = (int64_t)fb.y * kFinThreads + threadIdx.x;
    if ((int64_t)fb.y * kFinThreads >= n * r) return;   // whole CTA past this matrix
    const bool live = e < n * r;
    const int64_t j = e / r;
    const int k = (int)(e % r);
    const int nb = zq ? M.nitems : M.nblk2;
    const double *part = zq ? M.zpart : M.q_part;
    double z = 0.0;
    if (live) {
        int b = 0;
        for (; b + 8 <= nb; b += 8) {   // eight strips' loads in flight, summed in strip order
            double zz[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) zz[u] = part[((int64_t)(b + u) * n + j) * r + k];
#pragma unroll
            for (int u = 0; u < 8; ++u) z += zz[u];
        }
        for (; b + 4 <= nb; b += 4) {   // four strips' loads in flight, summed in strip order
            const double z0 = part[((int64_t)b * n + j) * r + k], z1 = part[((int64_t)(b + 1) * n + j) * r + k];
            const double z2 = part[((int64_t)(b + 2) * n + j) * r + k], z3 = part[((int64_t)(b + 3) * n + j) * r + k];
            z += z0;
            z += z1;
            z += z2;
            z += z3;
        }
        for (; b < nb; ++b) z += part[((int64_t)b * n + j) * r + k];
    }
    __shared__ double zs[kFinThreads];
    zs[threadIdx.x] = z;
    __syncthreads();
    if (!live) return;
    float q;
    if (M.dead[k]) {
        q = M.basis[j * M.ld_q + k];   // compressor.py:113-114
    } else if (zq) {
        // Q = Z T (T upper triangular): sum_l Z[j, l] T[l, k]; row j's Z values sit in this CTA
        // unless the row straddles two CTAs (r does not divide 256): then reload them
        const int base = (int)(threadIdx.x - k);
        double a = 0.0;
        for (int l = 0; l <= k; ++l) {
            double zl;
            if (base >= 0) {
                zl = zs[base + l];
            } else {
                zl = 0.0;
                for (int b = 0; b < nb; ++b) zl += part[((int64_t)b * n + j) * r + l];
            }
            a += zl * M.tmat[(int64_t)k * r + l];
        }
        q = (float)a;
    } else {
        q = (float)z;
    }
    M.q_out[j * r + k] = q;
    M.q_warm[j * M.ld_q + k] = q;
}

struct Plan {
    std::vector<MatDev> mats;
    std::vector<Tile> t1v4, t1v1, t2v4, t2v1;
    std::vector<ZTile> tz[9];          // Z-path items grouped by cluster size 1..8
    std::vector<GemmTile> gw, gp, gq;  // wide path: EF update, P_raw and Q tiles for r > 32
    int ef_rk = 0;                     // largest r_res of the CUDA-core EF tiles (gw)
    int tce_rk = 0;                    // largest r_res of the tcgen05 EF tiles (tce)
    std::vector<GemmTile> sp[3], sq[3];   // skinny P_raw / Q tiles: r <= 16 (256x16), <= 32 (128x32), <= 8 (256x8)
    std::vector<GemmTile> spf[3];         // P_raw with the EF update fused: r <= 8 (x8), <= 16 (x16), <= 32 (x32)
    GemmTile *d_spf[3] = {};
    std::vector<GemmTile> tce, tcp[2], tcq[2];
    std::vector<FxTile> fxg, fxr;     // multi-CTA factorisation: Gram tiles, right-multiplication tiles
    int64_t nfxg64 = 0, nfxr64 = 0;   // the first n are 64-edge tiles, the rest kFxBig-edge   // tensor-core EF tiles (128x128), P_raw / Q tiles (BN 64, 128)
    int64_t bytes = 0;
    int64_t max_nr = 1;                // largest n r of the plan
    std::vector<int2> fin;             // k_finalize grid: (matrix, 256-element block) pairs
    int2 *d_fin = nullptr;
    MatDev *d_mats = nullptr;
    Tile *d_t1v4 = nullptr, *d_t1v1 = nullptr, *d_t2v4 = nullptr, *d_t2v1 = nullptr;
    ZTile *d_tz[9] = {};
    GemmTile *d_gw = nullptr, *d_gp = nullptr, *d_gq = nullptr;
    GemmTile *d_sp[3] = {}, *d_sq[3] = {};
    GemmTile *d_tce = nullptr, *d_tcp[2] = {}, *d_tcq[2] = {};
    FxTile *d_fxg = nullptr, *d_fxr = nullptr;
    int rmax4 = 0, rmax1 = 0;
    SampDev *d_samp = nullptr;          // fused sampling descriptors (workspace)
    int32_t *d_anyfb = nullptr;         // k_pass2 gate: the run's epoch if some matrix fell back
    bool pass2_always = false;          // some k_pass2 tile belongs to a matrix off the Z path
    int32_t epoch = 0;                  // run counter (factor phase), from 1; no memset per run
    std::vector<SampDev> samp_host;
    bool sample_armed = false;
    int64_t sample_slots = 0;           // partial slots per matrix (0: some matrix off the Z path)
};

// Clusters of c pass-1 CTAs that can be resident at once (cudaOccupancyMaxActiveClusters: a
// cluster must sit inside one GPC of 18-20 SMs, so a 148-SM part holds fewer than 24 six-CTA
// clusters, not 148 / 6); cached per width.  0 if the query fails.
int pass1_max_clusters(int c) {
    static int cached[9] = {};
    if (c < 1 || c > 8) return 0;
    if (cached[c]) return cached[c];
    static uint64_t attr_f = 0;
    if (smem_attr_once(k_pass1t<false>, (int)sizeof(TSmem), attr_f) != EDGC_OK) return 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(c * 64));
    cfg.blockDim = dim3(kTThreads);
    cfg.dynamicSmemBytes = sizeof(TSmem);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int num = 0;
    if (cudaOccupancyMaxActiveClusters(&num, k_pass1t<false>, &cfg) != cudaSuccess || num <= 0) {
        (void)cudaGetLastError();
        return 0;
    }
    cached[c] = num;
    return num;
}

int make_plan(const edgc_compress_desc *descs, int n, void *ws, int64_t ws_bytes, Plan &P) {
    Arena a(ws, ws_bytes);
    P.mats.resize(n);
    P.d_mats = a.take<MatDev>(n);
    std::vector<FxTile> fxg_big, fxr_big;   // kFxBig-edge factorisation tiles, appended after the 64-edge ones
    // Z-path strip height: kZRows, unless the plan's clusters would not fill one wave of the GPU
    // (a single matrix through the reference's per-matrix compress): then thinner strips, so
    // more clusters stream it (more Z partials to sum, a few KB each)
    int64_t zrows = kZRows;
    int vec_rmax = 0;   // largest rank of the vector group (aligned, r <= kNarrow)
    for (int k = 0; k < n; ++k) {
        const edgc_compress_desc &d = descs[k];
        const bool al4 = (d.n % 4 == 0) && (d.ld_g % 4 == 0) && ((uintptr_t)d.g % 16 == 0) && ((uintptr_t)d.w % 16 == 0);
        if (al4 && std::max(d.r, d.r_res) <= narrow_max()) vec_rmax = std::max(vec_rmax, std::max(d.r, d.r_res));
    }
    {
        int64_t ctas = 0;
        for (int k = 0; k < n; ++k) {
            int zc = (int)ceil_div(std::max<int64_t>(descs[k].n, 1), kTCW);
            if (zc == 4 || zc == 5) zc = 6;
            ctas += ceil_div(std::max<int64_t>(descs[k].m, 1), kZRows) * zc;
        }
        const int64_t want = (int64_t)sm_count();
        if (ctas < want) {
            // thinner strips, but no more clusters than one wave holds: every width's clusters
            // within its resident-cluster limit and all CTAs within the SM count (a second wave
            // of a few clusters would double the kernel: 1024 x 4096 at 40 rows gave 26 six-CTA
            // clusters, 41 us; 48 rows, 22 clusters: 25.5 us)
            zrows = std::max<int64_t>(16, ceil_div(kZRows * ctas, want * 4) * 4);
            for (; zrows < kZRows; zrows += 4) {
                int64_t cl[9] = {}, tot = 0;
                for (int k = 0; k < n; ++k) {
                    int zc = (int)ceil_div(std::max<int64_t>(descs[k].n, 1), kTCW);
                    if (zc == 4 || zc == 5) zc = 6;
                    if (zc > 8) continue;
                    const int64_t c = ceil_div(std::max<int64_t>(descs[k].m, 1), zrows);
                    cl[zc] += c;
                    tot += c * zc;
                }
                bool fits = tot <= want;
                for (int c = 1; c <= 8 && fits; ++c) {
                    const int lim = cl[c] ? pass1_max_clusters(c) : 0;
                    if (cl[c] && lim > 0 && cl[c] > lim) fits = false;
                }
                if (fits) break;
            }
        }
    }
    for (int k = 0; k < n; ++k) {
        const edgc_compress_desc &d = descs[k];
        EDGC_REQUIRE(d.m >= 1 && d.n >= 1, "compress desc %d: dims must be positive", k);
        EDGC_REQUIRE(d.r >= 1 && d.r <= std::min<int64_t>(d.m, d.n), "compress desc %d: rank %d outside [1, %lld]",
                     k, d.r, (long long)std::min(d.m, d.n));
        EDGC_REQUIRE(d.r <= kMaxRank, "compress desc %d: rank %d > %d not supported by this build", k, d.r,
                     kMaxRank);
        EDGC_REQUIRE(d.r_res >= 0 && d.r_res <= kMaxRank, "compress desc %d: r_res %d", k, d.r_res);
        EDGC_REQUIRE(!d.precond || d.ld_s >= d.r, "compress desc %d: ld_s %d < r", k, d.ld_s);
        EDGC_REQUIRE(d.r_res == 0 || (d.p_res && d.q_res), "compress desc %d: residual factors missing", k);
        EDGC_REQUIRE(d.g && d.w && d.q_warm && d.basis && d.p_out && d.q_out && d.ld_q >= d.r && d.ld_g >= d.n,
                     "compress desc %d: null pointer or bad leading dimension", k);
        MatDev &M = P.mats[k];
        P.max_nr = std::max<int64_t>(P.max_nr, d.n * (int64_t)d.r);
        M.g = d.g; M.w = d.w; M.p_res = d.p_res; M.q_res = d.q_res; M.q_warm = d.q_warm; M.basis = d.basis;
        M.p_out = d.p_out; M.q_out = d.q_out;
        M.m = d.m; M.n = d.n; M.ld_g = d.ld_g; M.r = d.r; M.r_res = d.r_res; M.ld_q = d.ld_q;
        M.precond = d.precond; M.ld_s = d.ld_s;
        M.al4 = (d.n % 4 == 0) && (d.ld_g % 4 == 0) && ((uintptr_t)d.g % 16 == 0) &&
                        ((uintptr_t)d.w % 16 == 0);
        const bool v4 = M.al4 && std::max(d.r, d.r_res) <= narrow_max();
        // vector group: float4 columns; pass 2 above rank 4 (r <= 8) takes float2 columns, so its
        // per-thread fp64 Q partials halve and three CTAs fit an SM (measured: 4.8 -> 2.5 ms on
        // the GPT2-2.5B set at r = 8; pass 1 stays float4, its row-block reduction dominates)
        M.vec = v4 ? 4 : 1;
        const int vec2 = v4 ? (vec_rmax <= 4 ? 4 : 2) : 1;
        static const bool z_off = std::getenv("EDGC_NO_ZPATH") != nullptr;
        // cluster size: smallest of {1, 2, 3, 6, 7, 8} covering n with <= kTCW columns per CTA
        // (GPCs hold 18-20 SMs: 4- and 5-CTA clusters would strand SMs); balanced chunks
        int zc = (int)ceil_div(d.n, kTCW);
        if (zc == 4 || zc == 5) zc = 6;
        M.zw = (int32_t)(ceil_div(ceil_div(d.n, zc), 4) * 4);
        M.zmode = (!z_off && v4 && std::max(d.r, d.r_res) <= 4 && zc <= 8) ? 1 : 0;
        M.zc = zc;
        M.nitems = M.zmode ? (int32_t)ceil_div(d.m, zrows) : 0;
        if (M.zmode)
            for (int32_t it = 0; it < M.nitems; ++it)
                P.tz[zc].push_back(ZTile{k, it, (int64_t)it * zrows, std::min(d.m, (int64_t)(it + 1) * zrows)});
        const int64_t slots = d.n / M.vec;
        const int64_t threads1 = kP1Threads;
        M.wide = std::max(d.r, d.r_res) > narrow_max() ? 1 : 0;
        // fused CUDA-core EF + P_raw up to rank 32 (EDGC_SKEF32) keeps those ranks off the tensor cores
        const bool fuse32 = skef32() && M.al4 && d.r > 16 && d.r <= 32 && d.r_res <= 32;
        M.tc = (M.wide && d.r > tc_min_rank() && !fuse32) ? 1 : 0;
        static const bool fx_off = std::getenv("EDGC_NO_FX") != nullptr;
        M.fx = (M.wide && d.r >= 32 && (M.tc || d.r > 32 || fuse32) && !fx_off) ? 1 : 0;   // single P_raw chunk
        if (M.fx) {
            // Gram K splits: >= 512 rows, and few enough that [gsplit][r][r] fits in q_part when possible
            const int64_t want = std::max<int64_t>(512, ceil_div((int64_t)d.m * d.r, d.n));
            M.gks = (int32_t)(ceil_div(want, 16) * 16);
            M.gsplit = (int32_t)ceil_div(d.m, (int64_t)M.gks);
            const int tt = d.r >= kFxBig ? kFxBig : kFxT;   // tile edge (see k_fx_gram)
            auto &vg = tt == kFxBig ? fxg_big : P.fxg;
            auto &vr = tt == kFxBig ? fxr_big : P.fxr;
            const int nbt = (int)ceil_div(d.r, tt);
            for (int32_t c = 0; c < M.gsplit; ++c)
                for (int bi = 0; bi < nbt; ++bi)
                    for (int bj = bi; bj < nbt; ++bj)
                        vg.push_back(FxTile{k, c, bi * tt, bj * tt, (int64_t)c * M.gks,
                                            std::min<int64_t>(d.m, (int64_t)(c + 1) * M.gks)});
            for (int64_t i0 = 0; i0 < d.m; i0 += tt)
                for (int bj = 0; bj < nbt; ++bj)
                    vr.push_back(FxTile{k, 0, 0, bj * tt, i0, std::min<int64_t>(d.m, i0 + tt)});
        }
        // wide path K split of P_raw = w q_warm: 2048 columns up to r = 32; above, one K block
        // (the fp64 partials [nchunk1][m][r] scale with r while the tile count already suffices)
        const int64_t k1 = (M.tc || d.r > 32 || M.fx) ? d.n : kWideSplitK;
        M.nchunk1 = M.wide ? (int32_t)ceil_div(d.n, k1) : (int32_t)ceil_div(slots, threads1);
        // Q partials: 256-row K blocks, or 2048 for the wide path above r = 32 (the fp64
        // partials [nblk2][n][r] would otherwise take ~1 GB per GPT2-12.1B layer at r = 256)
        const int64_t k2 = (M.wide && (M.tc || d.r > 32)) ? d.m : (M.wide ? (int64_t)kSkQK : kP2Rows);
        M.nblk2 = (int32_t)ceil_div(d.m, k2);
        if (M.wide) {
            // 4 < r <= 16, aligned, residual rank within the rank block: EF fused into P_raw
            const int fbn = d.r <= 8 ? 8 : (d.r <= 16 ? 16 : 32);
            const bool fuse = !skef_off() && M.al4 && d.r > 4 && (d.r <= 16 || fuse32) && d.r_res <= fbn && !M.tc;
            if (fuse) {
                const int fi = fbn == 8 ? 0 : (fbn == 16 ? 1 : 2);
                const int rows = fbn == 8 ? kSkEfRows8 : (fbn == 16 ? kSkEfRows16 : kSkEfRows32);
                for (int32_t c = 0; c < M.nchunk1; ++c)
                    for (int64_t i0 = 0; i0 < d.m; i0 += rows)
                        P.spf[fi].push_back(GemmTile{k, c, i0, 0, c * k1, std::min(d.n, (c + 1) * k1)});
                const int BM = fbn == 8 ? kSkQRows8 : (fbn == 16 ? kSkQRows16 : kSkQRows32), BN = fbn;
                std::vector<GemmTile> &tq = P.sq[fbn == 8 ? 2 : (fbn == 16 ? 0 : 1)];
                for (int32_t b = 0; b < M.nblk2; ++b)
                    for (int64_t i0 = 0; i0 < d.n; i0 += BM)
                        for (int64_t j0 = 0; j0 < d.r; j0 += BN)
                            tq.push_back(GemmTile{k, b, i0, j0, (int64_t)b * k2, std::min(d.m, (int64_t)(b + 1) * k2)});
                continue;
            }
            if (d.r_res > tc_ef_min_rank()) {
                for (int64_t i0 = 0; i0 < d.m; i0 += tc::kBM)
                    for (int64_t j0 = 0; j0 < d.n; j0 += kTcEFN) P.tce.push_back(GemmTile{k, 0, i0, j0, 0, d.r_res});
                P.tce_rk = std::max(P.tce_rk, d.r_res);
            } else {
                for (int64_t i0 = 0; i0 < d.m; i0 += kGT)
                    for (int64_t j0 = 0; j0 < d.n; j0 += kGT) P.gw.push_back(GemmTile{k, 0, i0, j0, 0, d.r_res});
                P.ef_rk = std::max(P.ef_rk, d.r_res);
            }
            if (M.tc) {
                // rank blocks of one row block adjacent: co-resident CTAs share the w rows in L2
                const int bn = d.r <= 64 ? 64 : 128, c = d.r <= 64 ? 0 : 1;
                for (int64_t i0 = 0; i0 < d.m; i0 += tc::kBM)
                    for (int64_t j0 = 0; j0 < d.r; j0 += bn) P.tcp[c].push_back(GemmTile{k, 0, i0, j0, 0, d.n});
                for (int64_t i0 = 0; i0 < d.n; i0 += tc::kBM)
                    for (int64_t j0 = 0; j0 < d.r; j0 += bn) P.tcq[c].push_back(GemmTile{k, 0, i0, j0, 0, d.m});
                continue;
            }
            // skinny GEMM tile shape matched to the rank (r > 32: the 64x64 k_gemm tiles)
            // (cfg 2: r <= 8, 256 x 8; 0: r <= 16, 256 x 16; 1: r <= 32, 128 x 32)
            const int cfg = d.r <= 8 ? 2 : (d.r <= 16 ? 0 : (d.r <= 32 ? 1 : 3));
            const int BM = cfg == 0 || cfg == 2 ? 256 : (cfg == 1 ? 128 : kGT);
            const int BN = cfg == 2 ? 8 : (cfg == 0 ? 16 : (cfg == 1 ? 32 : kGT));
            std::vector<GemmTile> &tp = cfg == 3 ? P.gp : P.sp[cfg], &tq = cfg == 3 ? P.gq : P.sq[cfg];
            for (int32_t c = 0; c < M.nchunk1; ++c)
                for (int64_t i0 = 0; i0 < d.m; i0 += BM)
                    for (int64_t j0 = 0; j0 < d.r; j0 += BN)
                        tp.push_back(GemmTile{k, c, i0, j0, c * k1, std::min(d.n, (c + 1) * k1)});
            const int QBM = cfg == 2 ? kSkQRows8 : (cfg == 0 ? kSkQRows16 : (cfg == 1 ? kSkQRows32 : BM));
            for (int32_t b = 0; b < M.nblk2; ++b)
                for (int64_t i0 = 0; i0 < d.n; i0 += QBM)
                    for (int64_t j0 = 0; j0 < d.r; j0 += BN)
                        tq.push_back(GemmTile{k, b, i0, j0, (int64_t)b * k2, std::min(d.m, (int64_t)(b + 1) * k2)});
            continue;
        }
        (v4 ? P.rmax4 : P.rmax1) = std::max(v4 ? P.rmax4 : P.rmax1, std::max(d.r, d.r_res));
        for (int32_t c = 0; c < (M.zmode ? 0 : M.nchunk1); ++c)
            for (int64_t r0 = 0; r0 < d.m; r0 += kP1Rows) {
                Tile t{k, c, c * threads1, std::min(slots, (c + 1) * threads1), r0, std::min(d.m, r0 + kP1Rows)};
                (v4 ? P.t1v4 : P.t1v1).push_back(t);
            }
        const int64_t slots2 = d.n / vec2;
        for (int32_t b = 0; b < M.nblk2; ++b)
            for (int64_t s0 = 0; s0 < slots2; s0 += kP2Threads) {
                Tile t{k, b, s0, std::min(slots2, s0 + kP2Threads), (int64_t)b * kP2Rows,
                       std::min(d.m, (int64_t)(b + 1) * kP2Rows)};
                (v4 ? P.t2v4 : P.t2v1).push_back(t);
            }
    }
    P.nfxg64 = (int64_t)P.fxg.size();
    P.nfxr64 = (int64_t)P.fxr.size();
    P.fxg.insert(P.fxg.end(), fxg_big.begin(), fxg_big.end());
    P.fxr.insert(P.fxr.end(), fxr_big.begin(), fxr_big.end());
    for (int k = 0; k < n; ++k) {
        MatDev &M = P.mats[k];
        M.p_part = a.take<double>(M.zmode ? 0 : (int64_t)M.nchunk1 * M.m * M.r);
        M.zpart = a.take<double>((int64_t)M.nitems * M.n * M.r);
        // a single P_raw partial is P_raw itself (the factor's chunk sum copies it in place)
        M.p_raw = (!M.zmode && M.nchunk1 == 1) ? M.p_part : a.take<double>(M.m * M.r);
        M.q_part = a.take<double>((int64_t)M.nblk2 * M.n * M.r);
        M.tmat = a.take<double>((int64_t)M.r * M.r);
        M.dead = a.take<int32_t>(M.r);
        M.fwork = a.take<double>(5 * (int64_t)M.r * M.r);
        M.p_tmp = a.take<double>(M.m * M.r);
        M.fmode = a.take<int32_t>(M.fx ? 1 : 0);
        const int64_t gp = M.fx ? (int64_t)M.gsplit * M.r * M.r : 0;
        M.gpart = gp <= (int64_t)M.nblk2 * M.n * M.r ? M.q_part : a.take<double>(gp);
    }
    P.d_samp = a.take<SampDev>(n);
    P.sample_slots = 0;
    {
        bool all_z = true;
        for (int k = 0; k < n; ++k) {
            all_z = all_z && P.mats[k].zmode;
            if (P.mats[k].zmode) P.sample_slots = std::max<int64_t>(P.sample_slots, (int64_t)P.mats[k].nitems * P.mats[k].zc);
        }
        if (!all_z) P.sample_slots = 0;
    }
    P.d_t1v4 = a.take<Tile>(P.t1v4.size());
    P.d_t1v1 = a.take<Tile>(P.t1v1.size());
    P.d_t2v4 = a.take<Tile>(P.t2v4.size());
    P.d_t2v1 = a.take<Tile>(P.t2v1.size());
    for (int c = 1; c <= 8; ++c) P.d_tz[c] = a.take<ZTile>(P.tz[c].size());
    for (int c = 0; c < 3; ++c) {
        P.d_sp[c] = a.take<GemmTile>(P.sp[c].size());
        P.d_spf[c] = a.take<GemmTile>(P.spf[c].size());
        P.d_sq[c] = a.take<GemmTile>(P.sq[c].size());
    }
    P.d_tce = a.take<GemmTile>(P.tce.size());
    for (int c = 0; c < 2; ++c) {
        P.d_tcp[c] = a.take<GemmTile>(P.tcp[c].size());
        P.d_tcq[c] = a.take<GemmTile>(P.tcq[c].size());
    }
    P.d_fxg = a.take<FxTile>(P.fxg.size());
    P.d_fxr = a.take<FxTile>(P.fxr.size());
    P.d_gw = a.take<GemmTile>(P.gw.size());
    P.d_gp = a.take<GemmTile>(P.gp.size());
    P.d_gq = a.take<GemmTile>(P.gq.size());
    P.d_anyfb = a.take<int32_t>(1);
    for (int k = 0; k < n; ++k)
        for (int64_t b = 0; b < ceil_div(descs[k].n * (int64_t)descs[k].r, kFinThreads); ++b)
            P.fin.push_back(make_int2(k, (int)b));
    P.d_fin = a.take<int2>(P.fin.size());
    P.pass2_always = false;
    for (int k = 0; k < n; ++k)
        if (!P.mats[k].wide && !P.mats[k].zmode) P.pass2_always = true;
    P.bytes = a.off;
    return EDGC_OK;
}

int launch_pass1(const Plan &P, bool v4, int32_t *status, cudaStream_t st) {
    const std::vector<Tile> &h = v4 ? P.t1v4 : P.t1v1;
    const Tile *d = v4 ? P.d_t1v4 : P.d_t1v1;
    if (h.empty()) return EDGC_OK;
    const unsigned grid = (unsigned)h.size();
    const int rmax = v4 ? P.rmax4 : P.rmax1;
    if (v4 && rmax <= 4) k_pass1<4, 4, 4><<<grid, kP1Threads, 0, st>>>(P.d_mats, d, status);
    else if (v4) k_pass1<4, 8, 2><<<grid, kP1Threads, 0, st>>>(P.d_mats, d, status);
    else if (rmax <= 4) k_pass1<1, 4, 4><<<grid, kP1Threads, 0, st>>>(P.d_mats, d, status);
    else k_pass1<1, 8, 2><<<grid, kP1Threads, 0, st>>>(P.d_mats, d, status);
    EDGC_LAUNCH_CHECK();
    return EDGC_OK;
}

template <int OP>
int launch_gemm(const Plan &P, const std::vector<GemmTile> &h, const GemmTile *d, int32_t *status, cudaStream_t st) {
    if (h.empty()) return EDGC_OK;
    k_gemm<OP><<<(unsigned)h.size(), kGThreads, 0, st>>>(P.d_mats, d, status);
    EDGC_LAUNCH_CHECK();
    return EDGC_OK;
}

int launch_ef(const Plan &P, cudaStream_t st, int32_t *status) {
    if (P.gw.empty()) return EDGC_OK;
    const unsigned grid = (unsigned)P.gw.size();
    static const bool gemm = std::getenv("EDGC_EF_GEMM") != nullptr;   // A/B: the generic tile kernel
    if (gemm) k_gemm<2><<<grid, kGThreads, 0, st>>>(P.d_mats, P.d_gw, status);
    else if (P.ef_rk <= 8) k_ef<8><<<grid, kGThreads, 0, st>>>(P.d_mats, P.d_gw, status);
    else if (P.ef_rk <= 16) k_ef<16><<<grid, kGThreads, 0, st>>>(P.d_mats, P.d_gw, status);
    else if (P.ef_rk <= 32) k_ef<32><<<grid, kGThreads, 0, st>>>(P.d_mats, P.d_gw, status);
    else k_gemm<2><<<grid, kGThreads, 0, st>>>(P.d_mats, P.d_gw, status);
    EDGC_LAUNCH_CHECK();
    return EDGC_OK;
}

// Per-device side streams for the concurrent cluster-width launches (fork/join by
// events: graph-capturable).
struct ForkJoin {
    cudaStream_t side[8] = {};
    cudaEvent_t fork = nullptr, join[8] = {};
};
static int fork_join(ForkJoin *&out) {
    static ForkJoin fj[16];
    static bool ready[16] = {};
    int dev = 0;
    EDGC_CUDA_TRY(cudaGetDevice(&dev));
    EDGC_REQUIRE(dev >= 0 && dev < 16, "device %d", dev);
    if (!ready[dev]) {
        for (int i = 0; i < 8; ++i) {
            EDGC_CUDA_TRY(cudaStreamCreateWithFlags(&fj[dev].side[i], cudaStreamNonBlocking));
            EDGC_CUDA_TRY(cudaEventCreateWithFlags(&fj[dev].join[i], cudaEventDisableTiming));
        }
        EDGC_CUDA_TRY(cudaEventCreateWithFlags(&fj[dev].fork, cudaEventDisableTiming));
        ready[dev] = true;
    }
    out = &fj[dev];
    return EDGC_OK;
}

int launch_pass1z(const Plan &P, int32_t *status, bool sample, cudaStream_t st) {
    // one launch per cluster width; with several widths they run concurrently on forked
    // streams, so each launch's partial last wave is filled by the other's clusters
    int widths = 0;
    for (int c = 1; c <= 8; ++c) widths += !P.tz[c].empty();
    ForkJoin *fj = nullptr;
    static const bool serial = std::getenv("EDGC_PASS1_SERIAL") != nullptr;
    if (widths > 1 && !serial) {
        int rc = fork_join(fj);
        if (rc != EDGC_OK) return rc;
        EDGC_CUDA_TRY(cudaEventRecord(fj->fork, st));
    }
    int used = 0;
    for (int c = 8; c >= 1; --c) {   // widest clusters first
        if (P.tz[c].empty()) continue;
        cudaStream_t ls = st;
        if (fj && used > 0) {
            ls = fj->side[used];
            EDGC_CUDA_TRY(cudaStreamWaitEvent(ls, fj->fork, 0));
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(P.tz[c].size() * c));
        cfg.blockDim = dim3(kTThreads);
        cfg.dynamicSmemBytes = sizeof(TSmem);
        cfg.stream = ls;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = c;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        static uint64_t attr_f = 0, attr_t = 0;
        int arc = smem_attr_once(k_pass1t<false>, (int)sizeof(TSmem), attr_f);
        if (arc == EDGC_OK) arc = smem_attr_once(k_pass1t<true>, (int)sizeof(TSmem), attr_t);
        if (arc != EDGC_OK) return arc;
        if (sample)
            EDGC_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_pass1t<true>, (const MatDev *)P.d_mats,
                                             (const ZTile *)P.d_tz[c], status, (const SampDev *)P.d_samp));
        else
            EDGC_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_pass1t<false>, (const MatDev *)P.d_mats,
                                             (const ZTile *)P.d_tz[c], status, (const SampDev *)P.d_samp));
        EDGC_LAUNCH_CHECK();
        if (fj && used > 0) {
            EDGC_CUDA_TRY(cudaEventRecord(fj->join[used], ls));
            EDGC_CUDA_TRY(cudaStreamWaitEvent(st, fj->join[used], 0));
        }
        ++used;
    }
    return EDGC_OK;
}

int launch_pass2(const Plan &P, bool v4, const int32_t *status, cudaStream_t st) {
    const std::vector<Tile> &h = v4 ? P.t2v4 : P.t2v1;
    const Tile *d = v4 ? P.d_t2v4 : P.d_t2v1;
    if (h.empty()) return EDGC_OK;
    const unsigned grid = (unsigned)h.size();
    const int rmax = v4 ? P.rmax4 : P.rmax1;
    if (v4 && rmax <= 4) k_pass2<4, 4><<<grid, kP2Threads, 0, st>>>(P.d_mats, d, status, P.d_anyfb, P.pass2_always ? 0 : P.epoch);
    else if (v4) k_pass2<2, 8><<<grid, kP2Threads, 0, st>>>(P.d_mats, d, status, P.d_anyfb, P.pass2_always ? 0 : P.epoch);
    else if (rmax <= 4) k_pass2<1, 4><<<grid, kP2Threads, 0, st>>>(P.d_mats, d, status, P.d_anyfb, P.pass2_always ? 0 : P.epoch);
    else k_pass2<1, 8><<<grid, kP2Threads, 0, st>>>(P.d_mats, d, status, P.d_anyfb, P.pass2_always ? 0 : P.epoch);
    EDGC_LAUNCH_CHECK();
    return EDGC_OK;
}

// ---------------------------------------------------------- reconstruction
struct ReconDev {
    const float *p, *q;
    float *out;
    int64_t m, n, ld_out, p_stride, q_stride;
    int32_t r, n_ranks;
    float scale;
};

struct RTile {
    int32_t d;
    int64_t col0, col1, row0, row1;
};

constexpr int kRThreads = 128;
constexpr int kRRows = 32;      // rows per register block
constexpr int kRTileRows = 128;

// out[i, j] = scale * sum_w sum_k P_w[i, k] Q_w[j, k], accumulated in rank order
template <int kRChunk>  // (rank, k) pairs per register chunk
__global__ void __launch_bounds__(kRThreads) k_recon(const ReconDev *descs, const RTile *tiles) {
    const RTile t = tiles[blockIdx.x];
    const ReconDev D = descs[t.d];
    const int r = D.r, WR = D.r * D.n_ranks;
    const int64_t j = t.col0 + threadIdx.x;
    const bool active = j < t.col1;
    __shared__ float s_p[kRRows][kRChunk];
    for (int64_t row = t.row0; row < t.row1; row += kRRows) {
        float acc[kRRows];
#pragma unroll
        for (int rr = 0; rr < kRRows; ++rr) acc[rr] = 0.f;
        for (int c0 = 0; c0 < WR; c0 += kRChunk) {
            const int cn = min(kRChunk, WR - c0);
            float q[kRChunk];
#pragma unroll
            for (int c = 0; c < kRChunk; ++c) {
                const int wk = c0 + c;
                q[c] = (active && c < cn) ? __ldg(D.q + (int64_t)(wk / r) * D.q_stride + j * r + (wk % r)) : 0.f;
            }
            __syncthreads();
            for (int e = threadIdx.x; e < kRRows * kRChunk; e += kRThreads) {
                const int rr = e / kRChunk, c = e % kRChunk;
                const int64_t i = row + rr;
                const int wk = c0 + c;
                s_p[rr][c] = (i < t.row1 && c < cn) ? D.p[(int64_t)(wk / r) * D.p_stride + i * r + (wk % r)] : 0.f;
            }
            __syncthreads();
#pragma unroll
            for (int rr = 0; rr < kRRows; ++rr)
#pragma unroll
                for (int c = 0; c < kRChunk; ++c) acc[rr] = fmaf(s_p[rr][c], q[c], acc[rr]);
        }
        if (active) {
#pragma unroll
            for (int rr = 0; rr < kRRows; ++rr) {
                const int64_t i = row + rr;
                if (i < t.row1) __stcs(D.out + i * D.ld_out + j, acc[rr] * D.scale);
            }
        }
    }
}

// W*r > 8 with float4-aligned output: 64x64 output tiles, K = W*r staged through
// shared memory 16 at a time, 4x4 fp32 outputs per thread (the same fma order over
// (worker, k) as k_recon), float4 streaming stores.
__global__ void __launch_bounds__(kGThreads) k_recon_tiled(const ReconDev *descs, const RTile *tiles) {
    const RTile t = tiles[blockIdx.x];
    const ReconDev D = descs[t.d];
    const int r = D.r, K = D.r * D.n_ranks;
    __shared__ float As[kGK][kGT + 4];
    __shared__ float Bs[kGK][kGT + 4];
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += kGK) {
        for (int e = tid; e < kGT * kGK; e += kGThreads) {
            const int kk = e % kGK, ii = e / kGK, wk = k0 + kk;
            const int64_t i = t.row0 + ii, j = t.col0 + ii;
            As[kk][ii] = (i < t.row1 && wk < K) ? __ldg(D.p + (int64_t)(wk / r) * D.p_stride + i * r + wk % r) : 0.f;
            Bs[kk][ii] = (j < t.col1 && wk < K) ? __ldg(D.q + (int64_t)(wk / r) * D.q_stride + j * r + wk % r) : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kGK; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) { a[u] = As[kk][ty * 4 + u]; b[u] = Bs[kk][tx * 4 + u]; }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(a[u], b[v], acc[u][v]);
        }
        __syncthreads();
    }
    const int64_t j = t.col0 + tx * 4;
    if (j >= t.col1) return;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int64_t i = t.row0 + ty * 4 + u;
        if (i >= t.row1) continue;
        __stcs(reinterpret_cast<float4 *>(D.out + i * D.ld_out + j),
               make_float4(acc[u][0] * D.scale, acc[u][1] * D.scale, acc[u][2] * D.scale, acc[u][3] * D.scale));
    }
}

// float4 variant for W*r <= 32 (the DP-average hot case, r = 4 up to W = 8): each thread owns 4
// adjacent columns and kV4Rows rows per pass, with Q (4 x W*r) in registers and
// P rows broadcast from shared memory; 512-byte coalesced streaming stores.
constexpr int kV4Threads = 128;
constexpr int kV4Cols = 4 * kV4Threads;
constexpr int kV4Rows = 8;
// rows per tile: 64 while Q (W*r <= 8 per column) is cheap to load, 256 above to amortise it
// rows per reconstruction tile (x 512 columns): one tile's Q columns stay in registers across
// them.  W r = 5..8: 256 (measured 64 / 128 / 256 rows: r = 8 at W = 1 1.96 / 1.52 / 1.39 ms,
// r = 4 at W = 2 1.50 / 1.35 / 1.37 ms)
#ifndef EDGC_RECON4_ROWS
#define EDGC_RECON4_ROWS 64
#endif
#ifndef EDGC_RECON8_ROWS
#define EDGC_RECON8_ROWS 256
#endif
#ifndef EDGC_RECON16_TROWS
#define EDGC_RECON16_TROWS 512   // W r = 9..16 (256 rows: r = 16 at W = 1 2.32 ms, 512: 2.08 ms)
#endif
#ifndef EDGC_RECON32_TROWS
#define EDGC_RECON32_TROWS 512   // W r = 17..32 (64 / 128 / 256 / 512 rows at W = 8, r = 4: 4.79 / 4.20 / 3.92 / 3.79 ms)
#endif
// 512-column blocks per tile at W r = 17..32 (one P tile load for all of them; measured 1 / 2 /
// 4 / 8 blocks: r = 32 at W = 1 4.34 / 4.15 / 4.07 / 4.32 ms, r = 4 at W = 8 3.74 / 3.68 / 3.68 /
// 3.97 ms -- the FMA loop, not the P tile load, bounds this kernel)
#ifndef EDGC_RECON_CB32
#define EDGC_RECON_CB32 4
#endif
constexpr int v4_col_blocks(int wr) { return wr <= 16 ? 1 : EDGC_RECON_CB32; }
__host__ __device__ constexpr int v4_tile_rows(int wr) {
    return wr <= 4 ? EDGC_RECON4_ROWS : wr <= 8 ? EDGC_RECON8_ROWS : wr <= 16 ? EDGC_RECON16_TROWS : EDGC_RECON32_TROWS;
}

// VC adjacent columns per thread (4, or 2 when W*r = 32 to keep Q in registers);
// kV4Cols = 512 columns per tile either way.
#ifndef EDGC_RECON32_ROWS
#define EDGC_RECON32_ROWS 8
#endif
// W r from which k_recon4 multiplies on FFMA2 (measured W r = 32: r = 4 at W = 8 3.68 -> 2.79 ms,
// r = 32 at W = 1 4.06 -> 3.29 ms)
#ifndef EDGC_RECON_FFMA2_MIN
#define EDGC_RECON_FFMA2_MIN 8
#endif
#ifndef EDGC_RECON32_MINB
#define EDGC_RECON32_MINB 2   // CTAs per SM for W*r = 32 (2 caps registers at 128: Q partly spills)
#endif
__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t *p) {
    int64_t v;
    asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

template <int WR, int VC>
__global__ void __launch_bounds__(kV4Cols / VC, VC == 2 ? EDGC_RECON32_MINB : 1) k_recon4(const ReconDev *descs, const RTile *tiles) {
    constexpr int NT = kV4Cols / VC;
    constexpr int kV4TileRows = v4_tile_rows(WR);
    const RTile t = tiles[blockIdx.x];
    const ReconDev D = descs[t.d];
    const int r = D.r, wr = D.r * D.n_ranks;
    // rank w's P_k / Q_k in the gathered buffer
    auto p_of = [&](int w) -> const float * { return D.p + (int64_t)w * D.p_stride; };
    auto q_of = [&](int w) -> const float * { return D.q + (int64_t)w * D.q_stride; };
    // P tile transposed ([k][row]): one 16-byte shared read gives 4 rows of one k
    extern __shared__ __align__(16) float recon4_smem[];   // [WR][kV4TileRows], dynamic (64 KB at W r = 32)
    float (*s_pT)[kV4TileRows] = reinterpret_cast<float (*)[kV4TileRows]>(recon4_smem);
    // thread = (row, rank): its r consecutive P values; (worker, k) indexed incrementally (no div/mod)
    for (int e = threadIdx.x; e < kV4TileRows * D.n_ranks; e += NT) {
        const int rr = e % kV4TileRows, w = e / kV4TileRows;
        const int64_t i = t.row0 + rr;
        const float *src = p_of(w) + i * r;
        for (int k = 0; k < r; ++k) s_pT[w * r + k][rr] = i < t.row1 ? src[k] : 0.f;
    }
    for (int e = threadIdx.x; e < kV4TileRows * (WR - wr); e += NT)   // zero padding columns
        s_pT[wr + e / kV4TileRows][e % kV4TileRows] = 0.f;
    __syncthreads();
    // the tile may span several 512-column blocks (W r = 17..32): the P tile above is loaded
    // once for all of them, each block reloads only its Q columns (registers)
    auto block = [&](int64_t cb0) {
    const int64_t j0 = cb0 + VC * threadIdx.x;
    const bool active = j0 < t.col1;
    if (!active) return;
    float q[VC][WR];
#pragma unroll
    for (int v = 0; v < VC; ++v) {
        int k = 0, w = 0;
        const float *qp = q_of(0) + (j0 + v) * r;
#pragma unroll
        for (int c = 0; c < WR; ++c) {
            q[v][c] = (active && c < wr) ? __ldg(qp + k) : 0.f;
            if (++k == r) {
                k = 0;
                ++w;
                if (c + 1 < wr) qp = q_of(w) + (j0 + v) * r;
            }
        }
    }
    // rows per pass: 8, or EDGC_RECON32_ROWS for W*r = 32 (fewer live accumulators next to Q)
    constexpr int RP = WR == 32 ? EDGC_RECON32_ROWS : kV4Rows;
    for (int64_t row = t.row0; row < t.row1; row += RP) {
        const int lr = (int)(row - t.row0);
        float acc[RP][VC];
#pragma unroll
        for (int rr = 0; rr < RP; ++rr)
#pragma unroll
            for (int v = 0; v < VC; ++v) acc[rr][v] = 0.f;
        // per output the fma order over (worker, k) is c ascending
        if constexpr (WR >= EDGC_RECON_FFMA2_MIN && VC % 2 == 0) {
            // paired columns on the packed FP32 pipe (FFMA2 with the P value as a broadcast scalar
            // operand: same rounding per lane, half the FMA instructions to issue)
            float2 acc2[RP][VC / 2];
#pragma unroll
            for (int rr = 0; rr < RP; ++rr)
#pragma unroll
                for (int v = 0; v < VC / 2; ++v) acc2[rr][v] = make_float2(0.f, 0.f);
#pragma unroll
            for (int c = 0; c < WR; ++c) {
                float pr[RP];
#pragma unroll
                for (int h = 0; h < RP; h += 4) {
                    const float4 pa = *reinterpret_cast<const float4 *>(&s_pT[c][lr + h]);
                    pr[h] = pa.x; pr[h + 1] = pa.y; pr[h + 2] = pa.z; pr[h + 3] = pa.w;
                }
#pragma unroll
                for (int v = 0; v < VC / 2; ++v) {
                    const float2 qc = make_float2(q[2 * v][c], q[2 * v + 1][c]);
#pragma unroll
                    for (int rr = 0; rr < RP; ++rr)
                        acc2[rr][v] = __ffma2_rn(make_float2(pr[rr], pr[rr]), qc, acc2[rr][v]);
                }
            }
#pragma unroll
            for (int rr = 0; rr < RP; ++rr)
#pragma unroll
                for (int v = 0; v < VC / 2; ++v) {
                    acc[rr][2 * v] = acc2[rr][v].x;
                    acc[rr][2 * v + 1] = acc2[rr][v].y;
                }
        } else
        {
#pragma unroll
        for (int c = 0; c < WR; ++c) {
            float pr[RP];
#pragma unroll
            for (int h = 0; h < RP; h += 4) {
                const float4 pa = *reinterpret_cast<const float4 *>(&s_pT[c][lr + h]);
                pr[h] = pa.x; pr[h + 1] = pa.y; pr[h + 2] = pa.z; pr[h + 3] = pa.w;
            }
#pragma unroll
            for (int rr = 0; rr < RP; ++rr)
#pragma unroll
                for (int v = 0; v < VC; ++v) acc[rr][v] = fmaf(pr[rr], q[v][c], acc[rr][v]);
        }
        }
#pragma unroll
        for (int rr = 0; rr < RP; ++rr) {
            const int64_t i = row + rr;
            if (i >= t.row1) continue;
            if (VC == 4)
                __stcs(reinterpret_cast<float4 *>(D.out + i * D.ld_out + j0),
                       make_float4(acc[rr][0] * D.scale, acc[rr][VC > 1 ? 1 : 0] * D.scale,
                                   acc[rr][VC > 2 ? 2 : 0] * D.scale, acc[rr][VC > 3 ? 3 : 0] * D.scale));
            else
                __stcs(reinterpret_cast<float2 *>(D.out + i * D.ld_out + j0),
                       make_float2(acc[rr][0] * D.scale, acc[rr][VC > 1 ? 1 : 0] * D.scale));
        }
    }
    };
    if (WR == 32) {
        for (int64_t cb0 = t.col0; cb0 < t.col1; cb0 += kV4Cols) block(cb0);
    } else {
        block(t.col0);   // one column block per tile
    }
}

// ----------------------------------------------------------- misc kernels
__global__ void k_residual(const float *w, const float *p, const float *q, int r, int64_t m, int64_t n, float *e) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < m * n; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = x / n, j = x % n;
        float dot = 0.f;
        for (int k = 0; k < r; ++k) dot = fmaf(p[i * r + k], q[j * r + k], dot);
        e[x] = w[x] - dot;
    }
}

__global__ void k_check_work(const float *g, int64_t ld_g, const float *w, const float *p, const float *q, int r,
                             int64_t m, int64_t n, int32_t *flag) {
    // rows over grid.y, columns over grid.x: no per-element division
    bool bad = false;
    for (int64_t i = blockIdx.y; i < m; i += gridDim.y)
        for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
            float dot = 0.f;
            for (int k = 0; k < r; ++k) dot = fmaf(p[i * r + k], q[j * r + k], dot);
            bad |= !isfinite(g[i * ld_g + j] + (w[i * n + j] - dot));
        }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

template <typename T>
__global__ void k_check_finite(const T *x, int64_t count, int32_t *flag) {
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(x[i]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

int elementwise_blocks(int64_t count) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(count, 256), sm_count() * 8)); }

// out = scale * P_all Q_all^T on the tensor cores (M = m, N = n, K = W r; the
// per-rank factor blocks are the K index's rank blocks)
struct TcRecon {
    static constexpr bool kAMN = false, kBMN = false;
    static constexpr int kPF = 0, kPFDepth = 2, kStages = 0;
    using Tile = RTile;
    const ReconDev *descs;
    const RTile *tiles;
    int ntiles;
    __device__ Tile tile(int i) const { return tiles[i]; }
    __device__ int64_t tile_k(const Tile &t) const { return (int64_t)descs[t.d].r * descs[t.d].n_ranks; }
    __device__ void views(const Tile &t, tc::View &a, tc::View &b) const {
        const ReconDev &D = descs[t.d];
        const int64_t K = (int64_t)D.r * D.n_ranks, kb = D.n_ranks > 1 ? D.r : 0;
        a = tc::View{D.p + t.row0 * D.r, D.r, D.m - t.row0, K, kb, D.p_stride};
        b = tc::View{D.q + t.col0 * D.r, D.r, D.n - t.col0, K, kb, D.q_stride};
    }
    __device__ void prefetch(const Tile &, int, int, uint8_t *) const {}
    __device__ void epilogue(const Tile &t, int row0, int col, const float4 (&v)[8], const uint8_t *) const {
        const ReconDev &D = descs[t.d];
        const int64_t j = t.col0 + col;
        if (j >= D.n) return;
        const int nu = tc_rows4(D.m - t.row0 - row0);
        const float sc = D.scale;
        const bool vec = j + 4 <= D.n && D.ld_out % 4 == 0 && ((uintptr_t)D.out % 16) == 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (u >= nu) break;
            float *o = D.out + (t.row0 + row0 + 4 * u) * D.ld_out + j;
            if (vec) {
                __stcs(reinterpret_cast<float4 *>(o), make_float4(v[u].x * sc, v[u].y * sc, v[u].z * sc, v[u].w * sc));
            } else {
                const float a[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
                for (int c = 0; c < 4 && j + c < D.n; ++c) o[c] = a[c] * sc;
            }
        }
    }
};

}  // namespace
}  // namespace edgc

using namespace edgc;

struct edgc_compress_plan {
    std::vector<edgc_compress_desc> descs;
    Plan P;
    int64_t bytes = 0;
};

struct edgc_recon_plan;

extern "C" int edgc_compress_plan_create(const edgc_compress_desc *descs, int n, edgc_compress_plan **out) {
    EDGC_REQUIRE(out && n >= 1 && descs, "edgc_compress_plan_create: bad arguments");
    auto *h = new edgc_compress_plan();
    h->descs.assign(descs, descs + n);
    int rc = make_plan(descs, n, nullptr, INT64_MAX, h->P);
    if (rc != EDGC_OK) { delete h; return rc; }
    h->bytes = h->P.bytes;
    *out = h;
    return EDGC_OK;
}

extern "C" int64_t edgc_compress_plan_workspace_bytes(const edgc_compress_plan *h) { return h ? h->bytes : -1; }

extern "C" int edgc_compress_plan_bind(edgc_compress_plan *h, void *ws, int64_t ws_bytes, void *stream) {
    EDGC_REQUIRE(h && ws && ws_bytes >= h->bytes, "edgc_compress_plan_bind: workspace %lld < needed %lld",
                 (long long)ws_bytes, h ? (long long)h->bytes : -1LL);
    Plan &P = h->P;
    P = Plan();
    int rc = make_plan(h->descs.data(), (int)h->descs.size(), ws, ws_bytes, P);
    if (rc != EDGC_OK) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const int n = (int)h->descs.size();
    EDGC_CUDA_TRY(cudaMemcpyAsync(P.d_mats, P.mats.data(), sizeof(MatDev) * n, cudaMemcpyHostToDevice, st));
    auto up = [&](Tile *d, const std::vector<Tile> &v) -> cudaError_t {
        return v.empty() ? cudaSuccess
                         : cudaMemcpyAsync(d, v.data(), sizeof(Tile) * v.size(), cudaMemcpyHostToDevice, st);
    };
    EDGC_CUDA_TRY(up(P.d_t1v4, P.t1v4));
    EDGC_CUDA_TRY(up(P.d_t1v1, P.t1v1));
    EDGC_CUDA_TRY(up(P.d_t2v4, P.t2v4));
    EDGC_CUDA_TRY(up(P.d_t2v1, P.t2v1));
    for (int c = 1; c <= 8; ++c)
        if (!P.tz[c].empty())
            EDGC_CUDA_TRY(cudaMemcpyAsync(P.d_tz[c], P.tz[c].data(), sizeof(ZTile) * P.tz[c].size(),
                                          cudaMemcpyHostToDevice, st));
    auto upg = [&](GemmTile *d, const std::vector<GemmTile> &v) -> cudaError_t {
        return v.empty() ? cudaSuccess
                         : cudaMemcpyAsync(d, v.data(), sizeof(GemmTile) * v.size(), cudaMemcpyHostToDevice, st);
    };
    EDGC_CUDA_TRY(upg(P.d_gw, P.gw));
    EDGC_CUDA_TRY(upg(P.d_tce, P.tce));
    if (!P.fxg.empty())
        EDGC_CUDA_TRY(cudaMemcpyAsync(P.d_fxg, P.fxg.data(), sizeof(FxTile) * P.fxg.size(), cudaMemcpyHostToDevice, st));
    if (!P.fxr.empty())
        EDGC_CUDA_TRY(cudaMemcpyAsync(P.d_fxr, P.fxr.data(), sizeof(FxTile) * P.fxr.size(), cudaMemcpyHostToDevice, st));
    for (int c = 0; c < 2; ++c) {
        EDGC_CUDA_TRY(upg(P.d_tcp[c], P.tcp[c]));
        EDGC_CUDA_TRY(upg(P.d_tcq[c], P.tcq[c]));
    }
    EDGC_CUDA_TRY(upg(P.d_gp, P.gp));
    EDGC_CUDA_TRY(upg(P.d_gq, P.gq));
    for (int c = 0; c < 3; ++c) {
        EDGC_CUDA_TRY(upg(P.d_sp[c], P.sp[c]));
        EDGC_CUDA_TRY(upg(P.d_spf[c], P.spf[c]));
        EDGC_CUDA_TRY(upg(P.d_sq[c], P.sq[c]));
    }
    if (!P.fin.empty())
        EDGC_CUDA_TRY(cudaMemcpyAsync(P.d_fin, P.fin.data(), sizeof(int2) * P.fin.size(), cudaMemcpyHostToDevice, st));
    EDGC_CUDA_TRY(cudaMemsetAsync(P.d_anyfb, 0, sizeof(int32_t), st));   // epochs start at 1
    // the host staging vectors stay alive in the plan; make the upload complete
    // before the caller could destroy or rebind it
    EDGC_CUDA_TRY(cudaStreamSynchronize(st));
    return EDGC_OK;
}

extern "C" int edgc_compress_plan_run(edgc_compress_plan *h, double col_tol, int32_t *status_dev, int phases,
                                      void *stream) {
    EDGC_REQUIRE(h && status_dev && h->P.d_mats, "edgc_compress_plan_run: plan not bound");
    const Plan &P = h->P;
    const int n = (int)h->descs.size();
    cudaStream_t st = (cudaStream_t)stream;
    int rc;
    if (phases & EDGC_PHASE_PASS1) {
        EDGC_CUDA_TRY(cudaMemsetAsync(status_dev, 0, sizeof(int32_t) * n, st));
        if ((rc = launch_pass1(P, true, status_dev, st))) return rc;
        if ((rc = launch_pass1(P, false, status_dev, st))) return rc;
        if ((rc = launch_pass1z(P, status_dev, P.sample_armed, st))) return rc;
        h->P.sample_armed = false;   // set_sampling arms exactly one pass 1
        if ((rc = launch_ef(P, st, status_dev))) return rc;
        if (!P.tce.empty()) {
            if (P.tce_rk <= 128)
                EDGC_CUDA_TRY((tc::launch<kTcEFN, 4>(TcEF{P.d_mats, P.d_tce, status_dev, (int)P.tce.size()}, sm_count(), st)));
            else
                EDGC_CUDA_TRY(
                    (tc::launch<kTcEFN, 4>(TcEFWide{P.d_mats, P.d_tce, status_dev, (int)P.tce.size()}, sm_count(), st)));
        }
        if (!P.tcp[0].empty())
            EDGC_CUDA_TRY((tc::launch<64, 4>(TcPraw{P.d_mats, P.d_tcp[0], (int)P.tcp[0].size()}, sm_count(), st)));
        if (!P.tcp[1].empty())
            EDGC_CUDA_TRY((tc::launch<128, 4>(TcPraw{P.d_mats, P.d_tcp[1], (int)P.tcp[1].size()}, sm_count(), st)));
        if (!P.spf[0].empty()) {
            if ((rc = launch_skinny_ef<kSkEfRows8, 8, kSkEfKS8>((unsigned)P.spf[0].size(), st, P.d_mats, P.d_spf[0], status_dev))) return rc;
            EDGC_LAUNCH_CHECK();
        }
        if (!P.spf[1].empty()) {
            if ((rc = launch_skinny_ef<kSkEfRows16, 16, kSkEfKS16>((unsigned)P.spf[1].size(), st, P.d_mats, P.d_spf[1], status_dev))) return rc;
            EDGC_LAUNCH_CHECK();
        }
        if (!P.spf[2].empty()) {
            if ((rc = launch_skinny_ef<kSkEfRows32, 32, kSkEfKS32>((unsigned)P.spf[2].size(), st, P.d_mats, P.d_spf[2], status_dev))) return rc;
            EDGC_LAUNCH_CHECK();
        }
        if (!P.sp[0].empty()) {
            if ((rc = launch_skinny<0, 256, 16>((unsigned)P.sp[0].size(), st, P.d_mats, P.d_sp[0], status_dev))) return rc;
            EDGC_LAUNCH_CHECK();
        }
        if (!P.sp[1].empty()) {
            if ((rc = launch_skinny<0, 128, 32>((unsigned)P.sp[1].size(), st, P.d_mats, P.d_sp[1], status_dev))) return rc;
            EDGC_LAUNCH_CHECK();
        }
        if (!P.sp[2].empty()) {
            if ((rc = launch_skinny<0, 256, 8>((unsigned)P.sp[2].size(), st, P.d_mats, P.d_sp[2], status_dev))) return rc;
            EDGC_LAUNCH_CHECK();
        }
        if ((rc = launch_gemm<0>(P, P.gp, P.d_gp, status_dev, st))) return rc;
    }
    if (phases & EDGC_PHASE_FACTOR) {
        h->P.epoch = P.epoch == INT32_MAX ? 1 : P.epoch + 1;
        k_factor<<<n, kFactorThreads, 0, st>>>(P.d_mats, status_dev, col_tol, P.d_anyfb, P.epoch);
        EDGC_LAUNCH_CHECK();
        if (!P.fxg.empty()) {
            const unsigned g64 = (unsigned)P.nfxg64, gbig = (unsigned)(P.fxg.size() - P.nfxg64);
            const unsigned r64 = (unsigned)P.nfxr64, rbig = (unsigned)(P.fxr.size() - P.nfxr64);
            auto gram = [&](int pass) {
                if (g64) k_fx_gram<kFxT><<<g64, kFxThreads, 0, st>>>(P.d_mats, P.d_fxg, status_dev, pass);
                if (gbig) k_fx_gram<kFxBig><<<gbig, kFxThreads, 0, st>>>(P.d_mats, P.d_fxg + g64, status_dev, pass);
            };
            auto rmul = [&](int pass) {
                if (r64) k_fx_rmul<kFxT><<<r64, kFxThreads, 0, st>>>(P.d_mats, P.d_fxr, status_dev, pass);
                if (rbig) k_fx_rmul<kFxBig><<<rbig, kFxThreads, 0, st>>>(P.d_mats, P.d_fxr + r64, status_dev, pass);
            };
            gram(1);
            k_fx_chol1<<<n, kCholThreads, 0, st>>>(P.d_mats, status_dev, col_tol);
            rmul(1);
            gram(2);
            k_fx_chol2<<<n, kCholThreads, 0, st>>>(P.d_mats, status_dev);
            rmul(2);
            EDGC_LAUNCH_CHECK();
        }
    }
    if (phases & EDGC_PHASE_PASS2) {
        if ((rc = launch_pass2(P, true, status_dev, st))) return rc;
        if ((rc = launch_pass2(P, false, status_dev, st))) return rc;
        if (!P.sq[0].empty()) {
            if ((rc = launch_skinny<1, kSkQRows16, 16>((unsigned)P.sq[0].size(), st, P.d_mats, P.d_sq[0], status_dev))) return rc;
            EDGC_LAUNCH_CHECK();
        }
        if (!P.sq[1].empty()) {
            if ((rc = launch_skinny<1, kSkQRows32, 32>((unsigned)P.sq[1].size(), st, P.d_mats, P.d_sq[1], status_dev))) return rc;
            EDGC_LAUNCH_CHECK();
        }
        if (!P.sq[2].empty()) {
            if ((rc = launch_skinny<1, kSkQRows8, 8>((unsigned)P.sq[2].size(), st, P.d_mats, P.d_sq[2], status_dev))) return rc;
            EDGC_LAUNCH_CHECK();
        }
        if ((rc = launch_gemm<1>(P, P.gq, P.d_gq, status_dev, st))) return rc;
        if (!P.tcq[0].empty())
            EDGC_CUDA_TRY((tc::launch<64, 4>(TcQ{P.d_mats, P.d_tcq[0], status_dev, (int)P.tcq[0].size()}, sm_count(), st)));
        if (!P.tcq[1].empty())
            EDGC_CUDA_TRY((tc::launch<128, 4>(TcQ{P.d_mats, P.d_tcq[1], status_dev, (int)P.tcq[1].size()}, sm_count(), st)));
    }
    if (phases & EDGC_PHASE_FINALIZE) {
        // one matrix (the per-matrix API): its blocks directly (measured 4 us faster there than
        // the table lookup); several: the flat table
        if (n == 1)
            k_finalize<<<(unsigned)P.fin.size(), kFinThreads, 0, st>>>(P.d_mats, nullptr, status_dev);
        else
            k_finalize<<<(unsigned)P.fin.size(), kFinThreads, 0, st>>>(P.d_mats, P.d_fin, status_dev);
        EDGC_LAUNCH_CHECK();
    }
    return EDGC_OK;
}

extern "C" int64_t edgc_compress_plan_sample_slots(const edgc_compress_plan *h) {
    return (h && h->P.d_mats) ? h->P.sample_slots : -1;
}

extern "C" int edgc_compress_plan_set_sampling(edgc_compress_plan *h, const edgc_sample_desc *descs, int n,
                                               double *partials_dev, void *stream) {
    EDGC_REQUIRE(h && h->P.d_mats && descs && partials_dev, "edgc_compress_plan_set_sampling: bad arguments");
    Plan &P = h->P;
    EDGC_REQUIRE(n == (int)h->descs.size(), "edgc_compress_plan_set_sampling: %d descriptors for a %d-matrix plan", n,
                 (int)h->descs.size());
    EDGC_REQUIRE(P.sample_slots > 0, "edgc_compress_plan_set_sampling: a matrix of this plan is off the Z path");
    P.samp_host.resize(n);
    for (int k = 0; k < n; ++k)
        P.samp_host[k] = SampDev{descs[k].bitmap, descs[k].first, partials_dev + 2 * P.sample_slots * (int64_t)k};
    EDGC_CUDA_TRY(cudaMemcpyAsync(P.d_samp, P.samp_host.data(), sizeof(SampDev) * n, cudaMemcpyHostToDevice,
                                  (cudaStream_t)stream));
    P.sample_armed = true;
    return EDGC_OK;
}

extern "C" void edgc_compress_plan_destroy(edgc_compress_plan *h) { delete h; }

extern "C" int64_t edgc_compress_workspace_bytes(const edgc_compress_desc *descs, int n) {
    Plan P;
    if (n < 0 || make_plan(descs, n, nullptr, INT64_MAX, P) != EDGC_OK) return -1;
    return P.bytes;
}

extern "C" int edgc_compress(const edgc_compress_desc *descs, int n, double col_tol, int32_t *status_dev, void *ws,
                             int64_t ws_bytes, void *stream) {
    if (n == 0) return EDGC_OK;
    edgc_compress_plan *h = nullptr;
    int rc = edgc_compress_plan_create(descs, n, &h);
    if (rc != EDGC_OK) return rc;
    rc = edgc_compress_plan_bind(h, ws, ws_bytes, stream);
    if (rc == EDGC_OK) rc = edgc_compress_plan_run(h, col_tol, status_dev, EDGC_PHASE_ALL, stream);
    edgc_compress_plan_destroy(h);
    return rc;
}

namespace {
struct RPlan {
    std::vector<ReconDev> d;
    std::vector<RTile> tiles, tiles4;
    int64_t bytes = 0;
    ReconDev *dd = nullptr;
    RTile *dt = nullptr, *dt4 = nullptr, *dtT = nullptr, *dtc = nullptr;
    std::vector<RTile> tilesT;        // k_recon_tiled (W*r > 8, float4-aligned output)
    std::vector<RTile> tilesC;        // TcRecon (W*r above the tensor-core threshold)
};
int make_rplan(const edgc_recon_desc *descs, int n, void *ws, RPlan &P) {
    Arena a(ws, INT64_MAX);
    P.tiles.clear();
    P.tiles4.clear();
    P.tilesT.clear();
    P.tilesC.clear();
    P.d.resize(n);
    P.dd = a.take<ReconDev>(n);
    int wr4max = 0;   // as edgc_recon_plan_create's wr4
    for (int k = 0; k < n; ++k)
        if (descs[k].r * descs[k].n_ranks <= 32) wr4max = std::max(wr4max, descs[k].r * descs[k].n_ranks);
    for (int k = 0; k < n; ++k) {
        const edgc_recon_desc &s = descs[k];
        EDGC_REQUIRE(s.m >= 1 && s.n >= 1 && s.r >= 1 && s.n_ranks >= 1 && s.p && s.q && s.out && s.ld_out >= s.n,
                     "recon desc %d: bad arguments", k);
        P.d[k] = ReconDev{s.p, s.q, s.out, s.m, s.n, s.ld_out, s.p_rank_stride, s.q_rank_stride, s.r, s.n_ranks,
                          s.scale};
        const bool v4 = s.r * s.n_ranks <= 32 && s.n % 4 == 0 && s.ld_out % 4 == 0 && ((uintptr_t)s.out % 16 == 0);
        // tensor cores once W r passes the recon threshold (CUDA-core FMA bound beyond it); with
        // W > 1 the K index concatenates the ranks' r-wide blocks (float4 loads per block: 4 | r)
        const bool tcr = s.r * s.n_ranks >= tc_recon_min() && s.r % 4 == 0;
        if (tcr) {
            for (int64_t r0 = 0; r0 < s.m; r0 += tc::kBM)
                for (int64_t c0 = 0; c0 < s.n; c0 += 128)
                    P.tilesC.push_back(RTile{k, c0, std::min(s.n, c0 + 128), r0, std::min(s.m, r0 + tc::kBM)});
        } else if (v4) {
            // the launch's kernel is chosen by the largest W r of the float4 tiles: its tile height
            // (shared-memory P tile) bounds every tile's rows
            const int wrc = wr4max <= 4 ? 4 : wr4max <= 8 ? 8 : wr4max <= 16 ? 16 : 32;
            const int64_t tr = v4_tile_rows(wrc), tc = (int64_t)kV4Cols * v4_col_blocks(wrc);
            for (int64_t c0 = 0; c0 < s.n; c0 += tc)
                for (int64_t r0 = 0; r0 < s.m; r0 += tr)
                    P.tiles4.push_back(RTile{k, c0, std::min(s.n, c0 + tc), r0, std::min(s.m, r0 + tr)});
        } else if (s.n % 4 == 0 && s.ld_out % 4 == 0 && ((uintptr_t)s.out % 16 == 0)) {
            for (int64_t r0 = 0; r0 < s.m; r0 += kGT)
                for (int64_t c0 = 0; c0 < s.n; c0 += kGT)
                    P.tilesT.push_back(RTile{k, c0, std::min(s.n, c0 + kGT), r0, std::min(s.m, r0 + kGT)});
        } else {
            for (int64_t c0 = 0; c0 < s.n; c0 += kRThreads)
                for (int64_t r0 = 0; r0 < s.m; r0 += kRTileRows)
                    P.tiles.push_back(RTile{k, c0, std::min(s.n, c0 + kRThreads), r0, std::min(s.m, r0 + kRTileRows)});
        }
    }
    P.dt = a.take<RTile>(P.tiles.size());
    P.dt4 = a.take<RTile>(P.tiles4.size());
    P.dtT = a.take<RTile>(P.tilesT.size());
    P.dtc = a.take<RTile>(P.tilesC.size());
    P.bytes = a.off;
    return EDGC_OK;
}
}  // namespace

struct edgc_recon_plan {
    std::vector<edgc_recon_desc> descs;
    RPlan P;
    int wr = 0, wr4 = 0;
};

extern "C" int edgc_recon_plan_create(const edgc_recon_desc *descs, int n, edgc_recon_plan **out) {
    EDGC_REQUIRE(out && n >= 1 && descs, "edgc_recon_plan_create: bad arguments");
    auto *h = new edgc_recon_plan();
    h->descs.assign(descs, descs + n);
    int rc = make_rplan(descs, n, nullptr, h->P);
    if (rc != EDGC_OK) { delete h; return rc; }
    for (int k = 0; k < n; ++k) {
        const int wr = descs[k].r * descs[k].n_ranks;
        if (wr <= 32) h->wr4 = std::max(h->wr4, wr);
        h->wr = std::max(h->wr, wr);
    }
    *out = h;
    return EDGC_OK;
}

extern "C" int64_t edgc_recon_plan_workspace_bytes(const edgc_recon_plan *h) { return h ? h->P.bytes : -1; }

extern "C" int edgc_recon_plan_bind(edgc_recon_plan *h, void *ws, int64_t ws_bytes, void *stream) {
    EDGC_REQUIRE(h && ws && ws_bytes >= h->P.bytes, "edgc_recon_plan_bind: workspace");
    RPlan &P = h->P;
    P = RPlan();
    int rc = make_rplan(h->descs.data(), (int)h->descs.size(), ws, P);
    if (rc != EDGC_OK) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    EDGC_CUDA_TRY(cudaMemcpyAsync(P.dd, P.d.data(), sizeof(ReconDev) * P.d.size(), cudaMemcpyHostToDevice, st));
    if (!P.tiles.empty())
        EDGC_CUDA_TRY(
            cudaMemcpyAsync(P.dt, P.tiles.data(), sizeof(RTile) * P.tiles.size(), cudaMemcpyHostToDevice, st));
    if (!P.tiles4.empty())
        EDGC_CUDA_TRY(
            cudaMemcpyAsync(P.dt4, P.tiles4.data(), sizeof(RTile) * P.tiles4.size(), cudaMemcpyHostToDevice, st));
    if (!P.tilesT.empty())
        EDGC_CUDA_TRY(
            cudaMemcpyAsync(P.dtT, P.tilesT.data(), sizeof(RTile) * P.tilesT.size(), cudaMemcpyHostToDevice, st));
    if (!P.tilesC.empty())
        EDGC_CUDA_TRY(
            cudaMemcpyAsync(P.dtc, P.tilesC.data(), sizeof(RTile) * P.tilesC.size(), cudaMemcpyHostToDevice, st));
    EDGC_CUDA_TRY(cudaStreamSynchronize(st));
    return EDGC_OK;
}

extern "C" int edgc_recon_plan_run(edgc_recon_plan *h, void *stream) {
    EDGC_REQUIRE(h && h->P.dd, "edgc_recon_plan_run: plan not bound");
    cudaStream_t st = (cudaStream_t)stream;
    if (!h->P.tiles4.empty()) {
        const unsigned g4 = (unsigned)h->P.tiles4.size();
        constexpr size_t s4 = 4 * v4_tile_rows(4) * sizeof(float), s8 = 8 * v4_tile_rows(8) * sizeof(float);
        constexpr size_t s16 = 16 * v4_tile_rows(16) * sizeof(float), s32 = 32 * v4_tile_rows(32) * sizeof(float);
        static uint64_t a32 = 0;
        int rc;
        if (h->wr4 <= 4) k_recon4<4, 4><<<g4, kV4Cols / 4, s4, st>>>(h->P.dd, h->P.dt4);
        else if (h->wr4 <= 8) k_recon4<8, 4><<<g4, kV4Cols / 4, s8, st>>>(h->P.dd, h->P.dt4);
        else if (h->wr4 <= 16) {
            static uint64_t a16 = 0;
            if ((rc = smem_attr_once(k_recon4<16, 4>, (int)s16, a16))) return rc;
            k_recon4<16, 4><<<g4, kV4Cols / 4, s16, st>>>(h->P.dd, h->P.dt4);
        }
        else {
            if ((rc = smem_attr_once(k_recon4<32, 2>, (int)s32, a32))) return rc;
            k_recon4<32, 2><<<g4, kV4Cols / 2, s32, st>>>(h->P.dd, h->P.dt4);
        }
        EDGC_LAUNCH_CHECK();
    }
    if (!h->P.tiles.empty()) {
        const unsigned grid = (unsigned)h->P.tiles.size();
        if (h->wr <= 4) k_recon<4><<<grid, kRThreads, 0, st>>>(h->P.dd, h->P.dt);
        else if (h->wr <= 8) k_recon<8><<<grid, kRThreads, 0, st>>>(h->P.dd, h->P.dt);
        else if (h->wr <= 16) k_recon<16><<<grid, kRThreads, 0, st>>>(h->P.dd, h->P.dt);
        else k_recon<32><<<grid, kRThreads, 0, st>>>(h->P.dd, h->P.dt);
        EDGC_LAUNCH_CHECK();
    }
    if (!h->P.tilesT.empty()) {
        k_recon_tiled<<<(unsigned)h->P.tilesT.size(), kGThreads, 0, st>>>(h->P.dd, h->P.dtT);
        EDGC_LAUNCH_CHECK();
    }
    if (!h->P.tilesC.empty())
        EDGC_CUDA_TRY((tc::launch<128, 4>(TcRecon{h->P.dd, h->P.dtc, (int)h->P.tilesC.size()}, sm_count(), st)));
    return EDGC_OK;
}

namespace edgc {
namespace {
__global__ void k_p2p_signal(int64_t *const *peer_flags, int me, int nranks, int64_t *counter) {
    // this rank's factors (written by the kernels before this one on the stream) are complete:
    // publish the next step number into slot `me` of every rank's flags, release at system
    // scope, and advance this rank's device counter (graph replays see the live count)
    const int w = threadIdx.x;
    const int64_t epoch = *counter + 1;
    __syncthreads();
    if (w < nranks) {
        __threadfence_system();
        asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(peer_flags[w] + me), "l"(epoch) : "memory");
    }
    __syncthreads();
    if (w == 0) *counter = epoch;
}
}  // namespace
}  // namespace edgc

namespace edgc {
namespace {
// gathered[w * n .. (w + 1) * n) <- rank w's buffer, read over NVLink once rank w's flag for this
// step is up: kPullCtas CTAs per rank, 16-byte loads (8 in flight per thread), local stores
constexpr int kPullCtas = 32, kPullThreads = 256;
__global__ void __launch_bounds__(kPullThreads) k_p2p_pull(const float *const *bases, float *gathered, int64_t n,
                                                           const int64_t *flags, const int64_t *counter) {
    const int w = blockIdx.y;
    if (threadIdx.x == 0) {
        const int64_t epoch = *counter;   // this rank's step number, advanced by its k_p2p_signal
        while (ld_acquire_sys(flags + w) < epoch) __nanosleep(64);
    }
    __syncthreads();
    const float *src = bases[w];
    float *dst = gathered + (int64_t)w * n;
    const int64_t n4 = ((uintptr_t)src % 16 == 0 && (uintptr_t)dst % 16 == 0) ? n / 4 : 0;
    const int64_t stride = (int64_t)kPullCtas * kPullThreads;
    const float4 *s4 = reinterpret_cast<const float4 *>(src);
    float4 *d4 = reinterpret_cast<float4 *>(dst);
    for (int64_t i0 = (int64_t)blockIdx.x * kPullThreads + threadIdx.x; i0 < n4; i0 += 8 * stride) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (i0 + u * stride < n4) v[u] = __ldcv(s4 + i0 + u * stride);   // volatile: never a stale L1 line
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (i0 + u * stride < n4) d4[i0 + u * stride] = v[u];
    }
    for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * kPullThreads + threadIdx.x; i < n; i += stride)
        dst[i] = __ldcv(src + i);
}
}  // namespace
}  // namespace edgc

extern "C" int edgc_p2p_pull(const float *const *bases_dev, float *gathered, int64_t n, int nranks,
                             const int64_t *flags_dev, const int64_t *counter_dev, void *stream) {
    EDGC_REQUIRE(bases_dev && gathered && flags_dev && counter_dev && n >= 0 && nranks >= 1,
                 "edgc_p2p_pull: bad arguments");
    if (n == 0) return EDGC_OK;
    k_p2p_pull<<<dim3(kPullCtas, nranks), kPullThreads, 0, (cudaStream_t)stream>>>(bases_dev, gathered, n, flags_dev,
                                                                                  counter_dev);
    EDGC_LAUNCH_CHECK();
    return EDGC_OK;
}

extern "C" int edgc_p2p_signal(int64_t *const *peer_flags_dev, int me, int nranks, int64_t *counter_dev, void *stream) {
    EDGC_REQUIRE(peer_flags_dev && counter_dev && nranks >= 1 && nranks <= 1024 && me >= 0 && me < nranks,
                 "edgc_p2p_signal: bad arguments");
    k_p2p_signal<<<1, ((nranks + 31) / 32) * 32, 0, (cudaStream_t)stream>>>(peer_flags_dev, me, nranks, counter_dev);
    EDGC_LAUNCH_CHECK();
    return EDGC_OK;
}

// cuMemGetAddressRange through the runtime's driver entry point (no libcuda link)
typedef int (*MemRangeFn)(unsigned long long *base, size_t *size, unsigned long long dptr);

extern "C" int edgc_ipc_handle(const void *ptr, void *handle64, int64_t *offset) {
    EDGC_REQUIRE(ptr && handle64 && offset, "edgc_ipc_handle: bad arguments");
    static MemRangeFn range = nullptr;
    if (!range) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        EDGC_CUDA_TRY(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
        EDGC_REQUIRE(fn && q == cudaDriverEntryPointSuccess, "edgc_ipc_handle: cuMemGetAddressRange unavailable");
        range = (MemRangeFn)fn;
    }
    unsigned long long base = 0;
    size_t size = 0;
    EDGC_REQUIRE(range(&base, &size, (unsigned long long)(uintptr_t)ptr) == 0,
                 "edgc_ipc_handle: cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    EDGC_CUDA_TRY(cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base));
    memcpy(handle64, &h, sizeof(h));
    *offset = (int64_t)((uintptr_t)ptr - (uintptr_t)base);
    return EDGC_OK;
}

extern "C" int edgc_ipc_open(const void *handle64, void **ptr) {
    EDGC_REQUIRE(handle64 && ptr, "edgc_ipc_open: bad arguments");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof(h));
    EDGC_CUDA_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return EDGC_OK;
}

extern "C" int edgc_ipc_close(void *ptr) {
    EDGC_REQUIRE(ptr, "edgc_ipc_close: null pointer");
    EDGC_CUDA_TRY(cudaIpcCloseMemHandle(ptr));
    return EDGC_OK;
}

extern "C" void edgc_recon_plan_destroy(edgc_recon_plan *h) { delete h; }

extern "C" int64_t edgc_reconstruct_workspace_bytes(const edgc_recon_desc *descs, int n) {
    RPlan P;
    if (n < 0 || make_rplan(descs, n, nullptr, P) != EDGC_OK) return -1;
    return P.bytes;
}

extern "C" int edgc_reconstruct(const edgc_recon_desc *descs, int n, void *ws, int64_t ws_bytes, void *stream) {
    if (n == 0) return EDGC_OK;
    edgc_recon_plan *h = nullptr;
    int rc = edgc_recon_plan_create(descs, n, &h);
    if (rc != EDGC_OK) return rc;
    rc = edgc_recon_plan_bind(h, ws, ws_bytes, stream);
    if (rc == EDGC_OK) rc = edgc_recon_plan_run(h, stream);
    edgc_recon_plan_destroy(h);
    return rc;
}

extern "C" int edgc_residual(const float *w, const float *p_res, const float *q_res, int32_t r_res, int64_t m,
                             int64_t n, float *e_out, void *stream) {
    EDGC_REQUIRE(w && e_out && m >= 1 && n >= 1 && r_res >= 0 && (r_res == 0 || (p_res && q_res)),
                 "edgc_residual: bad arguments");
    k_residual<<<elementwise_blocks(m * n), 256, 0, (cudaStream_t)stream>>>(w, p_res, q_res, r_res, m, n, e_out);
    EDGC_LAUNCH_CHECK();
    return EDGC_OK;
}

extern "C" int edgc_check_work_finite(const float *g, int64_t ld_g, const float *w, const float *p_res,
                                      const float *q_res, int32_t r_res, int64_t m, int64_t n, int32_t *flag_dev,
                                      void *stream) {
    EDGC_REQUIRE(g && w && flag_dev && m >= 1 && n >= 1 && ld_g >= n && (r_res == 0 || (p_res && q_res)),
                 "edgc_check_work_finite: bad arguments");
    const unsigned gx = (unsigned)std::min<int64_t>(ceil_div(n, 256), 8);
    const unsigned gy = (unsigned)std::min<int64_t>(m, std::max<int64_t>(1, (int64_t)sm_count() * 8 / gx));
    k_check_work<<<dim3(gx, gy), 256, 0, (cudaStream_t)stream>>>(g, ld_g, w, p_res, q_res, r_res, m, n, flag_dev);
    EDGC_LAUNCH_CHECK();
    return EDGC_OK;
}

extern "C" int edgc_check_finite(int dtype, const void *x, int64_t count, int32_t *flag_dev, void *stream) {
    EDGC_REQUIRE((dtype == 0 || dtype == 1) && flag_dev && count >= 0, "edgc_check_finite: bad arguments");
    if (count == 0) return EDGC_OK;
    if (dtype == 0)
        k_check_finite<float><<<elementwise_blocks(count), 256, 0, (cudaStream_t)stream>>>((const float *)x, count,
                                                                                          flag_dev);
    else
        k_check_finite<double><<<elementwise_blocks(count), 256, 0, (cudaStream_t)stream>>>((const double *)x, count,
                                                                                           flag_dev);
    EDGC_LAUNCH_CHECK();
    return EDGC_OK;
}
