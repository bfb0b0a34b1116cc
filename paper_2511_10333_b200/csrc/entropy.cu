// Entropy estimators on the device.
//
// Gaussian plug-in (default estimator, entropy.py:82-90 / :143): fused
// gather + fp64 reduction, batched over all layers of one sampled iteration.
// FD histogram (entropy.py:93-107 -> np.histogram(x, bins="fd")): order
// statistics by 4-target radix select, NumPy's fp64 edge/index arithmetic with
// separately rounded operations (no FMA contraction), warp-aggregated shared-
// memory atomics for the counts, fp64 entropy reduction.  Counts and edges are
// bit-exact with NumPy 2.3.5 (restated in oracle/oracle.py:fd_histogram).
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace edgc {
namespace {

constexpr double kGaussConst = 1.4189385332046727;  // 0.5 * ln(2*pi*e), entropy.py:24
constexpr int kRedThreads = 256;
// Many blocks per layer, layers in blockIdx.y order: the whole GPU gathers from
// one or two matrices at a time, so their sectors stay in L2 and each matrix is
// read from DRAM about once (a scattered gather over all layers at once thrashes
// L2 and moves ~30x the algorithmic bytes).
#ifndef EDGC_GAUSS_UNROLL
#define EDGC_GAUSS_UNROLL 8   // measured 4: 2.16 ms, 2: 1.75, 8: 1.74 (GPT2-2.5B set)
#endif
#ifndef EDGC_GAUSS_BLOCKS
#define EDGC_GAUSS_BLOCKS 1184
#endif
constexpr int kGaussBlocksPerDesc = EDGC_GAUSS_BLOCKS;   // 8 x 148 SMs, persistent over layers

// ---------------------------------------------------------------- Gaussian
struct GaussDev {
    const void *src;
    const int32_t *idx;
    int64_t count;
    const uint32_t *bitmap;
    int64_t n_elems;
};

template <typename T>
__device__ __forceinline__ double load_sample(const GaussDev &d, int64_t i) {
    const int64_t k = d.idx ? (int64_t)__ldg(d.idx + i) : i;
    return (double)__ldg(reinterpret_cast<const T *>(d.src) + k);
}

// partial[desc][block] = {sum(x-K), sum((x-K)^2)} with the shift K = first sample
template <typename T>
__global__ void __launch_bounds__(kRedThreads) k_gauss_partial(const GaussDev *descs, int ndesc, double2 *partial) {
    // one persistent grid walks the layers in order (layer-major: the whole GPU
    // works on one matrix at a time, which keeps a gather's sectors in L2)
    for (int di = 0; di < ndesc; ++di) {
    const GaussDev d = descs[di];
    double s1 = 0.0, s2 = 0.0;
    if (d.count > 0 && d.bitmap && sizeof(T) == 4 && ((uintptr_t)d.src & 15) == 0) {
        // stream the whole matrix against the plan's membership bits: each lane reads 4
        // consecutive elements (16 bytes) and their 4 bits, 4 loads in flight per thread
        const double K = load_sample<T>(d, 0);
        const float4 *src4 = reinterpret_cast<const float4 *>(d.src);
        const int64_t nq = d.n_elems / 4;
        const int64_t stride = (int64_t)gridDim.x * kRedThreads;
        int64_t q = (int64_t)blockIdx.x * kRedThreads + threadIdx.x;
        auto take = [&](const float4 &v, uint32_t bits) {
            const float f[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if ((bits >> k) & 1u) {
                    const double x = (double)f[k] - K;
                    s1 += x;
                    s2 += x * x;
                }
        };
        constexpr int U = EDGC_GAUSS_UNROLL;   // float4 loads in flight per thread
        for (; q + (U - 1) * stride < nq; q += U * stride) {
            float4 v[U];
            uint32_t bw[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int64_t qq = q + k * stride;
                v[k] = __ldg(src4 + qq);
                bw[k] = __ldg(d.bitmap + (qq >> 3)) >> ((qq & 7) * 4);
            }
#pragma unroll
            for (int k = 0; k < U; ++k) take(v[k], bw[k]);
        }
        for (; q < nq; q += stride) take(__ldg(src4 + q), __ldg(d.bitmap + (q >> 3)) >> ((q & 7) * 4));
        const int64_t e = 4 * nq + threadIdx.x;   // ragged tail (< 4 elements)
        if (blockIdx.x == 0 && e < d.n_elems && ((__ldg(d.bitmap + (e >> 5)) >> (e & 31)) & 1u)) {
            const double x = (double)__ldg(reinterpret_cast<const float *>(d.src) + e) - K;
            s1 += x;
            s2 += x * x;
        }
    } else if (d.count > 0 && d.bitmap) {
        // stream the whole matrix, keep the plan's members: coalesced reads
        // instead of a random gather (a 4-byte gather moves ~64-128 bytes of DRAM)
        const double K = load_sample<T>(d, 0);
        const T *src = reinterpret_cast<const T *>(d.src);
        const int64_t nw = (d.n_elems + 31) / 32;
        const int lane = threadIdx.x & 31;
        const int64_t wstride = (int64_t)gridDim.x * (kRedThreads / 32);
        int64_t wi = (int64_t)blockIdx.x * (kRedThreads / 32) + (threadIdx.x >> 5);
        // one bitmap word per warp iteration: lane l owns element 32 wi + l (coalesced 128-byte reads)
        for (; wi + 3 * wstride < nw; wi += 4 * wstride) {
            uint32_t bw[4];
            double v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t w = wi + q * wstride;
                bw[q] = __ldg(d.bitmap + w);
                const int64_t e = w * 32 + lane;
                v[q] = (e < d.n_elems) ? (double)__ldg(src + e) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if ((bw[q] >> lane) & 1u) {
                    const double x = v[q] - K;
                    s1 += x;
                    s2 += x * x;
                }
        }
        for (; wi < nw; wi += wstride) {
            const uint32_t bw = __ldg(d.bitmap + wi);
            const int64_t e = wi * 32 + lane;
            if (e < d.n_elems && ((bw >> lane) & 1u)) {
                const double x = (double)__ldg(src + e) - K;
                s1 += x;
                s2 += x * x;
            }
        }
    } else if (d.count > 0) {
        const double K = load_sample<T>(d, 0);
        const int64_t stride = (int64_t)gridDim.x * kRedThreads;
        int64_t i = (int64_t)blockIdx.x * kRedThreads + threadIdx.x;
        // 4 independent loads in flight per thread
        for (; i + 3 * stride < d.count; i += 4 * stride) {
            double v0 = load_sample<T>(d, i) - K, v1 = load_sample<T>(d, i + stride) - K;
            double v2 = load_sample<T>(d, i + 2 * stride) - K, v3 = load_sample<T>(d, i + 3 * stride) - K;
            s1 += (v0 + v1) + (v2 + v3);
            s2 += (v0 * v0 + v1 * v1) + (v2 * v2 + v3 * v3);
        }
        for (; i < d.count; i += stride) {
            double v = load_sample<T>(d, i) - K;
            s1 += v;
            s2 += v * v;
        }
    }
    // one partial per warp (no block barrier between layers, so the load stream does not drain
    // at every matrix boundary); k_gauss_finish sums them in a fixed order
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0)
        partial[((int64_t)di * gridDim.x + blockIdx.x) * (kRedThreads / 32) + warp] = make_double2(s1, s2);
    }
}

__global__ void k_gauss_finish(const GaussDev *descs, int n, const double2 *partial, int nblk, double *h_out,
                               int32_t *status) {
    // a warp per descriptor: lane-strided partial sums, then a fixed shuffle tree (deterministic)
    const int i = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
    if (i >= n) return;
    const int64_t cnt = descs[i].count;
    double s1 = 0.0, s2 = 0.0;
    for (int b = lane; b < nblk; b += 32) { s1 += partial[(int64_t)i * nblk + b].x; s2 += partial[(int64_t)i * nblk + b].y; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane != 0) return;
    if (cnt < 2) { status[i] = EDGC_EINVAL; h_out[i] = NAN; return; }
    const double nn = (double)cnt;
    double var = (s2 - s1 * (s1 / nn)) / (nn - 1.0);
    if (var < 0.0) var = 0.0;
    const double sigma = sqrt(var);
    if (sigma == 0.0) { status[i] = EDGC_EDEGENERATE; h_out[i] = NAN; return; }
    status[i] = EDGC_OK;
    h_out[i] = log(sigma) + kGaussConst;
}

// fused partials (edgc_compress_plan_set_sampling): slots summed in fixed order
__global__ void k_gauss_finish_slots(const double *part, int64_t slots, const int64_t *counts, int n, double *h_out,
                                     int32_t *status) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t cnt = counts[i];
    if (cnt < 2) { status[i] = EDGC_EINVAL; h_out[i] = NAN; return; }
    double s1 = 0.0, s2 = 0.0;
    for (int64_t b = 0; b < slots; ++b) { s1 += part[(i * slots + b) * 2]; s2 += part[(i * slots + b) * 2 + 1]; }
    const double nn = (double)cnt;
    double var = (s2 - s1 * (s1 / nn)) / (nn - 1.0);
    if (var < 0.0) var = 0.0;
    const double sigma = sqrt(var);
    if (sigma == 0.0) { status[i] = EDGC_EDEGENERATE; h_out[i] = NAN; return; }
    status[i] = EDGC_OK;
    h_out[i] = log(sigma) + kGaussConst;
}

// --------------------------------------------------------------- histogram
// independent element loads in flight per thread in the streaming histogram passes
constexpr int kHistUnroll = 8;
// radix-select digit width: 11 bits -> three passes for fp32 keys (6 for fp64)
constexpr int kDigitBits = 11;
constexpr int kDigits = 1 << kDigitBits;

template <typename T> struct KeyOf;
template <> struct KeyOf<float> {
    typedef uint32_t K;
    static constexpr int kBits = 32;
    __device__ static K key(float x) {
        uint32_t b = __float_as_uint(x);
        return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    }
    __device__ static double value(K k) {
        uint32_t b = (k & 0x80000000u) ? (k ^ 0x80000000u) : ~k;
        return (double)__uint_as_float(b);
    }
};
template <> struct KeyOf<double> {
    typedef unsigned long long K;
    static constexpr int kBits = 64;
    __device__ static K key(double x) {
        unsigned long long b = (unsigned long long)__double_as_longlong(x);
        return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    }
    __device__ static double value(K k) {
        unsigned long long b = (k >> 63) ? (k ^ 0x8000000000000000ull) : ~k;
        return __longlong_as_double((long long)b);
    }
};

struct HistState {
    // order statistics: targets 0..3 = ranks lo25, lo25+1, lo75, lo75+1
    unsigned long long prefix[4];
    long long rank[4];
    double minv, maxv;
    double first, last, delta, step, width;
    long long nb;
    int fixed;
};

template <typename T>
__global__ void __launch_bounds__(kRedThreads) k_minmax(const T *x, int64_t n, double2 *partial) {
    double lo = INFINITY, hi = -INFINITY;
    const int64_t stride = (int64_t)gridDim.x * kRedThreads, base = (int64_t)blockIdx.x * kRedThreads + threadIdx.x;
    const int64_t n_iter = (n + stride - 1) / stride;
    for (int64_t it0 = 0; it0 < n_iter; it0 += kHistUnroll) {
        T v[kHistUnroll];  // independent loads in flight; out-of-range lanes repeat x[0] (min/max-neutral)
#pragma unroll
        for (int u = 0; u < kHistUnroll; ++u) {
            const int64_t i = (it0 + u) * stride + base;
            v[u] = __ldg(x + (i < n ? i : 0));
        }
#pragma unroll
        for (int u = 0; u < kHistUnroll; ++u) {
            // NaN is skipped by fmin/fmax: fold it into the max as +inf so the range is non-finite
            lo = fmin(lo, (double)v[u]);
            hi = fmax(hi, v[u] != v[u] ? (double)INFINITY : (double)v[u]);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    __shared__ double2 s[kRedThreads / 32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = make_double2(lo, hi);
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kRedThreads / 32; ++w) { lo = fmin(lo, s[w].x); hi = fmax(hi, s[w].y); }
        lo = fmin(lo, s[0].x);
        hi = fmax(hi, s[0].y);
        partial[blockIdx.x] = make_double2(lo, hi);
    }
}

// one warp: strided partial min/max, then a shuffle reduction (fmin/fmax are exact)
__device__ __forceinline__ double2 warp_minmax(const double2 *mm, int nblk) {
    double lo = INFINITY, hi = -INFINITY;
    for (int b = threadIdx.x & 31; b < nblk; b += 32) { lo = fmin(lo, mm[b].x); hi = fmax(hi, mm[b].y); }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    return make_double2(lo, hi);
}

// mm == NULL: the min/max comes later, from the first radix pass (k_radix_pick)
__global__ void k_hist_init(HistState *st, const double2 *mm, int nblk, int64_t n, int fixed, int32_t *status,
                            double *result) {
    double lo = 0.0, hi = 1.0;
    if (mm) {
        const double2 r = warp_minmax(mm, nblk);
        lo = r.x;
        hi = r.y;
    }
    if (threadIdx.x != 0) return;
    st->minv = lo;
    st->maxv = hi;
    st->fixed = fixed;
    // numpy percentile 'linear': virtual index (n-1)*q, floor, +1
    const double v25 = (double)(n - 1) * 0.25, v75 = (double)(n - 1) * 0.75;
    const long long l25 = (long long)floor(v25), l75 = (long long)floor(v75);
    st->rank[0] = l25;
    st->rank[1] = min(l25 + 1, (long long)n - 1);
    st->rank[2] = l75;
    st->rank[3] = min(l75 + 1, (long long)n - 1);
    for (int t = 0; t < 4; ++t) st->prefix[t] = 0ull;
    *status = EDGC_OK;
    if (n < 2) *status = EDGC_EINVAL;
    else if (mm && !(isfinite(lo) && isfinite(hi))) *status = EDGC_ENONFINITE;  // np.histogram: range not finite
    else if (lo == hi) *status = EDGC_EDEGENERATE;
    for (int i = 0; i < 5; ++i) result[i] = NAN;
}

// one radix-select digit pass (8-bit digits, most significant first)
template <typename T, bool kMinMax>
__global__ void __launch_bounds__(kRedThreads) k_radix_hist(const T *x, int64_t n, const HistState *st, int shift,
                                                           int width, unsigned int *ghist /*[4][kDigits]*/,
                                                           double2 *mm_out /* first pass: per-CTA min/max */) {
    typedef typename KeyOf<T>::K K;
    __shared__ unsigned int h[4][kDigits];
    for (int i = threadIdx.x; i < 4 * kDigits; i += kRedThreads) (&h[0][0])[i] = 0u;
    __syncthreads();
    const int kbits = KeyOf<T>::kBits;
    const K hi_mask = (shift + width >= kbits) ? (K)0 : (K)(~(K)0) << (shift + width);
    // min/max fused into the first pass (mm_out), in T: exact, and fp32 min/max
    // avoids the fp64 pipe (the fused pass was SM-bound with double compares)
    T lo = T(INFINITY), hi = T(-INFINITY);
    const unsigned dmask = (1u << width) - 1u;
    K pre[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) pre[t] = (K)st->prefix[t];
    // Gaussian-like data puts most keys on a handful of digits (the first pass
    // sees only sign + exponent bits) and the four targets usually share their
    // prefix: aggregate per warp on (digit, target mask) so each distinct pair
    // costs one shared atomic per target instead of one per element and target.
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * kRedThreads;
    const int64_t n_iter = (n + stride - 1) / stride;
    const int64_t base = (int64_t)blockIdx.x * kRedThreads + threadIdx.x;
    for (int64_t it0 = 0; it0 < n_iter; it0 += kHistUnroll) {
        T v[kHistUnroll];  // kHistUnroll independent coalesced loads in flight per thread
#pragma unroll
        for (int u = 0; u < kHistUnroll; ++u) {
            const int64_t i = (it0 + u) * stride + base;
            v[u] = i < n ? __ldg(x + i) : T(0);
        }
#pragma unroll
        for (int u = 0; u < kHistUnroll; ++u) {
        const int64_t i = (it0 + u) * stride + base;
        if (kMinMax && i < n) {
            lo = fmin(lo, v[u]);
            hi = fmax(hi, v[u] != v[u] ? T(INFINITY) : v[u]);  // NaN -> non-finite range
        }
        unsigned tag = 0u;  // bits 0-10 digit, 12-15 matching targets; 0 = nothing to count
        if (i < n) {
            const K k = KeyOf<T>::key(v[u]);
            unsigned m = 0u;
#pragma unroll
            for (int t = 0; t < 4; ++t) m |= (((k ^ pre[t]) & hi_mask) == 0) ? (1u << t) : 0u;
            if (m) tag = ((unsigned)(k >> shift) & dmask) | (m << 12);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, tag);
        if (tag && lane == __ffs(peers) - 1) {
            const unsigned c = (unsigned)__popc(peers), dig = tag & 0x7FFu;
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (tag & (1u << (12 + t))) atomicAdd(&h[t][dig], c);
        }
        }
    }
    if constexpr (kMinMax) {
        __shared__ double2 s_mm[kRedThreads / 32];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) s_mm[threadIdx.x >> 5] = make_double2((double)lo, (double)hi);
        __syncthreads();
        if (threadIdx.x == 0) {
            double dlo = s_mm[0].x, dhi = s_mm[0].y;
            for (int w = 1; w < kRedThreads / 32; ++w) { dlo = fmin(dlo, s_mm[w].x); dhi = fmax(dhi, s_mm[w].y); }
            mm_out[blockIdx.x] = make_double2(dlo, dhi);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4 * kDigits; i += kRedThreads) {
        const unsigned v = (&h[0][0])[i];
        if (v) atomicAdd(ghist + i, v);
    }
}

__global__ void k_radix_pick(HistState *st, unsigned int *ghist, int shift, const double2 *mm, int nblk,
                             int32_t *status) {
    // warp t < 4 picks target t's digit: each lane owns kDigits/32 consecutive
    // digits, a warp scan of the lane sums finds the lane holding rank r
    __shared__ unsigned sh[4 * kDigits];  // coalesced staging, then zero the global counts
    for (int i = threadIdx.x; i < 4 * kDigits; i += blockDim.x) { sh[i] = ghist[i]; ghist[i] = 0u; }
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (mm && w == 4) {  // first pass: finish the fused min/max (k_hist_init's second half)
        const double2 r = warp_minmax(mm, nblk);
        if (lane == 0) {
            st->minv = r.x;
            st->maxv = r.y;
            if (*status == EDGC_OK && !(isfinite(r.x) && isfinite(r.y))) *status = EDGC_ENONFINITE;
            else if (*status == EDGC_OK && r.x == r.y) *status = EDGC_EDEGENERATE;
        }
    }
    if (w < 4) {
        const long long r = st->rank[w];
        constexpr int kPer = kDigits / 32;
        const unsigned *c = sh + w * kDigits + lane * kPer;
        long long local = 0;
#pragma unroll 16
        for (int j = 0; j < kPer; ++j) local += c[j];
        long long incl = local;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        long long cum = incl - local;
        if (cum <= r && r < incl) {
            int d = lane * kPer;
            for (int j = 0; j < kPer; ++j) {
                if (r < cum + c[j]) { d = lane * kPer + j; break; }
                cum += c[j];
            }
            st->prefix[w] |= ((unsigned long long)d) << shift;
            st->rank[w] = r - cum;
        }
    }
}

__device__ __forceinline__ double np_lerp(double a, double b, double t) {
    // numpy/lib/_function_base_impl.py:4657-4678, each op rounded separately
    const double diff = __dsub_rn(b, a);
    double out = __dadd_rn(a, __dmul_rn(diff, t));
    if (t >= 0.5) out = __dsub_rn(b, __dmul_rn(diff, __dsub_rn(1.0, t)));
    return out;
}

__device__ __forceinline__ double edge_at(const HistState &s, long long k) {
    // numpy/_core/function_base.py:139-172 (linspace): y = k*step + start, last = stop
    if (k >= s.nb) return s.last;
    if (s.step == 0.0) return __dadd_rn(__dmul_rn(__ddiv_rn((double)k, (double)s.nb), s.delta), s.first);
    return __dadd_rn(__dmul_rn((double)k, s.step), s.first);
}

template <typename T>
__global__ void k_hist_params(HistState *st, int64_t n, double inv_cbrt_n, long long fixed_bins, long long cap,
                              int32_t *status, double *result) {
    if (*status != EDGC_OK) return;
    typedef KeyOf<T> KO;
    double q[4];
    for (int t = 0; t < 4; ++t) q[t] = KO::value((typename KO::K)st->prefix[t]);
    const double v25 = __dmul_rn((double)(n - 1), 0.25), v75 = __dmul_rn((double)(n - 1), 0.75);
    const double g25 = __dsub_rn(v25, floor(v25)), g75 = __dsub_rn(v75, floor(v75));
    const double p25 = (v25 >= (double)(n - 1)) ? st->maxv : np_lerp(q[0], q[1], g25);
    const double p75 = (v75 >= (double)(n - 1)) ? st->maxv : np_lerp(q[2], q[3], g75);
    double first = st->minv, last = st->maxv;
    if (first == last) { first = __dsub_rn(first, 0.5); last = __dadd_rn(last, 0.5); }
    const double delta = __dsub_rn(last, first);
    long long nb;
    double width = 0.0;
    if (fixed_bins > 0) {
        nb = fixed_bins;
    } else {
        const double iqr = __dsub_rn(p75, p25);
        width = __dmul_rn(__dmul_rn(2.0, iqr), inv_cbrt_n);
        nb = (width != 0.0) ? (long long)ceil(__ddiv_rn(delta, width)) : 1;
    }
    st->first = first;
    st->last = last;
    st->delta = delta;
    st->nb = nb;
    st->width = width;
    st->step = __ddiv_rn(delta, (double)nb);
    result[1] = first;
    result[2] = last;
    result[3] = width;
    result[4] = (double)nb;
    if (nb > cap) *status = EDGC_ECAPACITY;
}

__global__ void k_hist_edges(const HistState *st, const int32_t *status, double *edges_out, int32_t *status_w) {
    if (*status != EDGC_OK) return;
    const HistState s = *st;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k <= s.nb;
         k += (long long)gridDim.x * blockDim.x) {
        const double e = edge_at(s, k);
        if (edges_out) edges_out[k] = e;
        if (k < s.nb && !(e < edge_at(s, k + 1))) *status_w = EDGC_ETOOMANYBINS;
    }
}

// numpy/lib/_histograms_impl.py:836-863: index, edge correction, bincount
template <typename T>
__device__ __forceinline__ long long bin_of(const HistState &s, double v) {
    const double f = __dmul_rn(__ddiv_rn(__dsub_rn(v, s.first), s.delta), (double)s.nb);
    long long idx = (long long)f;
    if (idx == s.nb) --idx;
    if (v < edge_at(s, idx)) --idx;
    if (idx != s.nb - 1 && v >= edge_at(s, idx + 1)) ++idx;
    return idx;
}

template <typename T>
__device__ __forceinline__ void k_hist_count_global_body(const T *x, int64_t n, const HistState &s, long long *counts,
                                                         int64_t block, int64_t nblocks) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = nblocks * kRedThreads;
    const int64_t n_iter = (n + stride - 1) / stride;
    for (int64_t it0 = 0; it0 < n_iter; it0 += kHistUnroll) {
        T v[kHistUnroll];
#pragma unroll
        for (int u = 0; u < kHistUnroll; ++u) {
            const int64_t i = (it0 + u) * stride + block * kRedThreads + threadIdx.x;
            v[u] = i < n ? __ldg(x + i) : T(0);
        }
#pragma unroll
        for (int u = 0; u < kHistUnroll; ++u) {
            const int64_t i = (it0 + u) * stride + block * kRedThreads + threadIdx.x;
            const bool live = i < n;
            const long long b = live ? bin_of<T>(s, (double)v[u]) : -1;
            const unsigned peers = __match_any_sync(0xffffffffu, b);
            const int leader = __ffs(peers) - 1;
            if (live && lane == leader)
                atomicAdd(reinterpret_cast<unsigned long long *>(counts) + b, (unsigned long long)__popc(peers));
        }
    }
}

// bins in shared memory when the device-side bin count fits kSmemBins, else the
// whole grid takes the global-atomic path (the decision needs nb, known only on
// the device after k_hist_params)
constexpr int kSmemBins = 16 * 1024;

template <typename T>
__global__ void __launch_bounds__(kRedThreads) k_hist_count_smem(const T *x, int64_t n, const HistState *st,
                                                                 const int32_t *status, long long *counts) {
    if (*status != EDGC_OK) return;
    extern __shared__ unsigned int sh[];
    const HistState s = *st;
    if (s.nb > kSmemBins) {
        k_hist_count_global_body<T>(x, n, s, counts, (int64_t)blockIdx.x, (int64_t)gridDim.x);
        return;
    }
    for (long long i = threadIdx.x; i < s.nb; i += kRedThreads) sh[i] = 0u;
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * kRedThreads;
    const int64_t n_iter = (n + stride - 1) / stride;
    for (int64_t it0 = 0; it0 < n_iter; it0 += kHistUnroll) {
        T v[kHistUnroll];
#pragma unroll
        for (int u = 0; u < kHistUnroll; ++u) {
            const int64_t i = (it0 + u) * stride + (int64_t)blockIdx.x * kRedThreads + threadIdx.x;
            v[u] = i < n ? __ldg(x + i) : T(0);
        }
#pragma unroll
        for (int u = 0; u < kHistUnroll; ++u) {
            const int64_t i = (it0 + u) * stride + (int64_t)blockIdx.x * kRedThreads + threadIdx.x;
            const bool live = i < n;
            // FD bins are narrow (~1% of sigma): a warp's values rarely share a
            // bin, so direct shared atomics beat a match.any aggregation here
            if (live) atomicAdd(&sh[(int)bin_of<T>(s, (double)v[u])], 1u);
        }
    }
    __syncthreads();
    for (long long i = threadIdx.x; i < s.nb; i += kRedThreads) {
        const unsigned v = sh[i];
        if (v) atomicAdd(reinterpret_cast<unsigned long long *>(counts) + i, (unsigned long long)v);
    }
}

template <typename T>
__global__ void __launch_bounds__(kRedThreads) k_hist_count_global(const T *x, int64_t n, const HistState *st,
                                                                   const int32_t *status, long long *counts) {
    if (*status != EDGC_OK) return;
    k_hist_count_global_body<T>(x, n, *st, counts, (int64_t)blockIdx.x, (int64_t)gridDim.x);
}

__global__ void __launch_bounds__(kRedThreads) k_hist_entropy_partial(const HistState *st, const int32_t *status,
                                                                      const long long *counts, int64_t total,
                                                                      double *partial) {
    double acc = 0.0;
    if (*status == EDGC_OK) {
        const HistState s = *st;
        const double tot = (double)total;
        for (long long k = (long long)blockIdx.x * kRedThreads + threadIdx.x; k < s.nb;
             k += (long long)gridDim.x * kRedThreads) {
            const long long c = counts[k];
            if (c > 0) {
                const double p = __ddiv_rn((double)c, tot);
                const double w = __dsub_rn(edge_at(s, k + 1), edge_at(s, k));
                acc += p * log(__ddiv_rn(p, w));
            }
        }
    }
    acc = warp_sum(acc);
    __shared__ double s_red[kRedThreads / 32];
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int w = 0; w < kRedThreads / 32; ++w) a += s_red[w];
        partial[blockIdx.x] = a;
    }
}

__global__ void k_hist_entropy_final(const double *partial, int nblk, const int32_t *status, double *result) {
    if (*status != EDGC_OK) return;
    double a = 0.0;
    for (int b = 0; b < nblk; ++b) a += partial[b];
    result[0] = -a;
}

constexpr int kMinMaxBlocks = 592;
constexpr int kEntBlocks = 148;

struct HistLayout {
    HistState *st;
    double2 *mm;
    unsigned int *ghist;
    double *ent;
    int64_t bytes;
};

HistLayout hist_layout(void *ws) {
    Arena a(ws, INT64_MAX);
    HistLayout L;
    L.st = a.take<HistState>(1);
    L.mm = a.take<double2>(kMinMaxBlocks);
    L.ghist = a.take<unsigned int>(4 * kDigits);
    L.ent = a.take<double>(kEntBlocks);
    L.bytes = a.off;
    return L;
}

template <typename T>
int run_histogram(const T *x, int64_t n, double inv_cbrt_n, int64_t fixed_bins, int64_t cap, long long *counts,
                  double *edges, double *result, int32_t *status, void *ws, cudaStream_t st) {
    HistLayout L = hist_layout(ws);
    const int sms = sm_count();
    const int mmb = (int)std::max<int64_t>(1, std::min<int64_t>(kMinMaxBlocks, ceil_div(n, kRedThreads)));
    if (fixed_bins > 0) {  // no select passes: a separate min/max pass
        k_minmax<T><<<mmb, kRedThreads, 0, st>>>(x, n, L.mm);
        EDGC_LAUNCH_CHECK();
    }
    k_hist_init<<<1, 32, 0, st>>>(L.st, fixed_bins > 0 ? L.mm : nullptr, mmb, n, fixed_bins > 0, status, result);
    EDGC_LAUNCH_CHECK();
    EDGC_CUDA_TRY(cudaMemsetAsync(L.ghist, 0, 4 * kDigits * sizeof(unsigned int), st));
    const int kbits = KeyOf<T>::kBits;
    const int hb = (int)std::max<int64_t>(
        1, std::min<int64_t>(std::min<int64_t>((int64_t)sms * 4, kMinMaxBlocks), ceil_div(n, kRedThreads)));
    if (fixed_bins <= 0) {
        // kDigitBits-wide digits, most significant first; the last one takes the rest
        for (int hi = kbits; hi > 0; hi -= kDigitBits) {
            const int width = std::min(kDigitBits, hi), shift = hi - width;
            const bool first = hi == kbits;
            if (first)
                k_radix_hist<T, true><<<hb, kRedThreads, 0, st>>>(x, n, L.st, shift, width, L.ghist, L.mm);
            else
                k_radix_hist<T, false><<<hb, kRedThreads, 0, st>>>(x, n, L.st, shift, width, L.ghist, nullptr);
            EDGC_LAUNCH_CHECK();
            k_radix_pick<<<1, 256, 0, st>>>(L.st, L.ghist, shift, first ? L.mm : nullptr, hb, status);
            EDGC_LAUNCH_CHECK();
        }
    }
    k_hist_params<T><<<1, 1, 0, st>>>(L.st, n, inv_cbrt_n, fixed_bins, cap, status, result);
    EDGC_LAUNCH_CHECK();
    k_hist_edges<<<sms, 256, 0, st>>>(L.st, status, edges, status);
    EDGC_LAUNCH_CHECK();
    EDGC_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(long long) * cap, st));
    // counts go to shared memory when the device-side bin count fits kSmemBins
    // (the kernel decides), else global atomics
    const int cb = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * 3, ceil_div(n, kRedThreads)));
    if (cap <= kSmemBins || fixed_bins <= 0) {
        const size_t smem = sizeof(unsigned int) * (size_t)std::min<int64_t>(std::max<int64_t>(cap, 1), kSmemBins);
        EDGC_CUDA_TRY(cudaFuncSetAttribute(k_hist_count_smem<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(kSmemBins * sizeof(unsigned int))));
        k_hist_count_smem<T><<<cb, kRedThreads, smem, st>>>(x, n, L.st, status, counts);
    } else {
        k_hist_count_global<T><<<cb * 4, kRedThreads, 0, st>>>(x, n, L.st, status, counts);
    }
    EDGC_LAUNCH_CHECK();
    k_hist_entropy_partial<<<kEntBlocks, kRedThreads, 0, st>>>(L.st, status, counts, n, L.ent);
    EDGC_LAUNCH_CHECK();
    k_hist_entropy_final<<<1, 1, 0, st>>>(L.ent, kEntBlocks, status, result);
    EDGC_LAUNCH_CHECK();
    return EDGC_OK;
}

}  // namespace
}  // namespace edgc

using namespace edgc;

extern "C" int64_t edgc_entropy_gaussian_workspace_bytes(const edgc_gauss_desc *descs, int n) {
    (void)descs;
    return align256(sizeof(GaussDev) * (int64_t)std::max(n, 1)) +
           align256(sizeof(double2) * (int64_t)std::max(n, 1) * kGaussBlocksPerDesc * (kRedThreads / 32));
}

extern "C" int edgc_entropy_gaussian(int src_dtype, const edgc_gauss_desc *descs, int n, double *h_out,
                                     int32_t *status_dev, void *ws, int64_t ws_bytes, void *stream) {
    if (n == 0) return EDGC_OK;
    EDGC_REQUIRE(n > 0 && descs && h_out && status_dev && (src_dtype == 0 || src_dtype == 1),
                 "edgc_entropy_gaussian: bad arguments");
    EDGC_REQUIRE(ws_bytes >= edgc_entropy_gaussian_workspace_bytes(descs, n), "edgc_entropy_gaussian: workspace");
    Arena a(ws, ws_bytes);
    GaussDev *d = a.take<GaussDev>(n);
    double2 *part = a.take<double2>((int64_t)n * kGaussBlocksPerDesc * (kRedThreads / 32));
    std::vector<GaussDev> h(n);
    for (int i = 0; i < n; ++i) {
        EDGC_REQUIRE(!descs[i].bitmap || descs[i].idx, "gauss desc %d: a bitmap needs idx (for the shift)", i);
        h[i] = GaussDev{descs[i].src, descs[i].idx, descs[i].count, descs[i].bitmap, descs[i].n_elems};
    }
    cudaStream_t st = (cudaStream_t)stream;
    EDGC_CUDA_TRY(cudaMemcpyAsync(d, h.data(), sizeof(GaussDev) * n, cudaMemcpyHostToDevice, st));
    if (src_dtype == 0)
        k_gauss_partial<float><<<kGaussBlocksPerDesc, kRedThreads, 0, st>>>(d, n, part);
    else
        k_gauss_partial<double><<<kGaussBlocksPerDesc, kRedThreads, 0, st>>>(d, n, part);
    EDGC_LAUNCH_CHECK();
    k_gauss_finish<<<(n + 3) / 4, 128, 0, st>>>(d, n, part, kGaussBlocksPerDesc * (kRedThreads / 32), h_out,
                                                 status_dev);
    EDGC_LAUNCH_CHECK();
    return EDGC_OK;
}

extern "C" int64_t edgc_entropy_histogram_workspace_bytes(int64_t count) {
    (void)count;
    return hist_layout(nullptr).bytes;
}

extern "C" int edgc_entropy_histogram(int dtype, const void *samples, int64_t count, double inv_cbrt_n,
                                      int64_t fixed_bins, int64_t bins_cap, int64_t *counts_dev, double *edges_dev,
                                      double *result_dev, int32_t *status_dev, void *ws, int64_t ws_bytes,
                                      void *stream) {
    EDGC_REQUIRE((dtype == 0 || dtype == 1) && samples && count >= 1 && bins_cap >= 1 && counts_dev &&
                     result_dev && status_dev,
                 "edgc_entropy_histogram: bad arguments");
    EDGC_REQUIRE(ws_bytes >= edgc_entropy_histogram_workspace_bytes(count), "edgc_entropy_histogram: workspace");
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == 0)
        return run_histogram<float>((const float *)samples, count, inv_cbrt_n, fixed_bins, bins_cap,
                                    (long long *)counts_dev, edges_dev, result_dev, status_dev, ws, st);
    return run_histogram<double>((const double *)samples, count, inv_cbrt_n, fixed_bins, bins_cap,
                                 (long long *)counts_dev, edges_dev, result_dev, status_dev, ws, st);
}

extern "C" int edgc_entropy_gaussian_partials(const double *partials_dev, int64_t slots, const int64_t *counts_dev,
                                              int n, double *h_out, int32_t *status_dev, void *stream) {
    EDGC_REQUIRE(n >= 0 && slots >= 1 && (n == 0 || (partials_dev && counts_dev && h_out && status_dev)),
                 "edgc_entropy_gaussian_partials: bad arguments");
    if (n == 0) return EDGC_OK;
    k_gauss_finish_slots<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(partials_dev, slots, counts_dev, n, h_out,
                                                                           status_dev);
    EDGC_LAUNCH_CHECK();
    return EDGC_OK;
}
