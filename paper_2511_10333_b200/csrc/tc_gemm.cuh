// tcgen05 (5th-generation tensor core) GEMM core for the wide-rank path:
// D[128 x BN] = sum_k A[i, k] B[j, k] with fp32 operands split 3xTF32
// (a = a_hi + a_lo, both exact TF32; a.b ~= a_hi b_hi + a_hi b_lo + a_lo b_hi)
// and fp32 accumulation in tensor memory.
//
// Accuracy.  The products are exact to ~2^-22 relative, but the tensor core's
// fp32 accumulation truncates: measured on B200 the result shrinks by ~6e-9
// per accumulated K element (rel. error 1.4e-5 at K = 2048, tools/probe/tcprobe).
// Long contractions are therefore cut into chunks of KCH x 32 K elements, each
// accumulated fresh in TMEM and folded by the epilogue warps into a running
// fp32 sum (round-to-nearest adds) kept in a third TMEM buffer; the error is
// then that of one chunk (~1e-6 at 128).
//
// One persistent CTA per SM (352 threads, 11 warps):
//   warps 0-3   epilogue: tcgen05.ld of the finished chunk (row = TMEM lane),
//               fold into the running sum (tcgen05.st) or, after the last
//               chunk of a tile, transpose 32 x 32 slices through shared
//               memory and hand them to Op::epilogue as coalesced float4 rows
//   warps 4-9   producers, two groups of three warps taking alternate K blocks:
//               coalesced float4 global loads of the fp32 operand tiles (issued
//               before the stage wait), hi/lo split with integer rounding,
//               stores into the swizzled K-major or MN-major canonical UMMA
//               layouts, fence.proxy.async, mbarrier arrive
//   warp 10     TMEM allocation; one lane issues tcgen05.mma (kind::tf32,
//               M = 128, N = BN, K = 8; three per K step) and tcgen05.commit to
//               the stage-empty / chunk-full barriers
// Two chunk accumulators alternate, so the epilogue of one chunk (or tile)
// overlaps the MMAs of the next.  Operands come through registers rather than
// TMA: every operand is split into two planes anyway, and the wide-path
// operands come in both majorities and with rank-block strides.
//
// Op interface (by value, kernel parameter):
//   int ntiles;  struct Tile;  Tile tile(int idx) const;
//   static constexpr bool kAMN, kBMN;   // operand majority in global memory
//   int64_t tile_k(const Tile&) -> number of K elements (>= 1)
//   void views(const Tile&, View &a, View &b) const   // operand windows at the tile origin
//   void epilogue(const Tile&, int row0, int col, const float4 (&v)[8], const uint8_t *pf) const
//     v[u] = tile rows row0 + 4u, columns col .. col+3 (8 lanes cover 128
//     contiguous bytes of a row: the accumulator slice is transposed through
//     shared memory so global accesses coalesce); rows / columns outside the
//     problem are the Op's to skip
//   static constexpr int kPF;   // > 0: the epilogue reads kPF float4 of global input per
//     thread and slice; the Op's prefetch(t, row0, col, uint8_t *dst) issues them as
//     cp.async into per-thread slots (slot u at dst + u * 2048) one slice ahead (the
//     first slice of a tile before its accumulator is ready), and epilogue() gets
//     the slots in pf
#pragma once

#include <stdint.h>

#include "ptx.cuh"

namespace edgc {
namespace tc {

constexpr int kBM = 128;   // MMA M (TMEM lanes)
constexpr int kBK = 32;    // K elements per stage (one 128-byte swizzle row of fp32)
constexpr int kEpiWarps = 4, kProdWarps = 6;
constexpr int kMmaWarp = kEpiWarps + kProdWarps;
constexpr int kThreads = (kMmaWarp + 1) * 32;
constexpr int kGroupThreads = kProdWarps / 2 * 32;

// operand window: element (row, k) at p + row * ld + kmap(k) (K-major) or
// p + kmap(k) * ld + row (MN-major), kmap(k) = (k / kblk) * kstride + k % kblk
// (kblk = 0: kmap(k) = k; rank blocks of the averaged reconstruction otherwise)
struct View {
    const float *p;
    int64_t ld, rows, K, kblk, kstride;
};

// PFD: prefetch depth (slices of epilogue input in flight per warp); STAGES: operand stages
// (0: by tile width)
template <int BN, int KCH, int PF = 0, int PFD = 2, int STAGES = 0>
struct Cfg {
    static_assert(BN == 64 || BN == 128, "tile N");
    static_assert(PFD >= 2 && PFD <= 4, "prefetch depth");
    static constexpr int kAPlane = kBM * kBK * 4;          // bytes of one (hi or lo) plane
    static constexpr int kBPlane = BN * kBK * 4;
    static constexpr int kStageBytes = 2 * (kAPlane + kBPlane);
    static constexpr int kStages = STAGES > 0 ? STAGES : BN == 128 ? (PF > 0 ? 2 : 3) : 4;
    static constexpr int kPFBytes = PFD * PF * kEpiWarps * 32 * 16;   // PFD prefetch slot buffers
    static constexpr int kBarBytes = 8 * (2 * kStages + 4) + 16;
    static constexpr int kEpiBytes = kEpiWarps * 32 * 32 * 4;   // per-warp 32 x 32 transpose slices
    static constexpr int kSmem = kStages * kStageBytes + kEpiBytes + kPFBytes + kBarBytes + 1024;
    // two chunk accumulators (+ the running sum when chunked), power of two >= 32
    static constexpr uint32_t kCols = (KCH > 0 ? 3 : 2) * BN;
    static constexpr uint32_t kTmemCols = kCols <= 32 ? 32 : kCols <= 64 ? 64 : kCols <= 128 ? 128 : kCols <= 256 ? 256 : 512;
};

// ------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ void tmem_alloc(uint32_t *dst, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_addr(dst)),
                 "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols) : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     ptx::smem_addr(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float *v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float *v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16};" ::"r"(taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
        "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
        "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
        "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
        "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
        : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ptx::smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// hi = x with the 13 low mantissa bits cleared (exact TF32), lo = x - hi (exact in
// fp32, |lo| < 2^-10 |x|) rounded to the nearest TF32 with integer ops (the tensor
// core would truncate it): ~2^-22 relative error per product
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
__device__ __forceinline__ float tf32_rn(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// ---------------------------------------------------------------- layouts
// 128B-swizzled canonical layouts (Swizzle<3,4,3>: byte bits [4,7) ^= bits [7,10)),
// 1024-byte aligned planes.
// K-major plane of ROWS x 32 fp32: row r at r*128 bytes, 16-byte chunk q at (q ^ r%8).
__device__ __forceinline__ uint32_t off_kmajor(int row, int kq) {
    return (uint32_t)(row * 128 + (((kq) ^ (row & 7)) << 4));
}
// MN-major plane of 32 (K) x ROWS: tf32 MN-major operands only take the
// 128B_BASE32B swizzle (Swizzle<2,5,2>: byte bits [5,7) ^= bits [7,9)), atoms of
// 4 K rows x 128 bytes (32 MN elements); 4-row K groups of ROWS/32 atoms.
template <int ROWS>
__device__ __forceinline__ uint32_t off_mnmajor(int k, int mq) {
    return (uint32_t)((k >> 2) * (ROWS * 16) + (mq >> 3) * 512 + (k & 3) * 128 +
                      ((((mq & 7) >> 1) ^ (k & 3)) << 5) + ((mq & 1) << 4));
}

// shared-memory matrix descriptor (sm_100 UMMA): start >> 4 [0,14), LBO >> 4 [16,30),
// SBO >> 4 [32,46), version 1 [46,48), layout [61,64) (SWIZZLE_128B = 2, 128B_BASE32B = 1)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}
// K-major: SBO = 1024 (8-row groups), LBO unused (16); K step of 8 = +32 bytes
// MN-major: LBO = 512 (32-element MN atoms), SBO = 4-row K-group stride; K step of 8 = two K groups
template <bool MN, int ROWS>
__device__ __forceinline__ uint64_t operand_desc(uint32_t plane, int kk) {
    if (MN) return sdesc(plane + kk * (ROWS * 32), 512, ROWS * 16, 1);
    return sdesc(plane + kk * 32, 16, 1024, 2);
}

// instruction descriptor: D f32 [4,6) = 1, A/B tf32 [7,10)/[10,13) = 2, majors [15]/[16],
// N >> 3 [17,23), M >> 4 [24,29)
template <bool AMN, bool BMN, int BN>
__host__ __device__ constexpr uint32_t instr_desc() {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((AMN ? 1u : 0u) << 15) | ((BMN ? 1u : 0u) << 16) |
           ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
}

// ---------------------------------------------------------------- producer
// A group's 96 threads cover a plane of ROWS x 32 as float4 slots f = tid + 96 u:
// K-major  row = f / 8, k = 4 (f % 8)               -> row0 + 12 u, fixed k
// MN-major row = 4 (f % (ROWS/4)), k = f / (ROWS/4) -> fixed row, k0 + (96 / (ROWS/4)) u
template <bool MN, int ROWS>
struct Plane {
    static constexpr int kVec = ROWS * kBK / 4;   // float4 per plane
    static constexpr int kPer = (kVec + kGroupThreads - 1) / kGroupThreads;
    static constexpr int kStep = MN ? kGroupThreads / (ROWS / 4) : kGroupThreads / 8;
    static_assert(kGroupThreads % (MN ? ROWS / 4 : 8) == 0, "slot pattern");
    __device__ static __forceinline__ int row0(int tid) { return MN ? (tid % (ROWS / 4)) * 4 : tid / 8; }
    __device__ static __forceinline__ int k0(int tid) { return MN ? tid / (ROWS / 4) : (tid % 8) * 4; }
    __device__ static __forceinline__ uint32_t offset(int f) {
        return MN ? off_mnmajor<ROWS>(f / (ROWS / 4), f % (ROWS / 4)) : off_kmajor(f / 8, f % 8);
    }
};

__device__ __forceinline__ int64_t kmap(const View &v, int64_t k) {
    return v.kblk ? (k / v.kblk) * v.kstride + k % v.kblk : k;
}

// general path: bounds per element, zero fill
template <bool MN>
__device__ __forceinline__ float4 load_checked(const View &v, int row, int64_t k) {
    float e[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int r = MN ? row + j : row;
        const int64_t kk = MN ? k : k + j;
        e[j] = (r < v.rows && kk < v.K) ? __ldg(MN ? v.p + kmap(v, kk) * v.ld + r : v.p + (int64_t)r * v.ld + kmap(v, kk))
                                        : 0.f;
    }
    return make_float4(e[0], e[1], e[2], e[3]);
}

template <bool MN, int ROWS>
__device__ __forceinline__ void load_plane(const View &v, bool vec, int64_t kbase, int tid,
                                           float4 (&x)[Plane<MN, ROWS>::kPer]) {
    using PL = Plane<MN, ROWS>;
    const int r0 = PL::row0(tid), k0 = PL::k0(tid);
    const bool fast = vec && v.rows >= ROWS && kbase + kBK <= v.K && (v.kblk == 0 || v.kblk % kBK == 0);
    if (fast) {
        const int64_t koff = kmap(v, kbase);
        const float *p = MN ? v.p + (koff + k0) * v.ld + r0 : v.p + (int64_t)r0 * v.ld + koff + k0;
        // kStep rows (K-major) or K lines (MN-major), < 2^31 elements per plane.  Opaque per
        // K block: otherwise the compiler hoists the kPer 64-bit row addresses out of the K
        // loop and spills them (measured: LDL on the producer's critical path)
        uint32_t step = (uint32_t)(PL::kStep * v.ld);
        asm volatile("" : "+r"(step));
#pragma unroll
        for (int u = 0; u < PL::kPer; ++u) {
            if (PL::kVec % kGroupThreads != 0 && tid + u * kGroupThreads >= PL::kVec) break;
            x[u] = __ldg(reinterpret_cast<const float4 *>(p + (uint32_t)u * step));
        }
    } else if (!MN && vec && v.rows >= ROWS && v.kblk % 4 == 0) {
        // K-major operand whose K is the concatenation of narrow rank blocks (the averaged
        // reconstruction at W ranks of rank r, 4 | r): the thread's 4 consecutive k lie in one
        // rank block, so every row is one float4 at kmap(k0); k past K (K < a 32-wide block) is 0
        const int64_t k = kbase + k0;
        const bool in = k < v.K;
        const float *p = v.p + (int64_t)r0 * v.ld + (in ? kmap(v, k) : 0);
        uint32_t step = (uint32_t)(PL::kStep * v.ld);
        asm volatile("" : "+r"(step));
#pragma unroll
        for (int u = 0; u < PL::kPer; ++u) {
            if (PL::kVec % kGroupThreads != 0 && tid + u * kGroupThreads >= PL::kVec) break;
            x[u] = in ? __ldg(reinterpret_cast<const float4 *>(p + (uint32_t)u * step)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    } else {
#pragma unroll
        for (int u = 0; u < PL::kPer; ++u) {
            if (PL::kVec % kGroupThreads != 0 && tid + u * kGroupThreads >= PL::kVec) break;
            const int row = MN ? r0 : r0 + u * PL::kStep;
            const int64_t k = kbase + (MN ? k0 + u * PL::kStep : k0);
            x[u] = load_checked<MN>(v, row, k);
        }
    }
}

template <bool MN, int ROWS>
__device__ __forceinline__ void store_plane(uint8_t *hi, uint8_t *lo, int tid,
                                            const float4 (&x)[Plane<MN, ROWS>::kPer]) {
    using PL = Plane<MN, ROWS>;
#pragma unroll
    for (int u = 0; u < PL::kPer; ++u) {
        const int f = tid + u * kGroupThreads;
        if (PL::kVec % kGroupThreads != 0 && f >= PL::kVec) break;
        const uint32_t o = PL::offset(f);
        const float h0 = tf32_hi(x[u].x), h1 = tf32_hi(x[u].y), h2 = tf32_hi(x[u].z), h3 = tf32_hi(x[u].w);
        ptx::st_shared_v4(hi + o, h0, h1, h2, h3);
        ptx::st_shared_v4(lo + o, tf32_rn(x[u].x - h0), tf32_rn(x[u].y - h1), tf32_rn(x[u].z - h2),
                          tf32_rn(x[u].w - h3));
    }
}

// float4 loads need 16-byte aligned rows (K-major) / K lines (MN-major)
__device__ __forceinline__ bool view_vec(const View &v) {
    return ((uintptr_t)v.p % 16 == 0) && (v.ld % 4 == 0) && (v.kblk == 0 || (v.kblk % 4 == 0 && v.kstride % 4 == 0));
}

// ------------------------------------------------------------------ kernel
// KCH = K blocks (of 32) per accumulation chunk; 0 = the whole tile in one chunk
template <int BN, int KCH, class Op>
__global__ void __launch_bounds__(kThreads, 1) k_tc(const Op op) {
    constexpr int PF = Op::kPF, PFD = Op::kPFDepth;
    using C = Cfg<BN, KCH, PF, PFD, Op::kStages>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *epi_smem = smem + C::kStages * C::kStageBytes;
    uint8_t *pf_smem = epi_smem + C::kEpiBytes;
    uint64_t *full = (uint64_t *)(pf_smem + C::kPFBytes);
    uint64_t *empty = full + C::kStages;
    uint64_t *tfull = empty + C::kStages;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = (uint32_t *)(tempty + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            ptx::mbar_init(full + s, kProdWarps / 2);
            ptx::mbar_init(empty + s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(tfull + b, 1);
            ptx::mbar_init(tempty + b, kEpiWarps);
        }
        ptx::fence_mbar_init();
    }
    if (warp == kMmaWarp) tmem_alloc(tmem_slot, C::kTmemCols);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp >= kEpiWarps && warp < kMmaWarp) {
        // ------------------------------------------------ producers
        const int grp = (warp - kEpiWarps) / (kProdWarps / 2);
        const int tid = threadIdx.x - kEpiWarps * 32 - grp * kGroupThreads;
        int64_t q = 0;   // CTA-local K-block counter across tiles
        for (int ti = blockIdx.x; ti < op.ntiles; ti += gridDim.x) {
            const typename Op::Tile t = op.tile(ti);
            const int nkb = (int)((op.tile_k(t) + kBK - 1) / kBK);
            View av, bv;
            op.views(t, av, bv);
            const bool avec = view_vec(av), bvec = view_vec(bv);
            for (int kb = 0; kb < nkb; ++kb, ++q) {
                // two groups take alternate K blocks; with one operand stage a single group
                // (two would share the stage's barrier phases and one could run two phases ahead)
                if (C::kStages == 1 ? grp != 0 : (q & 1) != grp) continue;
                const int s = (int)(q % C::kStages);
                const uint32_t use = (uint32_t)(q / C::kStages);
                float4 va[Plane<Op::kAMN, kBM>::kPer], vb[Plane<Op::kBMN, BN>::kPer];
                // tid is made opaque per K block so the per-slot global / shared offsets are
                // recomputed (cheap integer ops) instead of hoisted out of the loop and spilled
                int otid = tid;
                asm volatile("" : "+r"(otid));
                load_plane<Op::kAMN, kBM>(av, avec, (int64_t)kb * kBK, otid, va);
                load_plane<Op::kBMN, BN>(bv, bvec, (int64_t)kb * kBK, otid, vb);
                ptx::mbar_wait(empty + s, (use & 1) ^ 1);
                uint8_t *st = smem + s * C::kStageBytes;
                asm volatile("" : "+r"(otid));
                store_plane<Op::kAMN, kBM>(st, st + C::kAPlane, otid, va);
                store_plane<Op::kBMN, BN>(st + 2 * C::kAPlane, st + 2 * C::kAPlane + C::kBPlane, otid, vb);
                fence_async_smem();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(full + s);
            }
        }
    } else if (warp == kMmaWarp) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc = instr_desc<Op::kAMN, Op::kBMN, BN>();
            const uint32_t sbase = ptx::smem_addr(smem);
            int64_t q = 0, cc = 0;   // K blocks, chunks
            for (int ti = blockIdx.x; ti < op.ntiles; ti += gridDim.x) {
                const typename Op::Tile t = op.tile(ti);
                const int nkb = (int)((op.tile_k(t) + kBK - 1) / kBK);
                const int kch = KCH > 0 ? KCH : nkb;
                for (int c0 = 0; c0 < nkb; c0 += kch, ++cc) {
                    const int b = (int)(cc & 1);
                    ptx::mbar_wait(tempty + b, (uint32_t)((cc >> 1) & 1) ^ 1);
                    fence_after();
                    const uint32_t d = tmem + b * BN;
                    const int c1 = c0 + kch < nkb ? c0 + kch : nkb;
                    for (int kb = c0; kb < c1; ++kb, ++q) {
                        const int s = (int)(q % C::kStages);
                        ptx::mbar_wait(full + s, (uint32_t)(q / C::kStages) & 1);
                        fence_after();
                        const uint32_t ahi = sbase + s * C::kStageBytes, alo = ahi + C::kAPlane;
                        const uint32_t bhi = ahi + 2 * C::kAPlane, blo = bhi + C::kBPlane;
#pragma unroll
                        for (int kk = 0; kk < kBK / 8; ++kk) {
                            const uint64_t a_h = operand_desc<Op::kAMN, kBM>(ahi, kk);
                            const uint64_t a_l = operand_desc<Op::kAMN, kBM>(alo, kk);
                            const uint64_t b_h = operand_desc<Op::kBMN, BN>(bhi, kk);
                            const uint64_t b_l = operand_desc<Op::kBMN, BN>(blo, kk);
                            mma_tf32(d, a_h, b_h, idesc, (kb > c0 || kk > 0) ? 1u : 0u);
#ifndef TC_HIHI_ONLY
                            mma_tf32(d, a_h, b_l, idesc, 1);
                            mma_tf32(d, a_l, b_h, idesc, 1);
#endif
                        }
                        mma_commit(empty + s);
                    }
                    mma_commit(tfull + b);
                }
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------ epilogue
        int64_t cc = 0;
        uint8_t *xs = epi_smem + warp * 4096;   // this warp's 32 x 32 fp32 slice, 16-byte chunks swizzled
        const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
        const uint32_t run = tmem + lane_off + 2 * BN;   // running sum (chunked)
        uint8_t *pf = pf_smem + threadIdx.x * 16;         // this thread's prefetch slots
        constexpr int kPFBuf = PF * kEpiWarps * 32 * 16;
        const int row0 = warp * 32 + lane / 8, lcol = (lane & 7) * 4;
        for (int ti = blockIdx.x; ti < op.ntiles; ti += gridDim.x) {
            const typename Op::Tile t = op.tile(ti);
            const int nkb = (int)((op.tile_k(t) + kBK - 1) / kBK);
            const int kch = KCH > 0 ? KCH : nkb;
            for (int c0 = 0; c0 < nkb; c0 += kch, ++cc) {
                const int b = (int)(cc & 1);
                const bool first = c0 == 0, last = c0 + kch >= nkb;
                if (PF > 0 && last) {
                    // the first PFD - 1 slices of the tile (one group each, empty past the tile)
#pragma unroll
                    for (int s = 0; s < PFD - 1; ++s) {
                        if (s * 32 < BN) op.prefetch(t, row0, s * 32 + lcol, pf + s * kPFBuf);
                        cp_async_commit();
                    }
                }
                ptx::mbar_wait(tfull + b, (uint32_t)(cc >> 1) & 1);
                fence_after();
                const uint32_t acc = tmem + lane_off + b * BN;
#pragma unroll 1
                for (int col = 0; col < BN; col += 32) {
                    if (PF > 0 && last) {
                        // slice + PFD - 1 into the buffer the previous slice released (a group per
                        // slice even past the tile, so the wait below is always PFD - 1 deep)
                        const int ahead = (col >> 5) + PFD - 1;
                        if (ahead * 32 < BN) op.prefetch(t, row0, ahead * 32 + lcol, pf + (ahead % PFD) * kPFBuf);
                        cp_async_commit();
                    }
                    float v[32];
                    tmem_ld16(acc + col, v);
                    tmem_ld16(acc + col + 16, v + 16);
                    if (KCH > 0 && !first) {
                        float r[32];
                        tmem_ld16(run + col, r);
                        tmem_ld16(run + col + 16, r + 16);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] += r[i];
                    } else {
                        tmem_ld_wait();
                    }
                    if (last) {
                        // row = lane -> 8 lanes per row, float4 columns
#pragma unroll
                        for (int c4 = 0; c4 < 8; ++c4)
                            ptx::st_shared_v4(xs + lane * 128 + ((c4 ^ (lane & 7)) << 4), v[4 * c4], v[4 * c4 + 1],
                                              v[4 * c4 + 2], v[4 * c4 + 3]);
                        __syncwarp();
                        float4 x[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int r = 4 * u + lane / 8;
                            x[u] = ptx::ld_shared_v4(xs + r * 128 + (((lane & 7) ^ (r & 7)) << 4));
                        }
                        __syncwarp();
                        if (PF > 0) cp_async_wait<PFD - 1>();
                        op.epilogue(t, row0, col + lcol, x, pf + ((col >> 5) % PFD) * kPFBuf);
                    } else {
                        tmem_st16(run + col, v);
                        tmem_st16(run + col + 16, v + 16);
                    }
                }
                if (!last) tmem_st_wait();
                fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(tempty + b);
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        fence_after();
        tmem_dealloc(tmem, C::kTmemCols);
    }
}

// launch helper: persistent grid of min(tiles, SMs) CTAs (measured: a 4-wave grid, meant to let
// free SMs absorb the CTAs of SMs the side-stream plans hold, is 3-10% slower alone and did not
// remove the plan interference at GPT2-12.1B r = 256)
template <int BN, int KCH, class Op>
inline cudaError_t launch(const Op &op, int sms, cudaStream_t st) {
    using C = Cfg<BN, KCH, Op::kPF, Op::kPFDepth, Op::kStages>;
    if (op.ntiles <= 0) return cudaSuccess;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_tc<BN, KCH, Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int grid = op.ntiles < sms ? op.ntiles : sms;
    k_tc<BN, KCH, Op><<<grid, kThreads, C::kSmem, st>>>(op);
    return cudaGetLastError();
}

}  // namespace tc
}  // namespace edgc
