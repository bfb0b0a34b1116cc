// Shared helpers for libedgc_b200.so (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/edgc_b200.h"

namespace edgc {

// Thread-local message for edgc_last_error().
void set_error(const char *fmt, ...);
// Process-wide count of kernels this library has launched (edgc_launch_count).
void count_launch();

#define EDGC_CUDA_TRY(expr)                                                          \
    do {                                                                              \
        cudaError_t _e = (expr);                                                      \
        if (_e != cudaSuccess) {                                                      \
            ::edgc::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,            \
                              cudaGetErrorString(_e));                                \
            return EDGC_ECUDA;                                                        \
        }                                                                             \
    } while (0)

#define EDGC_LAUNCH_CHECK()                                                          \
    do {                                                                              \
        ::edgc::count_launch();                                                       \
        cudaError_t _e = cudaGetLastError();                                          \
        if (_e != cudaSuccess) {                                                      \
            ::edgc::set_error("%s:%d launch: %s", __FILE__, __LINE__,               \
                              cudaGetErrorString(_e));                                \
            return EDGC_ECUDA;                                                        \
        }                                                                             \
    } while (0)

#define EDGC_REQUIRE(cond, ...)                                                      \
    do {                                                                              \
        if (!(cond)) {                                                                \
            ::edgc::set_error(__VA_ARGS__);                                           \
            return EDGC_EINVAL;                                                       \
        }                                                                             \
    } while (0)

// Bump allocator over a caller-provided workspace (256-byte aligned slices).
struct Arena {
    char *base;
    int64_t cap;
    int64_t off;
    __host__ Arena(void *p, int64_t c) : base((char *)p), cap(c), off(0) {}
    template <typename T>
    __host__ T *take(int64_t n) {
        off = (off + 255) & ~int64_t(255);
        T *p = (T *)(base ? base + off : nullptr);
        off += n * (int64_t)sizeof(T);
        return p;
    }
    __host__ bool ok() const { return off <= cap; }
};

static inline int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }
static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

int sm_count();

// ---- warp helpers ---------------------------------------------------------

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Sum V values held by every lane across the 32 lanes of a warp (V a power of
// two, V <= 32), in a butterfly that halves the live set each step: after the
// call lane l holds the full warp sum of value index (l / (32 / V)) in v[0]...
// Fixed association order => deterministic.
template <int V, typename T>
__device__ __forceinline__ T warp_reduce_scatter(T (&v)[V], int lane) {
    int cur = V;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        if (cur > 1) {
            const bool upper = (lane & o) != 0;
            const int half = cur >> 1;
#pragma unroll
            for (int i = 0; i < V / 2; ++i) {
                if (i < half) {
                    T send = upper ? v[i] : v[i + half];
                    T keep = upper ? v[i + half] : v[i];
                    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            cur = half;
        } else {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
        }
    }
    return v[0];
}

// For warp_reduce_scatter<V>: which value index lane `lane` ends up owning.
template <int V>
__device__ __forceinline__ int scatter_owner_index(int lane) {
    // Each halving step at offset o assigns the upper half to lanes with bit o
    // set; the first log2(V) offsets are 16, 8, ..., so the index bits are the
    // lane's high bits, most significant first.
    int idx = 0;
    int cur = V;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        if (cur > 1) {
            cur >>= 1;
            if (lane & o) idx += cur;
        }
    }
    return idx;
}

}  // namespace edgc
