// Throughput of the legacy warp-level tensor-core MMA (mma.sync m16n8k8 tf32) on sm_100a:
// each warp issues independent MMA chains from registers; reports TFLOP/s (2*16*8*8 per MMA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe/mmasync tools/probe/mmasync.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(float *out, int iters) {
    uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    float c[8][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile(
                "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0.f;
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float *out;
    cudaMalloc(&out, 148 * 8 * 1024 * 4);
    const int iters = 4096;
    for (int warps : {4, 8, 16, 32}) {
        const int blocks = 148 * 4, threads = warps * 32 / 4;
        k<<<blocks, threads>>>(out, 16);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        k<<<blocks, threads>>>(out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double flops = 2.0 * 16 * 8 * 8 * 8.0 * iters * (threads / 32) * (double)blocks;
        printf("warps/SM %d: %.1f TFLOP/s (tf32 mma.sync)\n", warps, flops / ms / 1e9);
    }
    return 0;
}
