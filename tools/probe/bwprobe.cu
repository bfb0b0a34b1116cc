// HBM probe: achievable bandwidth of the pass-1 traffic pattern (read g, read w,
// write w) versus a plain copy, with simple vectorised grid-stride kernels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bwprobe bwprobe.cu && ./bwprobe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_copy(const float4 *__restrict__ a, float4 *__restrict__ o, long n4) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) o[i] = a[i];
}
__global__ void k_2r1w(const float4 *__restrict__ g, float4 *__restrict__ w, long n4) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
        float4 a = g[i], b = w[i];
        w[i] = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
    }
}
__global__ void k_2r1w_cs(const float4 *__restrict__ g, float4 *__restrict__ w, long n4) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
        float4 a = __ldcs(g + i), b = __ldcs(w + i);
        __stcs(w + i, make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w));
    }
}
__global__ void k_read2(const float4 *__restrict__ g, const float4 *__restrict__ w, float *sink, long n4) {
    float acc = 0.f;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
        float4 a = g[i], b = w[i];
        acc += a.x + b.y + a.z + b.w;
    }
    if (acc == 12345.f) *sink = acc;
}
__global__ void k_write(float4 *__restrict__ o, long n4) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x)
        o[i] = make_float4(1.f, 2.f, 3.f, 4.f);
}

int main() {
    const long n = 2300000000L, n4 = n / 4;
    float4 *g, *w, *o;
    float *sink;
    cudaMalloc(&g, n * 4); cudaMalloc(&w, n * 4); cudaMalloc(&o, n * 4); cudaMalloc(&sink, 4);
    cudaMemset(g, 0, n * 4); cudaMemset(w, 0, n * 4); cudaMemset(o, 0, n * 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int bpsm : {4, 8, 16}) {
        const int grid = sms * bpsm, th = 512;
        float ms;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a); k_copy<<<grid, th>>>(g, o, n4); cudaEventRecord(b); cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b); if (rep) printf("blocks/SM %2d copy      %.0f GB/s\n", bpsm, 8.0 * n / ms / 1e6);
            cudaEventRecord(a); k_2r1w<<<grid, th>>>(g, w, n4); cudaEventRecord(b); cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b); if (rep) printf("blocks/SM %2d 2r1w      %.0f GB/s\n", bpsm, 12.0 * n / ms / 1e6);
            cudaEventRecord(a); k_2r1w_cs<<<grid, th>>>(g, w, n4); cudaEventRecord(b); cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b); if (rep) printf("blocks/SM %2d 2r1w_cs   %.0f GB/s\n", bpsm, 12.0 * n / ms / 1e6);
            cudaEventRecord(a); k_read2<<<grid, th>>>(g, w, sink, n4); cudaEventRecord(b); cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b); if (rep) printf("blocks/SM %2d read2     %.0f GB/s\n", bpsm, 8.0 * n / ms / 1e6);
            cudaEventRecord(a); k_write<<<grid, th>>>(o, n4); cudaEventRecord(b); cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b); if (rep) printf("blocks/SM %2d write     %.0f GB/s\n", bpsm, 4.0 * n / ms / 1e6);
        }
    }
    return 0;
}
