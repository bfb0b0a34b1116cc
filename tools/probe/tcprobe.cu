// Standalone check of the tcgen05 3xTF32 GEMM core (paper_2511_10333_b200/csrc/tc_gemm.cuh):
// C = A B^T-style products with K-major / MN-major operands against an fp64 host
// reference, then timing at wide-path shapes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o tools/probe/tcprobe tools/probe/tcprobe.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "../../paper_2511_10333_b200/csrc/tc_gemm.cuh"

using namespace edgc;

// C[i][j] = sum_k A(i,k) B(j,k); A K-major: A[i*lda + k]; MN-major: A[k*lda + i] (same for B)
template <bool AMN, bool BMN, int BN>
struct PlainOp {
    static constexpr bool kAMN = AMN, kBMN = BMN;
    static constexpr int kPF = 0;
    struct Tile {
        int64_t i0, j0;
    };
    int ntiles, tiles_n;
    int64_t M, N, K, lda, ldb, ldc;
    const float *A, *B;
    float *C;
    __device__ Tile tile(int idx) const { return Tile{(int64_t)(idx / tiles_n) * tc::kBM, (int64_t)(idx % tiles_n) * BN}; }
    __device__ int64_t tile_k(const Tile &) const { return K; }
    __device__ void views(const Tile &t, tc::View &a, tc::View &b) const {
        a = AMN ? tc::View{A + t.i0, lda, M - t.i0, K, 0, 0} : tc::View{A + t.i0 * lda, lda, M - t.i0, K, 0, 0};
        b = BMN ? tc::View{B + t.j0, ldb, N - t.j0, K, 0, 0} : tc::View{B + t.j0 * ldb, ldb, N - t.j0, K, 0, 0};
    }
    __device__ void prefetch(const Tile &, int, int, uint8_t *) const {}
    __device__ void epilogue(const Tile &t, int row0, int col, const float4 (&v)[8], const uint8_t *) const {
        const int64_t j = t.j0 + col;
        for (int u = 0; u < 8; ++u) {
            const int64_t i = t.i0 + row0 + 4 * u;
            if (i >= M) break;
            const float a[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
            if (N % 4 == 0 && j + 4 <= N) {
                __stcs(reinterpret_cast<float4 *>(C + i * ldc + j), v[u]);
            } else {
                for (int c = 0; c < 4; ++c)
                    if (j + c < N) C[i * ldc + j + c] = a[c];
            }
        }
    }
};

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

template <bool AMN, bool BMN, int BN, int KCH = 4>
double run(int64_t M, int64_t N, int64_t K, bool check, int iters) {
    const int64_t lda = AMN ? M : K, ldb = BMN ? N : K;
    const int64_t asz = AMN ? K * M : M * K, bsz = BMN ? K * N : N * K;
    std::vector<float> A(asz), B(bsz);
    std::mt19937 rng(1234);
    std::normal_distribution<float> nd;
    for (auto &x : A) x = nd(rng);
    for (auto &x : B) x = nd(rng);
    if (getenv("TCPROBE_TF32IN")) {   // exact-TF32 inputs: isolates the accumulation error
        for (auto *v : {&A, &B})
            for (auto &x : *v) {
                uint32_t u;
                memcpy(&u, &x, 4);
                u &= 0xffffe000u;
                memcpy(&x, &u, 4);
            }
    }
    float *dA, *dB, *dC;
    CK(cudaMalloc(&dA, asz * 4));
    CK(cudaMalloc(&dB, bsz * 4));
    CK(cudaMalloc(&dC, M * N * 4));
    CK(cudaMemcpy(dA, A.data(), asz * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), bsz * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(dC, 0xff, M * N * 4));
    PlainOp<AMN, BMN, BN> op;
    op.tiles_n = (int)((N + BN - 1) / BN);
    op.ntiles = (int)((M + 127) / 128) * op.tiles_n;
    op.M = M; op.N = N; op.K = K; op.lda = lda; op.ldb = ldb; op.ldc = N;
    op.A = dA; op.B = dB; op.C = dC;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK((tc::launch<BN, KCH>(op, sms, 0)));
    CK(cudaDeviceSynchronize());
    double err = 0;
    if (check) {
        std::vector<float> C(M * N);
        CK(cudaMemcpy(C.data(), dC, M * N * 4, cudaMemcpyDeviceToHost));
        double num = 0, den = 0, mx = 0;
        for (int64_t i = 0; i < M; ++i)
            for (int64_t j = 0; j < N; ++j) {
                double s = 0;
                for (int64_t k = 0; k < K; ++k)
                    s += (double)(AMN ? A[k * lda + i] : A[i * lda + k]) * (double)(BMN ? B[k * ldb + j] : B[j * ldb + k]);
                const double d = C[i * N + j] - s;
                num += d * d;
                den += s * s;
                mx = std::max(mx, std::fabs(d));
            }
        err = std::sqrt(num / den);
        // systematic part: least-squares slope of C on the reference, and the residual around it
        double cr = 0;
        for (int64_t i = 0; i < M; ++i)
            for (int64_t j = 0; j < N; ++j) {
                double s = 0;
                for (int64_t k = 0; k < K; ++k)
                    s += (double)(AMN ? A[k * lda + i] : A[i * lda + k]) * (double)(BMN ? B[k * ldb + j] : B[j * ldb + k]);
                cr += (double)C[i * N + j] * s;
            }
        const double slope = cr / den;
        double res = 0;
        for (int64_t i = 0; i < M; ++i)
            for (int64_t j = 0; j < N; ++j) {
                double s = 0;
                for (int64_t k = 0; k < K; ++k)
                    s += (double)(AMN ? A[k * lda + i] : A[i * lda + k]) * (double)(BMN ? B[k * ldb + j] : B[j * ldb + k]);
                const double d = C[i * N + j] - slope * s;
                res += d * d;
            }
        printf("check KCH=%d AMN=%d BMN=%d BN=%d M=%lld N=%lld K=%lld: rel_fro=%.3e max_abs=%.3e slope-1=%.3e resid=%.3e %s\n",
               KCH, AMN, BMN, BN, (long long)M, (long long)N, (long long)K, err, mx, slope - 1, std::sqrt(res / den),
               err < 2e-6 ? "OK" : "FAIL");
    }
    if (iters > 0) {
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0));
        for (int it = 0; it < iters; ++it) CK((tc::launch<BN, KCH>(op, sms, 0)));
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        ms /= iters;
        const double fl = 2.0 * M * N * K;
        const double bytes = 4.0 * (asz + bsz + M * N);
        printf("time KCH=%d AMN=%d BMN=%d BN=%d M=%lld N=%lld K=%lld: %.3f ms  %.1f TF/s useful (x3 = %.1f TF/s tf32)  %.0f GB/s\n",
               KCH, AMN, BMN, BN, (long long)M, (long long)N, (long long)K, ms, fl / ms / 1e9, 3 * fl / ms / 1e9,
               bytes / ms / 1e6);
    }
    CK(cudaFree(dA));
    CK(cudaFree(dB));
    CK(cudaFree(dC));
    return err;
}

int main(int argc, char **argv) {
    const bool timing = argc < 2 || std::atoi(argv[1]) != 0;
    run<false, false, 128, 0>(300, 500, 100, true, 0);
    run<false, false, 128, 0>(256, 256, 2048, true, 0);
    run<false, false, 128, 4>(256, 256, 2048, true, 0);
    run<false, false, 128, 4>(256, 256, 4096, true, 0);
    run<false, false, 128, 0>(1000, 700, 256, true, 0);
    run<false, true, 128, 4>(1000, 200, 777, true, 0);
    run<false, true, 64, 4>(1000, 48, 600, true, 0);
    run<true, true, 128, 4>(700, 130, 1000, true, 0);
    run<true, true, 64, 2>(700, 100, 333, true, 0);
    run<true, false, 128, 0>(520, 96, 200, true, 0);
    if (timing) {
        run<false, false, 128, 0>(8192, 8192, 256, false, 20);
        run<false, false, 128, 0>(16384, 20480, 256, false, 5);
        run<false, true, 128, 4>(20480, 256, 5120, false, 10);
        run<true, true, 128, 4>(5120, 256, 20480, false, 10);
        run<false, true, 128, 4>(20480, 128, 5120, false, 10);
        run<false, true, 64, 4>(20480, 64, 5120, false, 10);
    }
    return 0;
}
