// Standalone probe of the tcgen05 kind::tf32 path used by the tensor-core M2L:
// one 128 x 96 x 128 tile, operands in the canonical K-major no-swizzle layout,
// 3xTF32 split (A_hi B_hi + A_hi B_lo + A_lo B_hi) vs 1xTF32, checked against
// an FP64 host product.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O2 -std=c++17 -I paper_2409_12375_b200/csrc tools/tc_probe.cu -o tc_probe
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "tcgen05.h"

using namespace xrl::tc;

constexpr int M = 128, N = 96, K = 128;
constexpr int A_BYTES = M * K * 4, B_BYTES = N * K * 4;

static float tf32_host(float x)
{
    uint32_t u;
    std::memcpy(&u, &x, 4);
    u = (u + 0x1000u) & 0xFFFFE000u;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
}

__global__ void k_probe(const float* __restrict__ ahi_img, const float* __restrict__ alo_img,
                        const float* __restrict__ B /* [N][K] */, float* __restrict__ D /* [M][N] */, int three)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    float* Ah = reinterpret_cast<float*>(sm);
    float* Al = reinterpret_cast<float*>(sm + A_BYTES);
    float* Bh = reinterpret_cast<float*>(sm + 2 * A_BYTES);
    float* Bl = reinterpret_cast<float*>(sm + 2 * A_BYTES + B_BYTES);
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < M * K; i += blockDim.x) { Ah[i] = ahi_img[i]; Al[i] = alo_img[i]; }
    for (int i = tid; i < N * K; i += blockDim.x) {
        const int n = i / K, k = i % K;
        const float x = B[i];
        const float h = tf32_rna(x);
        Bh[core_offset(n, k, N) / 4] = h;
        Bl[core_offset(n, k, N) / 4] = x - h;
    }
    if (tid == 0) mbar_init(&bar, 1);
    if (warp == 0) tmem_alloc<128>(&tbase);
    fence_proxy_async();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t d = tbase;
    if (tid == 0) {
        const uint32_t idesc = idesc_tf32(M, N);
        const uint32_t a0 = smem_u32(Ah), al0 = smem_u32(Al), b0 = smem_u32(Bh), bl0 = smem_u32(Bl);
        const uint32_t lboA = (M / 8) * 128, lboB = (N / 8) * 128;
        for (int s = 0; s < K / 8; ++s) {
            const uint64_t ah = smem_desc(a0 + s * 2 * lboA, lboA, 128), al = smem_desc(al0 + s * 2 * lboA, lboA, 128);
            const uint64_t bh = smem_desc(b0 + s * 2 * lboB, lboB, 128), bl = smem_desc(bl0 + s * 2 * lboB, lboB, 128);
            mma_tf32(d, ah, bh, idesc, s > 0);
            if (three) {
                mma_tf32(d, ah, bl, idesc, 1);
                mma_tf32(d, al, bh, idesc, 1);
            }
        }
        commit(&bar);
    }
    mbar_wait(&bar, 0);
    fence_after();
    float v[32];
    for (int c = 0; c < N; c += 32) {
        tmem_ld32(d + ((uint32_t)(32 * warp) << 16) + c, v);
        for (int j = 0; j < 32; ++j) D[(32 * warp + lane) * N + c + j] = v[j];
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<128>(tbase);
}

// Variant: A (row-major [M][K], hi and lo) stored into TMEM with tcgen05.st (lane = row, column = k),
// MMA with A from TMEM ("TS" form).  TMEM: D cols [0,128), A_hi [128,256), A_lo [256,384).
__global__ void k_probe_ts(const float* __restrict__ A /* [M][K] */, const float* __restrict__ B /* [N][K] */,
                           float* __restrict__ D)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    float* Bh = reinterpret_cast<float*>(sm);
    float* Bl = reinterpret_cast<float*>(sm + B_BYTES);
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < N * K; i += blockDim.x) {
        const int n = i / K, k = i % K;
        const float x = B[i];
        const float h = tf32_rna(x);
        Bh[core_offset(n, k, N) / 4] = h;
        Bl[core_offset(n, k, N) / 4] = x - h;
    }
    if (tid == 0) mbar_init(&bar, 1);
    if (warp == 0) tmem_alloc<512>(&tbase);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t d = tbase;
    {
        const int row = 32 * warp + lane;
        float hv[32], lv[32];
        for (int c = 0; c < K; c += 32) {
            for (int j = 0; j < 32; ++j) {
                const float a = A[row * K + c + j];
                hv[j] = tf32_rna(a);
                lv[j] = a - hv[j];
            }
            tmem_st32(d + ((uint32_t)(32 * warp) << 16) + 128 + c, hv);
            tmem_st32(d + ((uint32_t)(32 * warp) << 16) + 256 + c, lv);
        }
        tmem_st_wait();
    }
    fence_proxy_async();
    fence_before();
    __syncthreads();
    fence_after();
    if (tid == 0) {
        const uint32_t idesc = idesc_tf32(M, N);
        const uint32_t b0 = smem_u32(Bh), bl0 = smem_u32(Bl);
        const uint32_t lboB = (N / 8) * 128;
        for (int s = 0; s < K / 8; ++s) {
            const uint64_t bh = smem_desc(b0 + s * 2 * lboB, lboB, 128), bl = smem_desc(bl0 + s * 2 * lboB, lboB, 128);
            mma_tf32_ts(d, d + 256 + 8 * s, bh, idesc, s > 0);
            mma_tf32_ts(d, d + 128 + 8 * s, bl, idesc, 1);
            mma_tf32_ts(d, d + 128 + 8 * s, bh, idesc, 1);
        }
        commit(&bar);
    }
    mbar_wait(&bar, 0);
    fence_after();
    float v[32];
    for (int c = 0; c < N; c += 32) {
        tmem_ld32(d + ((uint32_t)(32 * warp) << 16) + c, v);
        for (int j = 0; j < 32; ++j) D[(32 * warp + lane) * N + c + j] = v[j];
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tbase);
}

int main()
{
    std::mt19937 g(1);
    std::uniform_real_distribution<float> u(-1, 1);
    std::vector<float> A(M * K, 0.f), B(N * K), ahi(M * K, 0.f), alo(M * K, 0.f);
    for (int i = 0; i < 121; ++i)
        for (int k = 0; k < 121; ++k) A[i * K + k] = u(g) * std::pow(10.f, (float)(i % 7) - 3.f);
    for (auto& x : B) x = u(g);
    for (int i = 0; i < M; ++i)
        for (int k = 0; k < K; ++k) {
            const float a = A[i * K + k], h = tf32_host(a);
            ahi[core_offset(i, k, M) / 4] = h;
            alo[core_offset(i, k, M) / 4] = a - h;
        }
    float *dA, *dAl, *dB, *dD;
    cudaMalloc(&dA, A_BYTES); cudaMalloc(&dAl, A_BYTES); cudaMalloc(&dB, B_BYTES); cudaMalloc(&dD, M * N * 4);
    cudaMemcpy(dA, ahi.data(), A_BYTES, cudaMemcpyHostToDevice);
    cudaMemcpy(dAl, alo.data(), A_BYTES, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B_BYTES, cudaMemcpyHostToDevice);
    const int smem = 2 * A_BYTES + 2 * B_BYTES;
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int fails = 0;
    for (int three = 0; three < 2; ++three) {
        cudaMemset(dD, 0, M * N * 4);
        k_probe<<<1, 128, smem>>>(dA, dAl, dB, dD, three);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { std::printf("CUDA error %s\n", cudaGetErrorString(e)); return 2; }
        std::vector<float> D(M * N);
        cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
        double emax = 0, rel_rms_num = 0, rel_rms_den = 0;
        for (int i = 0; i < M; ++i)
            for (int n = 0; n < N; ++n) {
                double ref = 0;
                for (int k = 0; k < K; ++k) ref += (double)A[i * K + k] * B[n * K + k];
                double row_scale = 0;
                for (int k = 0; k < K; ++k) row_scale += std::fabs((double)A[i * K + k] * B[n * K + k]);
                const double err = std::fabs(D[i * N + n] - ref);
                if (row_scale > 0) emax = std::max(emax, err / row_scale);
                rel_rms_num += err * err;
                rel_rms_den += ref * ref;
            }
        const double rel = std::sqrt(rel_rms_num / rel_rms_den);
        std::printf("%s: max err / sum|a b| = %.3e   rel L2 = %.3e\n", three ? "3xTF32" : "1xTF32", emax, rel);
        if (three && !(emax < 2e-6)) ++fails;
        if (!three && !(emax < 2e-2)) ++fails;
    }
    {
        float* dAf;
        cudaMalloc(&dAf, A_BYTES);
        cudaMemcpy(dAf, A.data(), A_BYTES, cudaMemcpyHostToDevice);
        cudaFuncSetAttribute(k_probe_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * B_BYTES);
        cudaMemset(dD, 0, M * N * 4);
        k_probe_ts<<<1, 128, 2 * B_BYTES>>>(dAf, dB, dD);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { std::printf("CUDA error %s\n", cudaGetErrorString(e)); return 2; }
        std::vector<float> D(M * N);
        cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
        double emax = 0;
        for (int i = 0; i < M; ++i)
            for (int n = 0; n < N; ++n) {
                double ref = 0, sc = 0;
                for (int k = 0; k < K; ++k) { ref += (double)A[i * K + k] * B[n * K + k]; sc += std::fabs((double)A[i * K + k] * B[n * K + k]); }
                if (sc > 0) emax = std::max(emax, std::fabs(D[i * N + n] - ref) / sc);
            }
        std::printf("3xTF32 A-in-TMEM: max err / sum|a b| = %.3e\n", emax);
        if (!(emax < 2e-6)) ++fails;
    }
    std::printf("%s\n", fails ? "PROBE FAILED" : "PROBE OK");
    return fails ? 1 : 0;
}
