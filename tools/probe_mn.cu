// Probe: tcgen05.mma kind::tf32 M128 N16 K8 with A in TMEM and B in shared
// memory in the canonical MN-major (no swizzle) layout used by k_p2p_tc:
// B element (n, k) at byte (n%4)*4 + (n/4)*G + (k%8)*16 + (k/8)*128 (planes of
// G bytes), checked against a host product for candidate (LBO, SBO) encodings.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2409_12375_b200/csrc tools/probe_mn.cu -o probe_mn
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "tcgen05.h"

using namespace xrl::tc;

constexpr int M = 128, N = 16, K = 16, G = 1024;  // K = 16: two MMAs (K steps) to exercise the K-group stride

__global__ void k_probe(const float* __restrict__ A /* [M][K] */, const float* __restrict__ Bimg /* smem image */,
                        int img_floats, uint32_t lbo, uint32_t sbo, uint32_t mn, uint32_t kstep,
                        float* __restrict__ D /* [M][N] */)
{
    extern __shared__ __align__(1024) float sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < img_floats; i += blockDim.x) sm[i] = Bimg[i];
    if (tid == 0) mbar_init(&bar, 1);
    if (warp == 0) tmem_alloc<64>(&tbase);
    fence_proxy_async();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tm = tbase;
    {  // A row tid -> TMEM lane tid, columns 16..31
        float v[16];
        for (int k = 0; k < 16; ++k) v[k] = A[tid * K + k];
        float w[8];
        for (int q = 0; q < 8; ++q) w[q] = v[q];
        tmem_st8(tm + ((uint32_t)(32 * warp) << 16) + 16, w);
        for (int q = 0; q < 8; ++q) w[q] = v[8 + q];
        tmem_st8(tm + ((uint32_t)(32 * warp) << 16) + 24, w);
        tmem_st_wait();
    }
    fence_before();
    __syncthreads();
    fence_after();
    if (tid == 0) {
        const uint32_t idesc = idesc_tf32(M, N) | (mn << 16);
        const uint32_t b0 = smem_u32(sm);
        for (int ks = 0; ks < K / 8; ++ks)
            mma_tf32_ts(tm, tm + 16 + 8 * ks, smem_desc(b0 + kstep * ks, lbo, sbo), idesc, ks > 0);
        commit(&bar);
    }
    mbar_wait(&bar, 0);
    fence_after();
    float v[16];
    tmem_ld16(tm + ((uint32_t)(32 * warp) << 16), v);
    for (int n = 0; n < N; ++n) D[tid * N + n] = v[n];
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<64>(tbase);
}

int main()
{
    std::vector<float> A(M * K), B(N * K);
    for (int i = 0; i < M * K; ++i) A[i] = (float)((i * 37 % 101) - 50) / 64.f;  // exact in TF32
    for (int i = 0; i < N * K; ++i) B[i] = (float)((i * 53 % 97) - 48) / 32.f;
    // smem image: plane g = n/4 at g*G bytes, source k at (k%8)*16 + (k/8)*128, lane n%4
    const int img = 4 * G / 4;
    std::vector<float> im(img, 0.f);
    for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k) im[(n / 4) * (G / 4) + (k % 8) * 4 + (k / 8) * 32 + n % 4] = B[n * K + k];
    std::vector<double> ref(M * N, 0.0);
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n)
            for (int k = 0; k < K; ++k) ref[m * N + n] += (double)A[m * K + k] * B[n * K + k];
    float *dA, *dB, *dD;
    cudaMalloc(&dA, 4 * A.size());
    cudaMalloc(&dB, 4 * img);
    cudaMalloc(&dD, 4 * M * N);
    cudaMemcpy(dA, A.data(), 4 * A.size(), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * img);
    auto run = [&](const std::vector<float>& image, uint32_t lbo, uint32_t sbo, uint32_t mn, uint32_t kstep,
                   const char* name) {
        cudaMemcpy(dB, image.data(), 4 * img, cudaMemcpyHostToDevice);
        cudaMemset(dD, 0, 4 * M * N);
        k_probe<<<1, 128, 4 * img>>>(dA, dB, img, lbo, sbo, mn, kstep, dD);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> D(M * N);
        cudaMemcpy(D.data(), dD, 4 * M * N, cudaMemcpyDeviceToHost);
        double err = 0, nrm = 0;
        for (int i = 0; i < M * N; ++i) { err += (D[i] - ref[i]) * (D[i] - ref[i]); nrm += ref[i] * ref[i]; }
        printf("%-10s LBO %5u SBO %5u: %s rel err %.3e  D[0]=%g ref %g\n", name, lbo, sbo, cudaGetErrorString(e),
               std::sqrt(err / nrm), D[0], ref[0]);
    };
    // K-major control: element (n, k) at ((k/4)*2 + n/8)*128 + (n%8)*16 + (k%4)*4 bytes, LBO 256, SBO 128
    std::vector<float> kimg(img, 0.f);
    for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k) kimg[((k / 4) * 2 + n / 8) * 32 + (n % 8) * 4 + k % 4] = B[n * K + k];
    run(kimg, 256, 128, 0, 512, "K-major");
    const uint32_t cand[][2] = {{128, 1024}, {1024, 128}, {128, 512}, {512, 128}, {16, 1024}, {1024, 16}};
    for (auto& c : cand) run(im, c[0], c[1], 1, 128, "MN-major");
    return 0;
}
