// Microbenchmark: tcgen05.mma issue/completion rate per SM for the M2L shapes.
// One CTA per SM, one thread issues kReps x 48 MMAs (M128 N128, K = 8 tf32 / 16 bf16)
// into one TMEM accumulator; cycles per MMA from clock64 around issue + commit wait.
// Variants: B operand layout in shared memory (no swizzle with two LBO/SBO choices,
// 128B swizzle), A in TMEM (TS) or shared memory (SS), kind::tf32 vs kind::f16.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2409_12375_b200/csrc -o ubench_mma ubench_mma.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tcgen05.h"

using namespace xrl::tc;

constexpr int kReps = 64;

__device__ __forceinline__ uint64_t desc_sw(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout)
{
    uint64_t d = smem_desc(saddr, lbo, sbo);
    d |= (uint64_t)layout << 61;
    return d;
}

__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc, int f16)
{
    if (f16)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
                     "l"(a), "l"(b), "r"(idesc), "r"(acc));
    else
        mma_tf32(d_tmem, a, b, idesc, acc);
}
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc, int f16)
{
    if (f16)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
                     "r"(a), "l"(b), "r"(idesc), "r"(acc));
    else
        mma_tf32_ts(d_tmem, a, b, idesc, acc);
}

// variant: 0 TS noswz LBO128/SBO4096, 1 TS noswz LBO2048/SBO128, 2 TS sw128, 3 SS noswz, 4 SS sw128
__global__ void k_mma(int variant, int f16, long long* out)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 2 * 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.001f * (i & 255);
    if (tid == 0) mbar_init(&bar, 1);
    if (warp == 0) tmem_alloc<512>(&tbase);
    fence_proxy_async();
    fence_before();
    __syncthreads();
    fence_after();
    if (tid == 0) {
        // kind::f16 idesc: a/b format BF16 = 1 at bits 7, 10; D F32
        const uint32_t idesc = f16 ? ((1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24))
                                   : idesc_tf32(128, 128);
        const uint32_t b0 = smem_u32(sm), a0 = smem_u32(sm + 65536);
        const uint32_t d = tbase + 256;
        long long t0 = clock64();
        for (int rep = 0; rep < kReps; ++rep) {
            for (int m = 0; m < 48; ++m) {
                const int s = m % 16;  // K step (32 bytes of K)
                uint64_t bd, ad = 0;
                if (variant == 0 || variant == 3) bd = desc_sw(b0 + 256 * s, 128, 4096, 0);
                else if (variant == 1) bd = desc_sw(b0 + 2 * 2048 * s, 2048, 128, 0);
                else bd = desc_sw(b0 + (s / 4) * 16384 + (s % 4) * 32, 16, 1024, 2);
                if (variant == 3) ad = desc_sw(a0 + 256 * s, 128, 4096, 0);
                if (variant == 4) ad = desc_sw(a0 + (s / 4) * 16384 + (s % 4) * 32, 16, 1024, 2);
                if (variant <= 2) mma_ts(d, tbase + 8 * s, bd, idesc, (rep | m) != 0, f16);
                else mma_ss(d, ad, bd, idesc, (rep | m) != 0, f16);
            }
        }
        commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tbase);
}

// tight issue loop: descriptors precomputed, K steps unrolled; mode 0: lane 0 (divergent), 1: elect.sync in a converged warp
template <int kMode, int kLayout>
__global__ void k_mma_tight(long long* out)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 2 * 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.001f * (i & 255);
    if (tid == 0) mbar_init(&bar, 1);
    if (warp == 0) tmem_alloc<512>(&tbase);
    fence_proxy_async();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tb = tbase;
    const uint32_t idesc = idesc_tf32(128, 128);
    // layout 0: LBO 2048 / SBO 128 ([kc][ig][128 B]); 1: LBO 128 / SBO 4096 ([ig][kc][128 B]); 2: SW128 K-major
    const uint64_t b0 = kLayout == 0 ? smem_desc(smem_u32(sm), 2048, 128)
                      : kLayout == 1 ? smem_desc(smem_u32(sm), 128, 4096)
                                     : desc_sw(smem_u32(sm), 16, 1024, 2);
    if (warp == 0) {
        const bool leader = kMode == 0 ? lane == 0 : elect_one();
        long long t0 = clock64();
        if (kMode == 0 && lane != 0) { }
        else if (leader) {
            for (int rep = 0; rep < kReps; ++rep) {
#pragma unroll
                for (int s = 0; s < 16; ++s) {
                    const uint32_t boff = kLayout == 0 ? 2 * 2048 * s : kLayout == 1 ? 256 * s : (s / 4) * 16384 + (s % 4) * 32;
                    const uint64_t bd = b0 + (uint64_t)(boff >> 4);
                    mma_tf32_ts(tb + 256, tb + 8 * s, bd, idesc, (rep | s) != 0);
                    mma_tf32_ts(tb + 256, tb + 128 + 8 * s, bd, idesc, 1);
                    mma_tf32_ts(tb + 256, tb + 8 * s, bd, idesc, 1);
                }
            }
            commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (lane == 0) out[blockIdx.x] = t1 - t0;
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tbase);
}

int main()
{
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    long long* out;
    cudaMallocManaged(&out, nsm * sizeof(long long));
    cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 65536);
    const char* names[] = {"TS noswz LBO128 SBO4096", "TS noswz LBO2048 SBO128", "TS sw128", "SS noswz", "SS sw128"};
    for (int f16 = 0; f16 < 2; ++f16)
        for (int v = 0; v < 5; ++v) {
            k_mma<<<nsm, 128, 2 * 65536>>>(v, f16, out);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("%s: %s\n", names[v], cudaGetErrorString(e)); return 1; }
            double avg = 0;
            for (int i = 0; i < nsm; ++i) avg += out[i];
            avg /= nsm;
            printf("%s %-26s %8.1f cycles per MMA (M128 N128 K%d)\n", f16 ? "bf16" : "tf32", names[v],
                   avg / (kReps * 48), f16 ? 16 : 8);
        }
    auto tight = [&](auto kern, const char* name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 65536);
        kern<<<nsm, 128, 2 * 65536>>>(out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("tight: %s\n", cudaGetErrorString(e)); return; }
        double avg = 0;
        for (int i = 0; i < nsm; ++i) avg += out[i];
        avg /= nsm;
        printf("tf32 tight TS %-28s %8.1f cycles per MMA (M128 N128 K8)\n", name, avg / (kReps * 48));
    };
    tight(k_mma_tight<0, 0>, "lane0 LBO2048/SBO128");
    tight(k_mma_tight<1, 0>, "elect LBO2048/SBO128");
    tight(k_mma_tight<1, 1>, "elect LBO128/SBO4096");
    tight(k_mma_tight<1, 2>, "elect SW128");
    return 0;
}
