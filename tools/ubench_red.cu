// Microbenchmark: L2 reduction (red.global.add.f32) throughput by access pattern,
// for the M2L drain design.  Payload bytes / s into an L2-resident 24 MB buffer.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_red ubench_red.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kRows = 8192;        // rows of 768 floats (3 KB): 24 MB
constexpr int kRowF = 768;

__device__ __forceinline__ void red4(float* p, float a, float b, float c, float d)
{
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// (1) lane = row (stride 3 KB), each lane writes 31 x v4 along its row (current drain)
__global__ void k_rowlane(float* buf, int iters)
{
    const int lane = threadIdx.x & 31, w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (int it = 0; it < iters; ++it) {
        const int row = ((w * 32 + lane) * 7 + it * 131) % kRows;
        float* o = buf + (size_t)row * kRowF;
#pragma unroll 4
        for (int q = 0; q < 31; ++q) red4(o + 4 * q, 1.f, 1.f, 1.f, 1.f);
    }
}
// (2) warp covers one row contiguously with v4 (lane -> 4 floats, 32 lanes = 128 floats)
__global__ void k_contig_v4(float* buf, int iters)
{
    const int lane = threadIdx.x & 31, w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (int it = 0; it < iters; ++it) {
#pragma unroll 4
        for (int q = 0; q < 31; ++q) {
            const int row = ((w * 31 + q) * 7 + it * 131) % kRows;
            float* o = buf + (size_t)row * kRowF;
            if (lane < 31) red4(o + 4 * lane, 1.f, 1.f, 1.f, 1.f);
        }
    }
}
// (3) warp covers 32 consecutive floats with scalar red (lane = coefficient)
__global__ void k_contig_f32(float* buf, int iters)
{
    const int lane = threadIdx.x & 31, w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (int it = 0; it < iters; ++it) {
#pragma unroll 4
        for (int q = 0; q < 124; ++q) {  // same payload per warp as (1): 124 x 128 B
            const int row = ((w * 31 + q / 4) * 7 + it * 131) % kRows;
            float* o = buf + (size_t)row * kRowF + 32 * (q & 3);
            atomicAdd(o + lane, 1.f);
        }
    }
}
__device__ __forceinline__ void red2(float* p, float a, float b)
{
    asm volatile("red.global.add.v2.f32 [%0], {%1,%2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}
// (5) tcgen05.ld 16x256b-like layout: 4 lanes cover 32 B of one row, a warp 8 rows x 32 B per instruction (v2)
__global__ void k_rows8_v2(float* buf, int iters)
{
    const int lane = threadIdx.x & 31, w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (int it = 0; it < iters; ++it) {
        for (int g = 0; g < 4; ++g) {  // 4 groups of 8 rows = 32 rows per warp (as (1))
            const int row = ((w * 32 + 8 * g + lane / 4) * 7 + it * 131) % kRows;
            float* o = buf + (size_t)row * kRowF + 2 * (lane & 3);
#pragma unroll 4
            for (int q = 0; q < 16; ++q) red2(o + 8 * q, 1.f, 1.f);  // 128 floats per row (124 in (1))
        }
    }
}
// (6) 2 lanes cover 32 B of one row with v4: a warp 16 rows x 32 B per instruction
__global__ void k_rows16_v4(float* buf, int iters)
{
    const int lane = threadIdx.x & 31, w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (int it = 0; it < iters; ++it) {
        for (int g = 0; g < 2; ++g) {
            const int row = ((w * 32 + 16 * g + lane / 2) * 7 + it * 131) % kRows;
            float* o = buf + (size_t)row * kRowF + 4 * (lane & 1);
#pragma unroll 4
            for (int q = 0; q < 16; ++q) red4(o + 8 * q, 1.f, 1.f, 1.f, 1.f);
        }
    }
}
// (4) plain v4 stores, contiguous (reference)
__global__ void k_store(float* buf, int iters)
{
    const int lane = threadIdx.x & 31, w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (int it = 0; it < iters; ++it) {
#pragma unroll 4
        for (int q = 0; q < 31; ++q) {
            const int row = ((w * 31 + q) * 7 + it * 131) % kRows;
            float4* o = reinterpret_cast<float4*>(buf + (size_t)row * kRowF);
            if (lane < 31) o[lane] = make_float4(1.f, 1.f, 1.f, (float)it);
        }
    }
}

int main()
{
    float* buf;
    cudaMalloc(&buf, (size_t)kRows * kRowF * 4);
    cudaMemset(buf, 0, (size_t)kRows * kRowF * 4);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = nsm * 4, block = 256, iters = 16;
    const double warps = (double)grid * block / 32;
    auto run = [&](const char* name, auto launch, double bytes) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-12s %8.3f ms  %8.1f GB/s payload\n", name, ms / 5, bytes / (ms / 5 * 1e-3) / 1e9);
    };
    const double payload = warps * iters * 31 * 32 * 16.0;  // (1): per warp 31 x 32 lanes x 16 B
    run("rowlane_v4", [&] { k_rowlane<<<grid, block>>>(buf, iters); }, payload);
    run("contig_v4", [&] { k_contig_v4<<<grid, block>>>(buf, iters); }, warps * iters * 31 * 31 * 16.0);
    run("contig_f32", [&] { k_contig_f32<<<grid, block>>>(buf, iters); }, warps * iters * 124 * 128.0);
    run("rows8_v2", [&] { k_rows8_v2<<<grid, block>>>(buf, iters); }, warps * iters * 32 * 128 * 4.0);
    run("rows16_v4", [&] { k_rows16_v4<<<grid, block>>>(buf, iters); }, warps * iters * 32 * 128 * 4.0);
    run("store_v4", [&] { k_store<<<grid, block>>>(buf, iters); }, warps * iters * 31 * 31 * 16.0);
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
