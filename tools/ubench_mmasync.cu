// Microbenchmark: legacy warp-level mma.sync.m16n8k8 TF32 (f32 accumulate) issue throughput on sm_100a,
// for a P2P whose accumulation y += G q runs on the tensor core.  Independent accumulator chains per warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_mmasync.bin tools/ubench_mmasync.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int kChains>
__global__ void k_mma(float* out, int iters)
{
    unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    float d[kChains][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < kChains; ++c)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                         "{%0,%1,%2,%3};"
                         : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main()
{
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, 1 << 26);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int warps = 4; warps <= 16; warps *= 2) {
        const int grid = nsm * 2, block = 32 * warps;
        auto run = [&](auto kern, int chains) {
            kern<<<grid, block>>>(out, iters);
            cudaDeviceSynchronize();
            cudaEventRecord(e0);
            kern<<<grid, block>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double flops = 2.0 * 16 * 8 * 8 * chains * (double)iters * grid * warps;
            printf("warps/CTA %2d (2 CTA/SM) chains %d: %.1f TFLOP/s tf32 mma.sync (%.3f mma/clk/SM at 1965 MHz)\n",
                   warps, chains, flops / ms / 1e9, flops / 2048 / (ms * 1e-3) / nsm / 1.965e9);
        };
        run(k_mma<2>, 2);
        run(k_mma<4>, 4);
        run(k_mma<8>, 8);
    }
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
