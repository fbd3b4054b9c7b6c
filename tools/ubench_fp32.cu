// Microbenchmark: FP32 pipe throughput on B200 for the P2P inner loop choices.
//   FFMA (3-reg), FFMA2 (fma.rn.f32x2), MUFU.RSQ, and the two P2P pair bodies
//   (scalar 12 FP32 instr + RSQ, packed 6 f32x2 instr + RSQ).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_fp32 ubench_fp32.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void k_ffma(float* out, float s)
{
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
    const float b = s * 0.999f, c = s * 1e-4f;
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, c);
    float t = 0;
    for (int i = 0; i < 8; ++i) t += a[i];
    if (t == 12345.f) out[0] = t;
}

__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }

__global__ void k_ffma2(float* out, float s)
{
    unsigned long long a[8];
    for (int i = 0; i < 8; ++i) a[i] = f2u(make_float2(threadIdx.x * 1e-3f + i, i * 0.5f));
    const unsigned long long b = f2u(make_float2(s * 0.999f, s * 0.998f)), c = f2u(make_float2(s * 1e-4f, s * 2e-4f));
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(b), "l"(c));
    float t = 0;
    for (int i = 0; i < 8; ++i) { float2 v = *reinterpret_cast<float2*>(&a[i]); t += v.x + v.y; }
    if (t == 12345.f) out[0] = t;
}

__global__ void k_rsq(float* out, float s)
{
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = 1.f + threadIdx.x * 1e-3f + i;
    for (int it = 0; it < kIters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = rsqrtf(a[i]);
    float t = 0;
    for (int i = 0; i < 8; ++i) t += a[i];
    if (t == 12345.f) out[0] = t;
}

// scalar P2P body: 8 targets x 1 source per step (as k_p2p)
__global__ void k_p2p_scalar(const float4* __restrict__ src, float* out, int ns)
{
    float tx[8], ty[8], tz[8], f[8][6];
    for (int q = 0; q < 8; ++q) {
        tx[q] = threadIdx.x * 1e-3f + q; ty[q] = q * 0.3f; tz[q] = 0.1f * q;
        for (int r = 0; r < 6; ++r) f[q][r] = 0.f;
    }
    for (int rep = 0; rep < 8; ++rep)
        for (int j = 0; j < ns; ++j) {
            const float4 sp = src[2 * j], q0 = src[2 * j + 1];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const float dx = tx[q] - sp.x, dy = ty[q] - sp.y, dz = tz[q] - sp.z;
                const float ri = rsqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
                f[q][0] = fmaf(q0.x, ri, f[q][0]); f[q][1] = fmaf(q0.y, ri, f[q][1]);
                f[q][2] = fmaf(q0.z, ri, f[q][2]); f[q][3] = fmaf(q0.w, ri, f[q][3]);
                f[q][4] = fmaf(sp.w, ri, f[q][4]); f[q][5] = fmaf(q0.x, ri, f[q][5]);
            }
        }
    float t = 0;
    for (int q = 0; q < 8; ++q) for (int r = 0; r < 6; ++r) t += f[q][r];
    if (t == 12345.f) out[0] = t;
}

__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c)
{
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ unsigned long long sub2(unsigned long long a, unsigned long long b)
{
    unsigned long long d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long mul2(unsigned long long a, unsigned long long b)
{
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

// packed P2P body: 8 targets (4 packed pairs) x 1 source; accumulators packed over RHS pairs
__global__ void k_p2p_packed(const float4* __restrict__ src, float* out, int ns)
{
    unsigned long long tx[4], ty[4], tz[4], f[8][3];
    for (int q = 0; q < 4; ++q) {
        tx[q] = f2u(make_float2(threadIdx.x * 1e-3f + q, q + 0.5f));
        ty[q] = f2u(make_float2(q * 0.3f, q * 0.2f));
        tz[q] = f2u(make_float2(q * 0.1f, q * 0.7f));
    }
    for (int q = 0; q < 8; ++q) for (int r = 0; r < 3; ++r) f[q][r] = 0ull;
    for (int rep = 0; rep < 8; ++rep)
        for (int j = 0; j < ns; ++j) {
            const float4 sp = src[2 * j], q0 = src[2 * j + 1];
            const unsigned long long sx = f2u(make_float2(sp.x, sp.x)), sy = f2u(make_float2(sp.y, sp.y)),
                                     sz = f2u(make_float2(sp.z, sp.z));
            const unsigned long long qa = f2u(make_float2(q0.x, q0.y)), qb = f2u(make_float2(q0.z, q0.w)),
                                     qc = f2u(make_float2(sp.w, q0.x));
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const unsigned long long dx = sub2(tx[q], sx), dy = sub2(ty[q], sy), dz = sub2(tz[q], sz);
                const unsigned long long r2 = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
                const float2 r2v = *reinterpret_cast<const float2*>(&r2);
                const float ra = rsqrtf(r2v.x), rb = rsqrtf(r2v.y);
                const unsigned long long A = f2u(make_float2(ra, ra)), B = f2u(make_float2(rb, rb));
                f[2 * q][0] = fma2(qa, A, f[2 * q][0]); f[2 * q][1] = fma2(qb, A, f[2 * q][1]);
                f[2 * q][2] = fma2(qc, A, f[2 * q][2]);
                f[2 * q + 1][0] = fma2(qa, B, f[2 * q + 1][0]); f[2 * q + 1][1] = fma2(qb, B, f[2 * q + 1][1]);
                f[2 * q + 1][2] = fma2(qc, B, f[2 * q + 1][2]);
            }
        }
    float t = 0;
    for (int q = 0; q < 8; ++q) for (int r = 0; r < 3; ++r) { float2 v = *reinterpret_cast<float2*>(&f[q][r]); t += v.x + v.y; }
    if (t == 12345.f) out[0] = t;
}

int main()
{
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, 4);
    const int ns = 2048;
    float4* src;
    cudaMalloc(&src, 2 * ns * sizeof(float4));
    cudaMemset(src, 0, 2 * ns * sizeof(float4));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = nsm * 8, block = 256;
    auto run = [&](const char* name, auto launch, double ops_per_thread, const char* unit) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double tot = ops_per_thread * grid * block * 5;
        printf("%-14s %8.3f ms  %10.2f G%s/s  (%.2f per SM per clk @1965MHz)\n", name, ms / 5, tot / (ms * 1e-3) / 1e9, unit,
               tot / (ms * 1e-3) / nsm / 1.965e9);
    };
    run("ffma", [&] { k_ffma<<<grid, block>>>(out, 1.f); }, 8.0 * kIters, "inst");
    run("ffma2", [&] { k_ffma2<<<grid, block>>>(out, 1.f); }, 8.0 * kIters, "inst");
    run("rsqrt", [&] { k_rsq<<<grid, block>>>(out, 1.f); }, 8.0 * kIters, "inst");
    run("p2p_scalar", [&] { k_p2p_scalar<<<grid, block>>>(src, out, ns); }, 8.0 * 8 * ns, "pair");
    run("p2p_packed", [&] { k_p2p_packed<<<grid, block>>>(src, out, ns); }, 8.0 * 8 * ns, "pair");
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
