// xrl_mvm: the FMM-accelerated panel MVM.
//
// y_t = P x_t for t = 1..3 (Eq. 9: three panel-space
// applications of P per loop-space MVM, FMM over centroids PAPER.md:116).
// All six real right-hand sides (re/im of 3 components) go through one tree
// pass.  Far field: Laplace FMM (order p = 10, real semi-normalised solid
// harmonics, operators.h); near field: P2P over adjacent leaves plus the CSR
// correction N = P - 1/r (near.cu).
//
// Kernels (one launch each unless noted):
//   k_pack     complex64 [3][n] -> float [n][8] charges          (HBM, 48 B/panel)
//   k_p2m      leaf multipoles mu = sum q Rt(u)                   (per leaf)
//   k_m2m      child -> parent, per level (bottom-up)
//   k_m2l      V-list translations, batched by offset: the 121x121 operator
//              stays in shared memory while 32 (target, source) pairs x 6
//              RHS stream through it (SGEMM-like register tiling, 8x12 per
//              thread); results are accumulated with red.global.add.v4.f32
//   k_p2l      X-list particle -> local
//   k_l2l      parent -> child, per level (top-down)
//   k_leaf     per target leaf: L2P + M2P (W list) + P2P (U list) + near CSR,
//              writes y once
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "tcgen05.h"
#include "xrl_internal.h"

using namespace xrl;

__constant__ RecTables<float> c_tab;

namespace {

constexpr int kTP = 16;          // pairs per M2L tile
constexpr int kBCols = kTP * 6 + 4;  // 96 columns of the M2L B tile (+4 pad: spreads the gather over banks)

__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d)
{
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

__device__ __forceinline__ float3 box_center(int level, int ix, int iy, int iz)
{
    const float s = ldexpf(1.f, -level);
    return make_float3((ix + 0.5f) * s, (iy + 0.5f) * s, (iz + 0.5f) * s);
}

// ------------------------------------------------------------------ pack
__global__ void k_pack(int64_t n, const float2* __restrict__ x, float* __restrict__ xq)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    float2 a = x[i], b = x[n + i], c = x[2 * n + i];
    float4* o = reinterpret_cast<float4*>(xq + 8 * i);
    o[0] = make_float4(a.x, a.y, b.x, b.y);
    o[1] = make_float4(c.x, c.y, 0.f, 0.f);
}

// ------------------------------------------------------------------ P2M
constexpr int kChunk = 64;

__global__ void __launch_bounds__(128) k_p2m(const int32_t* __restrict__ leaves, const int32_t* __restrict__ pb,
                                             const int32_t* __restrict__ pe, const int32_t* __restrict__ level,
                                             const float4* __restrict__ loc, const float* __restrict__ xq,
                                             float* __restrict__ mu)
{
    __shared__ float H[kChunk][kNC];
    __shared__ float Q[kChunk][6];
    const int b = leaves[blockIdx.x];
    const int s = pb[b], e = pe[b];
    const float inv_s = ldexpf(1.f, level[b]);
    float acc[6];
#pragma unroll
    for (int j = 0; j < 6; ++j) acc[j] = 0.f;
    for (int c0 = s; c0 < e; c0 += kChunk) {
        const int cn = min(kChunk, e - c0);
        if (threadIdx.x < cn) {
            const int i = c0 + threadIdx.x;
            float4 p = loc[i];
            float h[kNC];
            regular_harmonics<kP>(p.x * inv_s, p.y * inv_s, p.z * inv_s, c_tab, h);
#pragma unroll
            for (int k = 0; k < kNC; ++k) H[threadIdx.x][k] = h[k];
#pragma unroll
            for (int r = 0; r < 6; ++r) Q[threadIdx.x][r] = xq[8 * (int64_t)i + r];
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            const int o = threadIdx.x + 128 * j;
            if (o < kNC * 6) {
                const int k = o / 6, r = o % 6;
                float a = acc[j];
                for (int p = 0; p < cn; ++p) a += H[p][k] * Q[p][r];
                acc[j] = a;
            }
        }
        __syncthreads();
    }
    float* out = mu + (size_t)b * kBoxStride;
#pragma unroll
    for (int j = 0; j < 6; ++j) {
        const int o = threadIdx.x + 128 * j;
        if (o < kNC * 6) out[o] = acc[j];
        else if (o < kBoxStride) out[o] = 0.f;
    }
}

// ------------------------------------------------------------------ M2M / L2L
// One CTA per output box; op layout [oct][k][kNCP] (i contiguous).
__device__ __forceinline__ int degree_of(int i)
{
    int n = 0;
    while ((n + 1) * (n + 1) <= i) ++n;
    return n;
}

__global__ void __launch_bounds__(128) k_m2m(const int32_t* __restrict__ parents, const int32_t* __restrict__ child,
                                             const int32_t* __restrict__ nchild, const int32_t* __restrict__ ix,
                                             const int32_t* __restrict__ iy, const int32_t* __restrict__ iz,
                                             const float* __restrict__ op, float* __restrict__ mu)
{
    __shared__ float src[kBoxStride];
    const int b = parents[blockIdx.x];
    const int c0 = child[b], nc = nchild[b];
    const int i = threadIdx.x;
    const int kmax = (i < kNC) ? (degree_of(i) + 1) * (degree_of(i) + 1) : 0;
    float acc[6] = {0, 0, 0, 0, 0, 0};
    for (int c = c0; c < c0 + nc; ++c) {
        __syncthreads();
        for (int j = threadIdx.x; j < kBoxStride / 4; j += blockDim.x)
            reinterpret_cast<float4*>(src)[j] = reinterpret_cast<const float4*>(mu + (size_t)c * kBoxStride)[j];
        __syncthreads();
        const int oct = (ix[c] & 1) | ((iy[c] & 1) << 1) | ((iz[c] & 1) << 2);
        const float* T = op + (size_t)oct * kNC * kNCP;
        for (int k = 0; k < kmax; ++k) {
            const float t = T[k * kNCP + i];
#pragma unroll
            for (int r = 0; r < 6; ++r) acc[r] += t * src[6 * k + r];
        }
    }
    if (i < kNC) {
        float* out = mu + (size_t)b * kBoxStride + 6 * i;
#pragma unroll
        for (int r = 0; r < 6; ++r) out[r] = acc[r];
    } else if (i == kNC) {
        mu[(size_t)b * kBoxStride + 726] = 0.f;
        mu[(size_t)b * kBoxStride + 727] = 0.f;
    }
}

__global__ void __launch_bounds__(128) k_l2l(const int32_t* __restrict__ boxes, const int32_t* __restrict__ parent,
                                             const int32_t* __restrict__ ix, const int32_t* __restrict__ iy,
                                             const int32_t* __restrict__ iz, const float* __restrict__ op,
                                             float* __restrict__ ell)
{
    __shared__ float src[kBoxStride];
    const int b = boxes[blockIdx.x];
    const int P = parent[b];
    for (int j = threadIdx.x; j < kBoxStride / 4; j += blockDim.x)
        reinterpret_cast<float4*>(src)[j] = reinterpret_cast<const float4*>(ell + (size_t)P * kBoxStride)[j];
    __syncthreads();
    const int i = threadIdx.x;
    if (i >= kNC) return;
    const int oct = (ix[b] & 1) | ((iy[b] & 1) << 1) | ((iz[b] & 1) << 2);
    const float* T = op + (size_t)oct * kNC * kNCP;
    const int n = degree_of(i);
    float acc[6] = {0, 0, 0, 0, 0, 0};
    for (int k = n * n; k < kNC; ++k) {
        const float t = T[k * kNCP + i];
#pragma unroll
        for (int r = 0; r < 6; ++r) acc[r] += t * src[6 * k + r];
    }
    float* out = ell + (size_t)b * kBoxStride + 6 * i;
#pragma unroll
    for (int r = 0; r < 6; ++r) out[r] += acc[r];
}

// ------------------------------------------------------------------ M2L
// Tile = (offset o, pairs [begin, begin+count)), count <= kTP = 16.  Tiles are
// ordered target-chunk-major (4096 target boxes per chunk), then by offset, so
// the mu gathers and the ell reductions of the tiles in flight stay in L2.
// C[128 x 96] = T_o[128 x 121] * B[121 x 96], B[k][p*6+r] = mu_src(p)[k][r].
// 256 threads: rg = tid % 16 owns rows rg*4..+3 and 64+rg*4..+3 (float4 rows
// contiguous across the 16 lanes: no bank conflicts), cg = tid / 16 owns pair cg.
// 108 KB shared memory -> 2 CTAs per SM so one CTA's loads overlap the other's FMAs.
constexpr int kM2LSmem = (kNC * kNCP + kNC * kBCols) * 4;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__global__ void __launch_bounds__(256, 2) k_m2l(const int4* __restrict__ tiles, const int32_t* __restrict__ tgt,
                                                const int32_t* __restrict__ srcb, const float* __restrict__ ops,
                                                const float* __restrict__ mu, float* __restrict__ ell)
{
    extern __shared__ __align__(16) float sm[];
    float* Ts = sm;                    // [121][128]
    float* Bs = sm + kNC * kNCP;       // [121][96]
    const int4 tile = tiles[blockIdx.x];
    const int off = tile.x, begin = tile.y, count = tile.z;
    const int tid = threadIdx.x;
    {
        const float4* g = reinterpret_cast<const float4*>(ops + (size_t)off * kNC * kNCP);
        float4* s = reinterpret_cast<float4*>(Ts);
        for (int j = tid; j < kNC * kNCP / 4; j += 256) cp_async16(s + j, g + j);
    }
    for (int j = tid; j < kTP * 363; j += 256) {
        const int p = j / 363, q = j % 363;
        const int k = q / 3, r2 = q % 3;
        float* dst = &Bs[k * kBCols + p * 6 + 2 * r2];
        if (p < count) cp_async8(dst, reinterpret_cast<const float2*>(mu + (size_t)srcb[begin + p] * kBoxStride) + q);
        else *reinterpret_cast<float2*>(dst) = make_float2(0.f, 0.f);
    }
    cp_async_wait_all();
    __syncthreads();
    const int rg = tid & 15, cg = tid >> 4;
    float acc[8][6];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int c = 0; c < 6; ++c) acc[a][c] = 0.f;
    const float* tp = Ts + rg * 4;
    const float* bp = Bs + cg * 6;
#pragma unroll 4
    for (int k = 0; k < kNC; ++k) {
        const float4 t0 = *reinterpret_cast<const float4*>(tp + k * kNCP);
        const float4 t1 = *reinterpret_cast<const float4*>(tp + k * kNCP + 64);
        const float2 b0 = *reinterpret_cast<const float2*>(bp + k * kBCols);
        const float2 b1 = *reinterpret_cast<const float2*>(bp + k * kBCols + 2);
        const float2 b2 = *reinterpret_cast<const float2*>(bp + k * kBCols + 4);
        const float tv[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
        const float bv[6] = {b0.x, b0.y, b1.x, b1.y, b2.x, b2.y};
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int c = 0; c < 6; ++c) acc[a][c] = fmaf(tv[a], bv[c], acc[a][c]);
    }
    if (cg >= count) return;
    float* base = ell + (size_t)tgt[begin + cg] * kBoxStride;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int i = (j >> 1) * 64 + rg * 4 + 2 * (j & 1);
        if (i >= kNC) continue;
        float* o = base + 6 * i;
        const float* a0 = acc[2 * j];
        const float* a1 = acc[2 * j + 1];
        red_add_v4(o, a0[0], a0[1], a0[2], a0[3]);
        red_add_v4(o + 4, a0[4], a0[5], a1[0], a1[1]);
        if (i + 1 < kNC) red_add_v4(o + 8, a1[2], a1[3], a1[4], a1[5]);
    }
}

// ------------------------------------------------------------------ M2L on tcgen05
// Tensor-core M2L.  After the upward pass every box's multipole is written once
// as a TF32 hi/lo "image" in the tcgen05 canonical K-major core-matrix layout
// with the 6 RHS padded to 8 rows, i.e. one 8-row core group per box:
//   img[box][hi|lo][kc = k/4][r = 0..7][k % 4]   (32 x 128 B per part, 8 KB per box).
// A sub-tile of 8 (target, source) pairs sharing one offset then needs as B
// operand [kc][pair][128 B] (LBO = 1024 B between K chunks, SBO = 128 B between
// pairs): pure 16-byte cp.async copies.  The operator T_o (hi and lo, 128 x 128
// TF32) lives in TMEM (lane = output coefficient, column = input coefficient),
// written with tcgen05.st when the offset changes, so the MMAs only read B from
// shared memory.  D[128 x 64] (TMEM, FP32) = T_o x B with 3xTF32
// (A_lo B_hi + A_hi B_lo + A_hi B_hi; 48 tcgen05.mma kind::tf32 M128 N64 K8).
// Pipeline (two B buffers, two TMEM accumulators): while MMA(t) runs, the 8
// warps issue the cp.async gather of t+1 and drain the accumulator of t-1
// (tcgen05.ld -> red.global.add.{v4,v2}.f32 into ell).  One persistent CTA per
// SM (TMEM 512 columns) walks blocks of kTcR tiles (same offset -> operator
// reuse), blocks dealt round-robin so all CTAs stay inside one L2-resident
// target chunk.  128 KB of shared memory leaves room for P2P CTAs on the SM.
constexpr int kTcP = 8;                             // pairs per sub-tile
constexpr int kTcN = kTcP * 8;                      // 64 MMA columns (6 RHS + 2 pad per pair)
constexpr int kTcBBytes = kTcN * 128 * 4;           // one B image (hi or lo): 32 KB
constexpr int kTcSmem = 4 * kTcBBytes;              // 2 buffers x (hi, lo)
constexpr int kTcR = 8;
constexpr int kTcThreads = 256;
constexpr int kImgFloats = 2 * 32 * 32;             // per box: hi + lo, 32 K-chunks x 32 floats
constexpr uint32_t kTcColD = 0, kTcColAh = 256, kTcColAl = 384;

__device__ __forceinline__ void red_add_v2(float* p, float a, float b)
{
    asm volatile("red.global.add.v2.f32 [%0], {%1,%2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}

// img[b][part][kc][r][j] = split(mu[b][4 kc + j][r]) for r < 6, k < 121; else 0.
__global__ void k_mu_img(int nbox, const float* __restrict__ mu, float* __restrict__ img)
{
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // one per (box, kc, r, j)
    if (e >= (int64_t)nbox * 1024) return;
    const int b = (int)(e >> 10), w = (int)(e & 1023);
    const int kc = w >> 5, r = (w >> 2) & 7, j = w & 3;
    const int k = 4 * kc + j;
    const float x = (r < 6 && k < kNC) ? mu[(size_t)b * kBoxStride + 6 * k + r] : 0.f;
    const float hi = tc::tf32_rna(x);
    img[(size_t)b * kImgFloats + w] = hi;
    img[(size_t)b * kImgFloats + 1024 + w] = x - hi;
}

__global__ void __launch_bounds__(kTcThreads, 1) k_m2l_tc(const int4* __restrict__ tiles, int ntiles,
                                                          const int32_t* __restrict__ tgt,
                                                          const int32_t* __restrict__ srcb,
                                                          const float* __restrict__ aimg,
                                                          const float* __restrict__ bimg, float* __restrict__ ell)
{
    extern __shared__ __align__(1024) uint8_t tsm[];
    float* Bbase = reinterpret_cast<float*>(tsm);  // [buf][hi/lo][32 kc][8 pairs][32 floats]
    __shared__ uint64_t bar[2];
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) { tc::mbar_init(&bar[0], 1); tc::mbar_init(&bar[1], 1); }
    if (warp == 0) tc::tmem_alloc<512>(&tbase);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t dtm = tbase;
    const uint32_t idesc = tc::idesc_tf32(128, kTcN);
    const uint32_t lboB = kTcP * 128;
    uint32_t ph[2] = {0, 0};
    int cur_off = -1;

    struct Sub { int off, begin, count; };
    auto sub_at = [&](int ti, int half) -> Sub {
        const int4 tile = tiles[ti];
        return {tile.x, tile.y + half * kTcP, min(kTcP, tile.z - half * kTcP)};
    };
    // cp.async of a sub-tile's B operand (hi and lo) into buffer buf: 2 x 32 kc x 8 pairs x 8 x 16 B
    auto gather = [&](const Sub& sb, int buf) {
        float* B = Bbase + (size_t)buf * 2 * (kTcBBytes / 4);
        for (int c = tid; c < 4096; c += kTcThreads) {
            const int part = c >> 11, kc = (c >> 6) & 31, p = (c >> 3) & 7, piece = c & 7;
            float4* dst = reinterpret_cast<float4*>(B + part * (kTcBBytes / 4) + kc * (kTcP * 32) + p * 32) + piece;
            if (p < sb.count) {
                const float4* src = reinterpret_cast<const float4*>(
                    bimg + (size_t)srcb[sb.begin + p] * kImgFloats + part * 1024 + kc * 32) + piece;
                cp_async16(dst, src);
            } else {
                *dst = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    };
    auto wait_mma = [&](int buf) {
        tc::mbar_wait(&bar[buf], ph[buf]);
        ph[buf] ^= 1;
        tc::fence_after();
    };
    auto drain = [&](int buf, const Sub& sb) {
        // lane quarter qd = warp % 4 (coefficients 32 qd + lane); pair group g = warp / 4 owns pairs g, g+2, ...
        const int qd = warp & 3, g = warp >> 2;
        const int i = 32 * qd + lane;
#pragma unroll
        for (int pp = 0; pp < kTcP / 2; ++pp) {
            const int p = g + 2 * pp;
            float v[8];
            tc::tmem_ld8(dtm + ((uint32_t)(32 * qd) << 16) + (uint32_t)(kTcColD + buf * 64 + 8 * p), v);
            if (i < kNC && p < sb.count) {
                float* o = ell + (size_t)tgt[sb.begin + p] * kBoxStride + 6 * i;
                if ((i & 1) == 0) {
                    red_add_v4(o, v[0], v[1], v[2], v[3]);
                    red_add_v2(o + 4, v[4], v[5]);
                } else {
                    red_add_v2(o, v[0], v[1]);
                    red_add_v4(o + 2, v[2], v[3], v[4], v[5]);
                }
            }
        }
    };
    auto epilogue = [&](int buf, const Sub& sb) { wait_mma(buf); drain(buf, sb); };
    // operator hi/lo rows into TMEM: warp w writes lanes of quarter w % 4, columns half (w / 4)
    auto load_a = [&](int off) {
        const int qd = warp & 3, hf = warp >> 2;
        const int i = 32 * qd + lane;
        const float* rowh = aimg + ((size_t)off * 2 * 128 + i) * 128 + 64 * hf;
        const float* rowl = rowh + 128 * 128;
        const uint32_t ta = dtm + ((uint32_t)(32 * qd) << 16) + 64 * hf;
        float v[32];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float4 q = __ldg(reinterpret_cast<const float4*>(rowh + 32 * c) + j);
                v[4 * j] = q.x; v[4 * j + 1] = q.y; v[4 * j + 2] = q.z; v[4 * j + 3] = q.w;
            }
            tc::tmem_st32(ta + kTcColAh + 32 * c, v);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float4 q = __ldg(reinterpret_cast<const float4*>(rowl + 32 * c) + j);
                v[4 * j] = q.x; v[4 * j + 1] = q.y; v[4 * j + 2] = q.z; v[4 * j + 3] = q.w;
            }
            tc::tmem_st32(ta + kTcColAl + 32 * c, v);
        }
        tc::tmem_st_wait();
    };

    int blk = blockIdx.x, ti = blk * kTcR, half = 0;
    auto valid = [&]() { return blk * kTcR < ntiles && ti < min(ntiles, (blk + 1) * kTcR); };
    auto advance = [&]() {
        if ((half + 1) * kTcP < tiles[ti].z) { ++half; return; }
        half = 0;
        ++ti;
        if (ti >= min(ntiles, (blk + 1) * kTcR)) { blk += gridDim.x; ti = blk * kTcR; }
    };
    if (valid()) {
        Sub cur = sub_at(ti, half);
        load_a(cur.off);
        cur_off = cur.off;
        gather(cur, 0);
        int t = 0;
        bool have_prev = false;
        Sub prev{};
        for (;;) {
            const int buf = t & 1;
            cp_async_wait_all();
            tc::fence_proxy_async();
            tc::fence_before();
            __syncthreads();
            tc::fence_after();
            if (tid == 0) {
                float* Bh = Bbase + (size_t)buf * 2 * (kTcBBytes / 4);
                const uint32_t b0 = tc::smem_u32(Bh), bl0 = tc::smem_u32(Bh + kTcBBytes / 4);
                const uint32_t dst = dtm + kTcColD + (uint32_t)(buf * 64);
#pragma unroll
                for (int s2 = 0; s2 < 16; ++s2) {
                    const uint64_t bh = tc::smem_desc(b0 + s2 * 2 * lboB, lboB, 128);
                    const uint64_t bl = tc::smem_desc(bl0 + s2 * 2 * lboB, lboB, 128);
                    tc::mma_tf32_ts(dst, dtm + kTcColAl + 8 * s2, bh, idesc, s2 > 0);
                    tc::mma_tf32_ts(dst, dtm + kTcColAh + 8 * s2, bl, idesc, 1);
                    tc::mma_tf32_ts(dst, dtm + kTcColAh + 8 * s2, bh, idesc, 1);
                }
                tc::commit(&bar[buf]);
            }
            // MMA(t-1) done -> its B buffer (buf^1) is free: issue the gather of t+1 first,
            // then drain the accumulator of t-1 while the copies and MMA(t) are in flight
            const bool had_prev = have_prev;
            const Sub pv = prev;
            if (had_prev) wait_mma(buf ^ 1);
            prev = cur;
            have_prev = true;
            advance();
            const bool more = valid();
            Sub nxt{};
            bool switch_a = false;
            if (more) {
                nxt = sub_at(ti, half);
                switch_a = nxt.off != cur_off;
                if (!switch_a) gather(nxt, buf ^ 1);
            }
            if (had_prev) drain(buf ^ 1, pv);
            if (!more) break;
            if (switch_a) {
                // the operator is about to change: wait for MMA(t) and drain it first
                epilogue(buf, cur);
                have_prev = false;
                tc::fence_before();
                __syncthreads();
                tc::fence_after();
                load_a(nxt.off);
                cur_off = nxt.off;
                gather(nxt, buf ^ 1);
            }
            cur = nxt;
            ++t;
        }
        if (have_prev) epilogue(t & 1, prev);
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<512>(tbase);
}

// ------------------------------------------------------------------ P2L (X list)
// One CTA per target box b; the panels of all leaves in X(b) are flattened and
// processed 128 at a time (one panel per thread computes It and its charges
// into shared memory, then 128 threads reduce the 726 outputs).
constexpr int kXWin = 64;                 // X leaves per window
constexpr int kP2LChunk = 128;
constexpr int kP2LSmem = kP2LChunk * (kNC + 6) * 4;

__device__ __forceinline__ int find_seg(const int* off, int n, int j)
{
    int lo = 0, hi = n - 1;  // largest i with off[i] <= j
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (off[mid] <= j) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__global__ void __launch_bounds__(128) k_p2l(const int32_t* __restrict__ xt, const int64_t* __restrict__ xptr,
                                             const int32_t* __restrict__ xsrc, const int32_t* __restrict__ level,
                                             const int32_t* __restrict__ ix, const int32_t* __restrict__ iy,
                                             const int32_t* __restrict__ iz, const int32_t* __restrict__ pb,
                                             const int32_t* __restrict__ pe, const float4* __restrict__ loc,
                                             const float* __restrict__ xq, float* __restrict__ ell)
{
    extern __shared__ __align__(16) float psm[];
    float* H = psm;                        // [128][121]
    float* Q = psm + kP2LChunk * kNC;      // [128][6]
    __shared__ int Xoff[kXWin + 1], Xid[kXWin];
    __shared__ float3 Xd[kXWin];
    const int b = xt[blockIdx.x];
    const int lb = level[b];
    const float3 cb = box_center(lb, ix[b], iy[b], iz[b]);
    const float inv_s = ldexpf(1.f, lb);
    float acc[6] = {0, 0, 0, 0, 0, 0};
    for (int64_t x0 = xptr[b]; x0 < xptr[b + 1]; x0 += kXWin) {
        const int nx = (int)min((int64_t)kXWin, xptr[b + 1] - x0);
        __syncthreads();
        if (threadIdx.x < nx) {
            const int L = xsrc[x0 + threadIdx.x];
            Xid[threadIdx.x] = L;
            const float3 cL = box_center(level[L], ix[L], iy[L], iz[L]);
            Xd[threadIdx.x] = make_float3(cL.x - cb.x, cL.y - cb.y, cL.z - cb.z);
        }
        if (threadIdx.x == 0) {
            int o = 0;
            for (int i = 0; i < nx; ++i) { Xoff[i] = o; const int L = xsrc[x0 + i]; o += pe[L] - pb[L]; }
            Xoff[nx] = o;
        }
        __syncthreads();
        const int total = Xoff[nx];
        for (int c0 = 0; c0 < total; c0 += kP2LChunk) {
            const int cn = min(kP2LChunk, total - c0);
            if (threadIdx.x < cn) {
                const int j = c0 + threadIdx.x;
                const int li = find_seg(Xoff, nx, j);
                const int i = pb[Xid[li]] + (j - Xoff[li]);
                const float3 d = Xd[li];
                const float4 p = loc[i];
                float h[kNC];
                irregular_harmonics<kP>((p.x + d.x) * inv_s, (p.y + d.y) * inv_s, (p.z + d.z) * inv_s, c_tab, h);
                float* Hr = H + threadIdx.x * kNC;
#pragma unroll
                for (int k = 0; k < kNC; ++k) Hr[k] = (degree_of(k) * degree_of(k) == k) ? h[k] : 2.f * h[k];
#pragma unroll
                for (int r = 0; r < 6; ++r) Q[threadIdx.x * 6 + r] = xq[8 * (int64_t)i + r];
            }
            __syncthreads();
#pragma unroll
            for (int jj = 0; jj < 6; ++jj) {
                const int o = threadIdx.x + 128 * jj;
                if (o < kNC * 6) {
                    const int k = o / 6, r = o % 6;
                    float a = acc[jj];
                    for (int p = 0; p < cn; ++p) a = fmaf(H[p * kNC + k], Q[p * 6 + r], a);
                    acc[jj] = a;
                }
            }
            __syncthreads();
        }
    }
    float* out = ell + (size_t)b * kBoxStride;
#pragma unroll
    for (int jj = 0; jj < 6; ++jj) {
        const int o = threadIdx.x + 128 * jj;
        if (o < kNC * 6) out[o] += acc[jj];
    }
}

// ------------------------------------------------------------------ near-field SpMV
// y = N x for the 6 real RHS (N: FP32 CSR of the near correction and the self
// terms).  HBM-bound: 8 B per nonzero (col + val) + the gathered charges
// (L2-resident) + 24 B of y per row.  8 lanes per row, 4 rows per warp; each
// lane issues 4 independent (col, val) loads before their 4 gathers (memory-
// level parallelism), shuffle reduction over the 8 lanes.
__global__ void __launch_bounds__(256) k_near_spmv(int64_t n, int64_t r0, const int64_t* __restrict__ ptr,
                                                   const int32_t* __restrict__ col, const float* __restrict__ val,
                                                   const float* __restrict__ xq, float2* __restrict__ y)
{
    // rows r0 .. r0+n-1 (owned range); y local [3][n]
    const int64_t lrow = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 3;
    const int64_t row = r0 + lrow;
    const int lane = threadIdx.x & 7;
    float a[6] = {0, 0, 0, 0, 0, 0};
    if (lrow < n) {
        const int64_t e = ptr[row + 1];
#pragma unroll 4
        for (int64_t j = ptr[row] + lane; j < e; j += 8) {
            const float v = __ldcs(val + j);
            const int64_t c = __ldcs(col + j);
            const float4 q0 = reinterpret_cast<const float4*>(xq + 8 * c)[0];
            const float2 q1 = reinterpret_cast<const float2*>(xq + 8 * c)[2];
            a[0] = fmaf(v, q0.x, a[0]); a[1] = fmaf(v, q0.y, a[1]); a[2] = fmaf(v, q0.z, a[2]);
            a[3] = fmaf(v, q0.w, a[3]); a[4] = fmaf(v, q1.x, a[4]); a[5] = fmaf(v, q1.y, a[5]);
        }
    }
#pragma unroll
    for (int r = 0; r < 6; ++r) {
        a[r] += __shfl_xor_sync(0xffffffffu, a[r], 1);
        a[r] += __shfl_xor_sync(0xffffffffu, a[r], 2);
        a[r] += __shfl_xor_sync(0xffffffffu, a[r], 4);
    }
    if (lrow < n && lane < 3) y[lane * n + lrow] = make_float2(a[2 * lane], a[2 * lane + 1]);
}

// ------------------------------------------------------------------ P2P
// One CTA (128 threads) per target leaf; targets in passes of <= 128*kTPT.
// Each thread owns kTPT consecutive targets (register blocking: one shared-
// memory source load feeds kTPT pairs); with NG = ceil(T/kTPT) target groups
// the CTA is split into S = 128/NG source groups.  U-list source leaves are
// flattened (warp-parallel prefix sum), staged 512 panels at a time in shared
// memory re-based to the target leaf centre (W units), and split over the
// groups.  Only the target's own leaf needs the r = 0 (self) guard.
// y += (1/W) sum_{l != k} x_l / r_kl.
constexpr int kUWin = 64;
constexpr int kSrcChunk = 512;
constexpr int kTPT = 8;

template <bool kSelf>
__device__ __forceinline__ void p2p_range(int j0, int j1, int S, const float4* __restrict__ Sp,
                                          const float4 (*__restrict__ Sq)[2], const float* tx, const float* ty,
                                          const float* tz, float (*far)[6])
{
#pragma unroll 2
    for (int j = j0; j < j1; j += S) {
        const float4 sp = Sp[j];
        const float4 q0 = Sq[j][0], q1 = Sq[j][1];
#pragma unroll
        for (int q = 0; q < kTPT; ++q) {
            const float dx = tx[q] - sp.x, dy = ty[q] - sp.y, dz = tz[q] - sp.z;
            const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
            float ri = rsqrtf(r2);
            if (kSelf) ri = r2 > 0.f ? ri : 0.f;
            far[q][0] = fmaf(q0.x, ri, far[q][0]); far[q][1] = fmaf(q0.y, ri, far[q][1]);
            far[q][2] = fmaf(q0.z, ri, far[q][2]); far[q][3] = fmaf(q0.w, ri, far[q][3]);
            far[q][4] = fmaf(q1.x, ri, far[q][4]); far[q][5] = fmaf(q1.y, ri, far[q][5]);
        }
    }
}

__device__ __forceinline__ int first_in_class(int lo, int sg, int S)
{
    // smallest j >= lo with j % S == sg
    const int r = lo % S;
    return lo + ((sg - r + S) % S);
}

__global__ void __launch_bounds__(128) k_p2p(
    const int32_t* __restrict__ leaves, const int32_t* __restrict__ level, const int32_t* __restrict__ ix,
    const int32_t* __restrict__ iy, const int32_t* __restrict__ iz, const int32_t* __restrict__ pb,
    const int32_t* __restrict__ pe, const int64_t* __restrict__ uptr, const int32_t* __restrict__ usrc,
    const float4* __restrict__ loc, const float* __restrict__ xq, float invW, int accumulate, int64_t n,
    int64_t p0, float2* __restrict__ y)
{
    // n, p0: owned panel range [p0, p0+n), y local [3][n]
    // the source staging buffers and the final reduction share one buffer
    constexpr int kStageF = kSrcChunk * 12, kRedF = 128 * (kTPT * 6 + 1);
    __shared__ __align__(16) float smraw[kStageF > kRedF ? kStageF : kRedF];
    float4* Sp = reinterpret_cast<float4*>(smraw);
    float4(*Sq)[2] = reinterpret_cast<float4(*)[2]>(smraw + 4 * kSrcChunk);
    float(*Red)[kTPT * 6 + 1] = reinterpret_cast<float(*)[kTPT * 6 + 1]>(smraw);
    __shared__ int Uoff[kUWin + 1], Uid[kUWin], Upb[kUWin];
    __shared__ float3 Ud[kUWin];
    __shared__ int wsum[2];
    const int b = leaves[blockIdx.x];
    const float3 cb = box_center(level[b], ix[b], iy[b], iz[b]);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int t0 = pb[b]; t0 < pe[b]; t0 += 128 * kTPT) {
        const int T = min(128 * kTPT, pe[b] - t0);
        const int NG = (T + kTPT - 1) / kTPT;
        const int S = max(1, 128 / NG);
        const int tg = tid % NG, sg = tid / NG;
        const bool act = sg < S;
        float tx[kTPT], ty[kTPT], tz[kTPT];
        float far[kTPT][6];
#pragma unroll
        for (int q = 0; q < kTPT; ++q) {
            const int ti = tg * kTPT + q;
            float4 p = make_float4(1e30f, 1e30f, 1e30f, 0.f);  // padding target: far away, discarded
            if (act && ti < T) p = loc[t0 + ti];
            tx[q] = p.x; ty[q] = p.y; tz[q] = p.z;
#pragma unroll
            for (int r = 0; r < 6; ++r) far[q][r] = 0.f;
        }
        for (int64_t u0 = uptr[b]; u0 < uptr[b + 1]; u0 += kUWin) {
            const int nu = (int)min((int64_t)kUWin, uptr[b + 1] - u0);
            __syncthreads();
            // window setup: ids, centre shifts and an exclusive prefix of the leaf sizes (2 warps)
            int sz = 0;
            if (tid < kUWin) {
                if (tid < nu) {
                    const int s = usrc[u0 + tid];
                    Uid[tid] = s;
                    Upb[tid] = pb[s];
                    sz = pe[s] - pb[s];
                    const float3 cs = box_center(level[s], ix[s], iy[s], iz[s]);
                    Ud[tid] = make_float3(cs.x - cb.x, cs.y - cb.y, cs.z - cb.z);
                }
                int inc = sz;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += v;
                }
                if (lane == 31) wsum[warp] = inc;
                Uoff[tid + 1] = inc;  // provisional (warp-local)
            }
            __syncthreads();
            if (tid >= 32 && tid < kUWin) Uoff[tid + 1] += wsum[0];
            if (tid == 0) Uoff[0] = 0;
            __syncthreads();
            const int total = Uoff[nu];
            // the target leaf's own panels in the flattened window (needs the r = 0 guard)
            int self_lo = 0, self_hi = 0;
            for (int i = 0; i < nu; ++i)
                if (Uid[i] == b) { self_lo = Uoff[i]; self_hi = Uoff[i + 1]; }
            for (int s0 = 0; s0 < total; s0 += kSrcChunk) {
                const int sn = min(kSrcChunk, total - s0);
                if (s0 > 0) __syncthreads();
                for (int j = tid; j < sn; j += 128) {
                    const int f = s0 + j;
                    const int li = find_seg(Uoff, nu, f);
                    const int i = Upb[li] + (f - Uoff[li]);
                    const float3 d = Ud[li];
                    const float4 p = loc[i];
                    Sp[j] = make_float4(p.x + d.x, p.y + d.y, p.z + d.z, 0.f);
                    const float4* q = reinterpret_cast<const float4*>(xq + 8 * (int64_t)i);
                    Sq[j][0] = q[0];
                    Sq[j][1] = q[1];
                }
                __syncthreads();
                if (act) {
                    const int a0 = max(0, min(sn, self_lo - s0)), a1 = max(0, min(sn, self_hi - s0));
                    p2p_range<false>(first_in_class(0, sg, S), a0, S, Sp, Sq, tx, ty, tz, far);
                    p2p_range<true>(first_in_class(a0, sg, S), a1, S, Sp, Sq, tx, ty, tz, far);
                    p2p_range<false>(first_in_class(a1, sg, S), sn, S, Sp, Sq, tx, ty, tz, far);
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kTPT; ++q)
#pragma unroll
            for (int r = 0; r < 6; ++r) Red[tid][q * 6 + r] = far[q][r];
        __syncthreads();
        // reduce over the S source groups: thread handles target index ti = tid, tid + 128, ...
        for (int ti = tid; ti < T; ti += 128) {
            const int g0 = ti / kTPT, q = ti % kTPT;
            float tot[6];
#pragma unroll
            for (int r = 0; r < 6; ++r) {
                float f = 0.f;
                for (int gg = 0; gg < S; ++gg) f += Red[g0 + gg * NG][q * 6 + r];
                tot[r] = f * invW;
            }
            const int64_t k = t0 + ti - p0;
            if (accumulate) {
                const float2 a = y[k], c = y[n + k], d = y[2 * n + k];
                tot[0] += a.x; tot[1] += a.y; tot[2] += c.x; tot[3] += c.y; tot[4] += d.x; tot[5] += d.y;
            }
            y[k] = make_float2(tot[0], tot[1]);
            y[n + k] = make_float2(tot[2], tot[3]);
            y[2 * n + k] = make_float2(tot[4], tot[5]);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ L2P + M2P
// One thread per target panel: y += (1/W) [ (1/s_b) sum ell_b Rt(u) + sum_{w in W(b)} (1/s_w) sum c mu_w It(u_w) ].
__global__ void __launch_bounds__(128) k_l2p_m2p(int64_t n, int64_t p0, const int32_t* __restrict__ panel_leaf,
                                                 const int32_t* __restrict__ level, const int32_t* __restrict__ ix,
                                                 const int32_t* __restrict__ iy, const int32_t* __restrict__ iz,
                                                 const int64_t* __restrict__ wptr, const int32_t* __restrict__ wsrc,
                                                 const float4* __restrict__ loc, const float* __restrict__ mu,
                                                 const float* __restrict__ ell, float invW, float2* __restrict__ y)
{
    const int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // local index, panel p0 + li
    if (li >= n) return;
    const int64_t i = p0 + li;
    const int b = panel_leaf[i];
    const int lb = level[b];
    const float3 cb = box_center(lb, ix[b], iy[b], iz[b]);
    const float inv_sb = ldexpf(1.f, lb);
    const float4 tp = loc[i];
    float far[6] = {0, 0, 0, 0, 0, 0};
    {
        float h[kNC];
        regular_harmonics<kP>(tp.x * inv_sb, tp.y * inv_sb, tp.z * inv_sb, c_tab, h);
        const float2* L = reinterpret_cast<const float2*>(ell + (size_t)b * kBoxStride);
#pragma unroll
        for (int k = 0; k < kNC; ++k) {
            const float2 l0 = __ldg(L + 3 * k), l1 = __ldg(L + 3 * k + 1), l2 = __ldg(L + 3 * k + 2);
            far[0] = fmaf(l0.x, h[k], far[0]); far[1] = fmaf(l0.y, h[k], far[1]);
            far[2] = fmaf(l1.x, h[k], far[2]); far[3] = fmaf(l1.y, h[k], far[3]);
            far[4] = fmaf(l2.x, h[k], far[4]); far[5] = fmaf(l2.y, h[k], far[5]);
        }
#pragma unroll
        for (int r = 0; r < 6; ++r) far[r] *= inv_sb;
    }
    for (int64_t wj = wptr[b]; wj < wptr[b + 1]; ++wj) {
        const int w = wsrc[wj];
        const int lw = level[w];
        const float3 cw = box_center(lw, ix[w], iy[w], iz[w]);
        const float inv_sw = ldexpf(1.f, lw);
        float h[kNC];
        irregular_harmonics<kP>((tp.x + cb.x - cw.x) * inv_sw, (tp.y + cb.y - cw.y) * inv_sw,
                                (tp.z + cb.z - cw.z) * inv_sw, c_tab, h);
        const float2* M = reinterpret_cast<const float2*>(mu + (size_t)w * kBoxStride);
        float a[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int k = 0; k < kNC; ++k) {
            const float hk = (degree_of(k) * degree_of(k) == k) ? h[k] : 2.f * h[k];
            const float2 m0 = __ldg(M + 3 * k), m1 = __ldg(M + 3 * k + 1), m2 = __ldg(M + 3 * k + 2);
            a[0] = fmaf(m0.x, hk, a[0]); a[1] = fmaf(m0.y, hk, a[1]);
            a[2] = fmaf(m1.x, hk, a[2]); a[3] = fmaf(m1.y, hk, a[3]);
            a[4] = fmaf(m2.x, hk, a[4]); a[5] = fmaf(m2.y, hk, a[5]);
        }
#pragma unroll
        for (int r = 0; r < 6; ++r) far[r] = fmaf(a[r], inv_sw, far[r]);
    }
    float2 a = y[li], c = y[n + li], d = y[2 * n + li];
    y[li] = make_float2(fmaf(far[0], invW, a.x), fmaf(far[1], invW, a.y));
    y[n + li] = make_float2(fmaf(far[2], invW, c.x), fmaf(far[3], invW, c.y));
    y[2 * n + li] = make_float2(fmaf(far[4], invW, d.x), fmaf(far[5], invW, d.y));
}

__global__ void k_permute(int64_t n, int nvec, const int32_t* __restrict__ idx, const float2* __restrict__ in,
                          float2* __restrict__ out)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t s = idx[i];
    for (int v = 0; v < nvec; ++v) out[(int64_t)v * n + i] = in[(int64_t)v * n + s];
}

inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

// Operators are built once per process in FP64 on the host.
const HostOperators& host_ops()
{
    static HostOperators ops;
    static std::once_flag once;
    std::call_once(once, [] { build_operators(ops); });
    return ops;
}

void upload_padded(DBuf<float>& dst, const std::vector<double>& src, int nmat)
{
    std::vector<float> h((size_t)nmat * kNC * kNCP, 0.f);
    for (int m = 0; m < nmat; ++m)
        for (int i = 0; i < kNC; ++i)
            for (int k = 0; k < kNC; ++k)
                h[(size_t)m * kNC * kNCP + (size_t)k * kNCP + i] = (float)src[(size_t)m * kNC * kNC + (size_t)i * kNC + k];
    dst.alloc(h.size());
    XRL_CUDA(cudaMemcpy(dst.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
}

float tf32_host(float x)
{
    uint32_t u;
    std::memcpy(&u, &x, 4);
    u = (u + 0x1000u) & 0xFFFFE000u;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
}

// M2L operator images for k_m2l_tc: per offset, the hi and lo TF32 parts of
// T[i][k] (i, k < 121, zero padded to 128), row-major [part][i][k] (one TMEM
// lane per row i).
void upload_tc_images(DBuf<float>& dst, const std::vector<double>& src)
{
    const size_t img = 128 * 128;
    std::vector<float> h((size_t)kNM2L * 2 * img, 0.f);
    for (int m = 0; m < kNM2L; ++m)
        for (int i = 0; i < kNC; ++i)
            for (int k = 0; k < kNC; ++k) {
                const float a = (float)src[(size_t)m * kNC * kNC + (size_t)i * kNC + k];
                const float hi = tf32_host(a);
                h[(size_t)m * 2 * img + (size_t)i * 128 + k] = hi;
                h[(size_t)m * 2 * img + img + (size_t)i * 128 + k] = a - hi;
            }
    dst.alloc(h.size());
    XRL_CUDA(cudaMemcpy(dst.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
}

}  // namespace

namespace xrl {

void upload_constants(xrl_ctx ctx)
{
    RecTables<float> tab;
    fill_recurrence_tables(tab);
    XRL_CUDA(cudaMemcpyToSymbol(c_tab, &tab, sizeof(tab)));
    const HostOperators& ops = host_ops();
    upload_padded(ctx->ops.m2m, ops.m2m, 8);
    upload_padded(ctx->ops.l2l, ops.l2l, 8);
    upload_padded(ctx->ops.m2l, ops.m2l, kNM2L);
    upload_tc_images(ctx->ops.m2l_tc, ops.m2l);
    XRL_CUDA(cudaFuncSetAttribute(k_m2l_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem));
    XRL_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device));
    const char* e = getenv("XRL_M2L_SIMT");  // SIMT FP32 M2L (ablation); default tcgen05 3xTF32
    ctx->m2l_simt = e && e[0] == '1';
    for (int i = 0; i < 343; ++i) ctx->ops.m2l_index[i] = ops.m2l_index[i];
    XRL_CUDA(cudaFuncSetAttribute(k_m2l, cudaFuncAttributeMaxDynamicSharedMemorySize, kM2LSmem));
    XRL_CUDA(cudaFuncSetAttribute(k_p2l, cudaFuncAttributeMaxDynamicSharedMemorySize, kP2LSmem));
}

}  // namespace xrl

// x: full (gathered) triple [3][n]; y: owned slice [3][n_local] of panels [p0, p1).
static void mvm_triple(xrl_tree t, xrl_near nr, const float2* x, float2* y, uint32_t flags)
{
    xrl_ctx ctx = t->ctx;
    cudaStream_t st = ctx->stream, side = ctx->side;
    const int64_t n = t->n;
    const int64_t nl = t->p1 - t->p0, p0 = t->p0;
    const bool do_far = flags != XRL_MVM_NEAR_ONLY;
    const bool do_near = flags != XRL_MVM_FAR_ONLY;
    const float invW = (float)(1.0 / t->W);
    cudaEvent_t ev;

    phase_begin(ctx, PH_PACK, &ev, st);
    k_pack<<<nblk(n, 256), 256, 0, st>>>(n, x, t->xq.p);
    XRL_LAUNCH_CHECK();
    ctx->launches += 1;
    phase_end(ctx, PH_PACK, ev, st);

    // fork: near SpMV and P2P depend only on the packed charges -> side stream,
    // overlapping the upward pass and the M2L on the main stream.
    XRL_CUDA(cudaEventRecord(ctx->ev_fork, st));
    XRL_CUDA(cudaStreamWaitEvent(side, ctx->ev_fork, 0));
    if (do_near) {
        phase_begin(ctx, PH_NEAR, &ev, side);
        if (nl > 0) k_near_spmv<<<nblk(8 * nl, 256), 256, 0, side>>>(nl, p0, nr->row_ptr.p, nr->col.p, nr->val.p, t->xq.p, y);
        XRL_LAUNCH_CHECK();
        ctx->launches += 1;
        phase_end(ctx, PH_NEAR, ev, side);
    }
    if (do_far) {
        phase_begin(ctx, PH_P2P, &ev, side);
        if (t->n_own_leaves > 0)
            k_p2p<<<t->n_own_leaves, 128, 0, side>>>(t->own_leaves.p, t->blevel.p, t->bix.p, t->biy.p, t->biz.p,
                                                     t->bpb.p, t->bpe.p, t->u_ptr.p, t->u_src.p, t->loc.p, t->xq.p,
                                                     invW, do_near ? 1 : 0, nl, p0, y);
        XRL_LAUNCH_CHECK();
        ctx->launches += 1;
        phase_end(ctx, PH_P2P, ev, side);
    }
    XRL_CUDA(cudaEventRecord(ctx->ev_join, side));

    if (do_far && t->nlevel > 1) {
        phase_begin(ctx, PH_P2M, &ev, st);
        k_p2m<<<t->nleaf, 128, 0, st>>>(t->leaves.p, t->bpb.p, t->bpe.p, t->blevel.p, t->loc.p, t->xq.p, t->mu.p);
        XRL_LAUNCH_CHECK();
        ctx->launches += 1;
        phase_end(ctx, PH_P2M, ev, st);

        phase_begin(ctx, PH_M2M, &ev, st);
        for (int l = t->nlevel - 2; l >= 2; --l) {
            const int np = t->par_start[l + 1] - t->par_start[l];
            if (np == 0) continue;
            k_m2m<<<np, 128, 0, st>>>(t->parents.p + t->par_start[l], t->bchild.p, t->bnchild.p, t->bix.p, t->biy.p,
                                      t->biz.p, ctx->ops.m2m.p, t->mu.p);
            XRL_LAUNCH_CHECK();
            ctx->launches += 1;
        }
        phase_end(ctx, PH_M2M, ev, st);

        phase_begin(ctx, PH_M2L, &ev, st);
        XRL_CUDA(cudaMemsetAsync(t->ell.p, 0, t->ell.bytes(), st));
        if (t->n_m2l_tiles > 0 && ctx->m2l_simt) {
            k_m2l<<<t->n_m2l_tiles, 256, kM2LSmem, st>>>(t->m2l_tiles.p, t->m2l_tgt.p, t->m2l_srcb.p, ctx->ops.m2l.p,
                                                         t->mu.p, t->ell.p);
            XRL_LAUNCH_CHECK();
            ctx->launches += 1;
        } else if (t->n_m2l_tiles > 0) {
            const int nblocks = (t->n_m2l_tiles + kTcR - 1) / kTcR;
            const int grid = std::min(ctx->num_sms, nblocks);
            if (t->mu_img.n < (size_t)t->nbox * kImgFloats) t->mu_img.alloc((size_t)t->nbox * kImgFloats);
            k_mu_img<<<nblk((int64_t)t->nbox * 1024, 256), 256, 0, st>>>(t->nbox, t->mu.p, t->mu_img.p);
            XRL_LAUNCH_CHECK();
            ctx->launches += 1;
            k_m2l_tc<<<grid, kTcThreads, kTcSmem, st>>>(t->m2l_tiles.p, t->n_m2l_tiles, t->m2l_tgt.p, t->m2l_srcb.p,
                                                        ctx->ops.m2l_tc.p, t->mu_img.p, t->ell.p);
            XRL_LAUNCH_CHECK();
            ctx->launches += 1;
        }
        phase_end(ctx, PH_M2L, ev, st);

        phase_begin(ctx, PH_P2L, &ev, st);
        if (t->n_x_targets > 0) {
            k_p2l<<<t->n_x_targets, 128, kP2LSmem, st>>>(t->x_targets.p, t->x_ptr.p, t->x_src.p, t->blevel.p, t->bix.p,
                                                         t->biy.p, t->biz.p, t->bpb.p, t->bpe.p, t->loc.p, t->xq.p,
                                                         t->ell.p);
            XRL_LAUNCH_CHECK();
            ctx->launches += 1;
        }
        phase_end(ctx, PH_P2L, ev, st);

        phase_begin(ctx, PH_L2L, &ev, st);
        for (int l = 3; l < t->nlevel; ++l) {
            const int b0 = t->l2l_start[l], nb = t->l2l_start[l + 1] - b0;
            if (nb == 0) continue;
            k_l2l<<<nb, 128, 0, st>>>(t->l2l_boxes.p + b0, t->bparent.p, t->bix.p, t->biy.p, t->biz.p, ctx->ops.l2l.p,
                                      t->ell.p);
            XRL_LAUNCH_CHECK();
            ctx->launches += 1;
        }
        phase_end(ctx, PH_L2L, ev, st);
    }
    // join, then the local-expansion / W-list evaluation completes y
    XRL_CUDA(cudaStreamWaitEvent(st, ctx->ev_join, 0));
    if (do_far && t->nlevel > 1 && nl > 0) {
        phase_begin(ctx, PH_L2P, &ev, st);
        k_l2p_m2p<<<nblk(nl, 128), 128, 0, st>>>(nl, p0, t->panel_leaf.p, t->blevel.p, t->bix.p, t->biy.p, t->biz.p,
                                                t->w_ptr.p, t->w_src.p, t->loc.p, t->mu.p, t->ell.p, invW, y);
        XRL_LAUNCH_CHECK();
        ctx->launches += 1;
        phase_end(ctx, PH_L2P, ev, st);
    }
}

extern "C" {

xrl_status xrl_mvm(xrl_tree t, xrl_near nr, const void* x, void* y, int32_t nvec, uint32_t flags)
{
    if (!t || !nr || !x || !y) { set_error("xrl_mvm: null argument"); return XRL_EINVAL; }
    if (nr->tree != t) { set_error("xrl_mvm: near handle built from another tree"); return XRL_EPROVENANCE; }
    if (nvec < 3 || nvec % 3) { set_error("xrl_mvm: nvec=%d must be a positive multiple of 3", nvec); return XRL_EDIM; }
    if (x == y) { set_error("xrl_mvm: x and y alias"); return XRL_EINVAL; }
    if (flags > XRL_MVM_FAR_ONLY) { set_error("xrl_mvm: bad flags"); return XRL_EINVAL; }
    if (((uintptr_t)x | (uintptr_t)y) & 15) { set_error("xrl_mvm: vectors must be 16-byte aligned"); return XRL_EINVAL; }
    try {
        XRL_CUDA(cudaSetDevice(t->ctx->device));
        const int64_t nl = t->p1 - t->p0;
        if (t->part_world == 1) {
            for (int v = 0; v < nvec; v += 3)
                mvm_triple(t, nr, (const float2*)x + (size_t)v * t->n, (float2*)y + (size_t)v * t->n, flags);
            return XRL_OK;
        }
        if (t->ctx->world == 1) {
            set_error("xrl_mvm: virtual partition (part_world > 1 on a single-rank context) needs xrl_mvm_gathered");
            return XRL_EUNSUPPORTED;
        }
        if (t->xfull.n < (size_t)3 * t->n) t->xfull.alloc((size_t)3 * t->n);
        for (int v = 0; v < nvec; v += 3) {
            // gather the owned slices of the 3 components into the full vectors (NCCL over NVLink)
            xrl_status s = gather_slices(t, (const float2*)x + (size_t)v * nl, t->xfull.p);
            if (s) return s;
            mvm_triple(t, nr, t->xfull.p, (float2*)y + (size_t)v * nl, flags);
        }
        return XRL_OK;
    } catch (const CudaError& e) {
        return e.code;
    }
}

xrl_status xrl_mvm_gathered(xrl_tree t, xrl_near nr, const void* x_full, void* y, int32_t nvec, uint32_t flags)
{
    if (!t || !nr || !x_full || !y) { set_error("xrl_mvm_gathered: null argument"); return XRL_EINVAL; }
    if (nr->tree != t) { set_error("xrl_mvm_gathered: near handle built from another tree"); return XRL_EPROVENANCE; }
    if (nvec < 3 || nvec % 3) { set_error("xrl_mvm_gathered: nvec=%d must be a positive multiple of 3", nvec); return XRL_EDIM; }
    if (x_full == y) { set_error("xrl_mvm_gathered: x and y alias"); return XRL_EINVAL; }
    if (flags > XRL_MVM_FAR_ONLY) { set_error("xrl_mvm_gathered: bad flags"); return XRL_EINVAL; }
    try {
        XRL_CUDA(cudaSetDevice(t->ctx->device));
        const int64_t nl = t->p1 - t->p0;
        for (int v = 0; v < nvec; v += 3)
            mvm_triple(t, nr, (const float2*)x_full + (size_t)v * t->n, (float2*)y + (size_t)v * nl, flags);
        return XRL_OK;
    } catch (const CudaError& e) {
        return e.code;
    }
}

xrl_status xrl_to_library_order(xrl_tree t, const void* x_user, void* x_lib, int32_t nvec)
{
    if (!t || !x_user || !x_lib || nvec < 1) { set_error("xrl_to_library_order: bad argument"); return XRL_EINVAL; }
    try {
        XRL_CUDA(cudaSetDevice(t->ctx->device));
        k_permute<<<nblk(t->n, 256), 256, 0, t->ctx->stream>>>(t->n, nvec, t->perm.p, (const float2*)x_user,
                                                                (float2*)x_lib);
        XRL_LAUNCH_CHECK();
        t->ctx->launches += 1;
        return XRL_OK;
    } catch (const CudaError& e) {
        return e.code;
    }
}

xrl_status xrl_from_library_order(xrl_tree t, const void* x_lib, void* x_user, int32_t nvec)
{
    if (!t || !x_user || !x_lib || nvec < 1) { set_error("xrl_from_library_order: bad argument"); return XRL_EINVAL; }
    try {
        XRL_CUDA(cudaSetDevice(t->ctx->device));
        k_permute<<<nblk(t->n, 256), 256, 0, t->ctx->stream>>>(t->n, nvec, t->iperm.p, (const float2*)x_lib,
                                                                (float2*)x_user);
        XRL_LAUNCH_CHECK();
        t->ctx->launches += 1;
        return XRL_OK;
    } catch (const CudaError& e) {
        return e.code;
    }
}

xrl_status xrl_mvm_host(xrl_tree t, xrl_near nr, const void* x_host, void* y_host, int32_t nvec, uint32_t flags)
{
    if (!t || !nr || !x_host || !y_host) { set_error("xrl_mvm_host: null argument"); return XRL_EINVAL; }
    if (nvec < 3 || nvec % 3) { set_error("xrl_mvm_host: nvec must be a positive multiple of 3"); return XRL_EDIM; }
    try {
        cudaStream_t st = t->ctx->stream;
        XRL_CUDA(cudaSetDevice(t->ctx->device));
        if (t->part_world > 1) {
            // multi-rank: host buffers are this rank's slice [nvec][n_local] in library order
            if (t->ctx->world == 1) { set_error("xrl_mvm_host: virtual partition not supported"); return XRL_EUNSUPPORTED; }
            const size_t cl = (size_t)nvec * (t->p1 - t->p0);
            if (t->xlib.n < cl) { t->xlib.alloc(cl); t->ylib.alloc(cl); }
            XRL_CUDA(cudaMemcpyAsync(t->xlib.p, x_host, cl * 8, cudaMemcpyHostToDevice, st));
            xrl_status s = xrl_mvm(t, nr, t->xlib.p, t->ylib.p, nvec, flags);
            if (s) return s;
            XRL_CUDA(cudaMemcpyAsync(y_host, t->ylib.p, cl * 8, cudaMemcpyDeviceToHost, st));
            XRL_CUDA(cudaStreamSynchronize(st));
            return XRL_OK;
        }
        const size_t cnt = (size_t)nvec * t->n;
        if (t->xtmp.n < cnt) { t->xtmp.alloc(cnt); t->ytmp.alloc(cnt); t->xlib.alloc(cnt); t->ylib.alloc(cnt); }
        float2 *xl = t->xlib.p, *yl = t->ylib.p;
        XRL_CUDA(cudaMemcpyAsync(t->xtmp.p, x_host, cnt * 8, cudaMemcpyHostToDevice, st));
        xrl_status s = xrl_to_library_order(t, t->xtmp.p, xl, nvec);
        if (s) return s;
        s = xrl_mvm(t, nr, xl, yl, nvec, flags);
        if (s) return s;
        s = xrl_from_library_order(t, yl, t->ytmp.p, nvec);
        if (s) return s;
        XRL_CUDA(cudaMemcpyAsync(y_host, t->ytmp.p, cnt * 8, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaStreamSynchronize(st));
        return XRL_OK;
    } catch (const CudaError& e) {
        return e.code;
    }
}

}  // extern "C"
