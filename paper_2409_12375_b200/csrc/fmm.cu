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
#include <mutex>

#include "xrl_internal.h"

using namespace xrl;

__constant__ RecTables<float> c_tab;

namespace {

constexpr int kTP = 32;          // pairs per M2L tile
constexpr int kBCols = kTP * 6;  // 192 columns of the M2L B tile

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

__global__ void __launch_bounds__(128) k_l2l(int b0, const int32_t* __restrict__ parent, const int32_t* __restrict__ ix,
                                             const int32_t* __restrict__ iy, const int32_t* __restrict__ iz,
                                             const float* __restrict__ op, float* __restrict__ ell)
{
    __shared__ float src[kBoxStride];
    const int b = b0 + blockIdx.x;
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
// Tile = (offset o, pairs [begin, begin+count)), count <= 32.
// C[128 x 192] = T_o[128 x 121] * B[121 x 192], B[k][p*6+r] = mu_src(p)[k][r].
// 256 threads: rg = tid % 16 owns rows rg*8..+7, pg = tid / 16 owns pairs 2pg, 2pg+1.
constexpr int kM2LSmem = (kNC * kNCP + kNC * kBCols) * 4;

__global__ void __launch_bounds__(256, 1) k_m2l(const int4* __restrict__ tiles, const int32_t* __restrict__ tgt,
                                                const int32_t* __restrict__ srcb, const float* __restrict__ ops,
                                                const float* __restrict__ mu, float* __restrict__ ell)
{
    extern __shared__ __align__(16) float sm[];
    float* Ts = sm;                    // [121][128]
    float* Bs = sm + kNC * kNCP;       // [121][192]
    const int4 tile = tiles[blockIdx.x];
    const int off = tile.x, begin = tile.y, count = tile.z;
    const int tid = threadIdx.x;
    {
        const float4* g = reinterpret_cast<const float4*>(ops + (size_t)off * kNC * kNCP);
        float4* s = reinterpret_cast<float4*>(Ts);
        for (int j = tid; j < kNC * kNCP / 4; j += 256) s[j] = g[j];
    }
    for (int j = tid; j < kTP * 363; j += 256) {
        const int p = j / 363, q = j % 363;
        float2 v = make_float2(0.f, 0.f);
        if (p < count) v = reinterpret_cast<const float2*>(mu + (size_t)srcb[begin + p] * kBoxStride)[q];
        const int k = q / 3, r2 = q % 3;
        *reinterpret_cast<float2*>(&Bs[k * kBCols + p * 6 + 2 * r2]) = v;
    }
    __syncthreads();
    const int rg = tid & 15, pg = tid >> 4;
    float acc[8][12];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int c = 0; c < 12; ++c) acc[a][c] = 0.f;
    const float* tp = Ts + rg * 8;
    const float* bp = Bs + pg * 12;
#pragma unroll 2
    for (int k = 0; k < kNC; ++k) {
        const float4 t0 = *reinterpret_cast<const float4*>(tp + k * kNCP);
        const float4 t1 = *reinterpret_cast<const float4*>(tp + k * kNCP + 4);
        const float4 b0 = *reinterpret_cast<const float4*>(bp + k * kBCols);
        const float4 b1 = *reinterpret_cast<const float4*>(bp + k * kBCols + 4);
        const float4 b2 = *reinterpret_cast<const float4*>(bp + k * kBCols + 8);
        const float tv[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
        const float bv[12] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x, b2.y, b2.z, b2.w};
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int c = 0; c < 12; ++c) acc[a][c] = fmaf(tv[a], bv[c], acc[a][c]);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int p = 2 * pg + q;
        if (p >= count) continue;
        float* base = ell + (size_t)tgt[begin + p] * kBoxStride;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int i = rg * 8 + 2 * j;
            if (i >= kNC) continue;
            float* o = base + 6 * i;
            const float* a0 = acc[2 * j] + 6 * q;
            const float* a1 = acc[2 * j + 1] + 6 * q;
            red_add_v4(o, a0[0], a0[1], a0[2], a0[3]);
            red_add_v4(o + 4, a0[4], a0[5], a1[0], a1[1]);
            if (i + 1 < kNC) red_add_v4(o + 8, a1[2], a1[3], a1[4], a1[5]);
        }
    }
}

// ------------------------------------------------------------------ P2L (X list)
__global__ void __launch_bounds__(128) k_p2l(const int32_t* __restrict__ xt, const int64_t* __restrict__ xptr,
                                             const int32_t* __restrict__ xsrc, const int32_t* __restrict__ level,
                                             const int32_t* __restrict__ ix, const int32_t* __restrict__ iy,
                                             const int32_t* __restrict__ iz, const int32_t* __restrict__ pb,
                                             const int32_t* __restrict__ pe, const float4* __restrict__ loc,
                                             const float* __restrict__ xq, float* __restrict__ ell)
{
    __shared__ float H[kChunk][kNC];
    __shared__ float Q[kChunk][6];
    const int b = xt[blockIdx.x];
    const int lb = level[b];
    const float3 cb = box_center(lb, ix[b], iy[b], iz[b]);
    const float inv_s = ldexpf(1.f, lb);
    float acc[6] = {0, 0, 0, 0, 0, 0};
    for (int64_t j = xptr[b]; j < xptr[b + 1]; ++j) {
        const int L = xsrc[j];
        const float3 cL = box_center(level[L], ix[L], iy[L], iz[L]);
        const float dx = cL.x - cb.x, dy = cL.y - cb.y, dz = cL.z - cb.z;
        for (int c0 = pb[L]; c0 < pe[L]; c0 += kChunk) {
            const int cn = min(kChunk, pe[L] - c0);
            if (threadIdx.x < cn) {
                const int i = c0 + threadIdx.x;
                const float4 p = loc[i];
                float h[kNC];
                irregular_harmonics<kP>((p.x + dx) * inv_s, (p.y + dy) * inv_s, (p.z + dz) * inv_s, c_tab, h);
#pragma unroll
                for (int k = 0; k < kNC; ++k) H[threadIdx.x][k] = (k == 0 || degree_of(k) * degree_of(k) == k) ? h[k] : 2.f * h[k];
#pragma unroll
                for (int r = 0; r < 6; ++r) Q[threadIdx.x][r] = xq[8 * (int64_t)i + r];
            }
            __syncthreads();
#pragma unroll
            for (int jj = 0; jj < 6; ++jj) {
                const int o = threadIdx.x + 128 * jj;
                if (o < kNC * 6) {
                    const int k = o / 6, r = o % 6;
                    float a = acc[jj];
                    for (int p = 0; p < cn; ++p) a += H[p][k] * Q[p][r];
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

// ------------------------------------------------------------------ leaf evaluation
// Per target leaf: L2P + M2P(W) + P2P(U) + near CSR; 128 threads = 2 halves x 64 targets.
__global__ void __launch_bounds__(128) k_leaf(
    const int32_t* __restrict__ leaves, const int32_t* __restrict__ level, const int32_t* __restrict__ ix,
    const int32_t* __restrict__ iy, const int32_t* __restrict__ iz, const int32_t* __restrict__ pb,
    const int32_t* __restrict__ pe, const int64_t* __restrict__ uptr, const int32_t* __restrict__ usrc,
    const int64_t* __restrict__ wptr, const int32_t* __restrict__ wsrc, const float4* __restrict__ loc,
    const float* __restrict__ xq, const float* __restrict__ mu, const float* __restrict__ ell,
    const int64_t* __restrict__ nptr, const int32_t* __restrict__ ncol, const float* __restrict__ nval, float invW,
    int do_far, int do_near, int64_t n, float2* __restrict__ y)
{
    __shared__ float Ls[kBoxStride];
    __shared__ float Ms[2][kBoxStride];
    __shared__ float4 Sp[128];
    __shared__ float Sq[128][6];
    __shared__ float Red[64][12];
    const int b = leaves[blockIdx.x];
    const int lb = level[b];
    const float3 cb = box_center(lb, ix[b], iy[b], iz[b]);
    const float inv_sb = ldexpf(1.f, lb);
    const int half = threadIdx.x >> 6, lane = threadIdx.x & 63;
    if (do_far)
        for (int j = threadIdx.x; j < kBoxStride / 4; j += 128)
            reinterpret_cast<float4*>(Ls)[j] = reinterpret_cast<const float4*>(ell + (size_t)b * kBoxStride)[j];
    for (int t0 = pb[b]; t0 < pe[b]; t0 += 64) {
        const int ti = t0 + lane;
        const bool act = ti < pe[b];
        float4 tp = make_float4(0.f, 0.f, 0.f, 0.f);
        if (act) tp = loc[ti];
        float far[6] = {0, 0, 0, 0, 0, 0}, nr[6] = {0, 0, 0, 0, 0, 0};
        __syncthreads();
        if (do_far) {
            // L2P
            if (half == 0 && act) {
                float h[kNC];
                regular_harmonics<kP>(tp.x * inv_sb, tp.y * inv_sb, tp.z * inv_sb, c_tab, h);
#pragma unroll
                for (int k = 0; k < kNC; ++k)
#pragma unroll
                    for (int r = 0; r < 6; ++r) far[r] += Ls[6 * k + r] * h[k];
#pragma unroll
                for (int r = 0; r < 6; ++r) far[r] *= inv_sb;
            }
            // M2P over the W list, two boxes per step (one per half)
            const int64_t w0 = wptr[b], w1 = wptr[b + 1];
            for (int64_t wj = w0; wj < w1; wj += 2) {
                __syncthreads();
                for (int j = threadIdx.x; j < 2 * (kBoxStride / 4); j += 128) {
                    const int hh = j / (kBoxStride / 4), q = j % (kBoxStride / 4);
                    if (wj + hh < w1)
                        reinterpret_cast<float4*>(Ms[hh])[q] =
                            reinterpret_cast<const float4*>(mu + (size_t)wsrc[wj + hh] * kBoxStride)[q];
                }
                __syncthreads();
                if (act && wj + half < w1) {
                    const int w = wsrc[wj + half];
                    const int lw = level[w];
                    const float3 cw = box_center(lw, ix[w], iy[w], iz[w]);
                    const float inv_sw = ldexpf(1.f, lw);
                    float h[kNC];
                    irregular_harmonics<kP>((tp.x + cb.x - cw.x) * inv_sw, (tp.y + cb.y - cw.y) * inv_sw,
                                            (tp.z + cb.z - cw.z) * inv_sw, c_tab, h);
                    float a[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
                    for (int k = 0; k < kNC; ++k) {
                        const float hk = (k == 0 || degree_of(k) * degree_of(k) == k) ? h[k] : 2.f * h[k];
#pragma unroll
                        for (int r = 0; r < 6; ++r) a[r] += Ms[half][6 * k + r] * hk;
                    }
#pragma unroll
                    for (int r = 0; r < 6; ++r) far[r] += a[r] * inv_sw;
                }
            }
            // P2P over the U list (W units)
            for (int64_t uj = uptr[b]; uj < uptr[b + 1]; ++uj) {
                const int s = usrc[uj];
                const float3 cs = box_center(level[s], ix[s], iy[s], iz[s]);
                const float dx = cs.x - cb.x, dy = cs.y - cb.y, dz = cs.z - cb.z;
                for (int s0 = pb[s]; s0 < pe[s]; s0 += 128) {
                    const int sn = min(128, pe[s] - s0);
                    __syncthreads();
                    if (threadIdx.x < sn) {
                        const int i = s0 + threadIdx.x;
                        const float4 p = loc[i];
                        Sp[threadIdx.x] = make_float4(p.x + dx, p.y + dy, p.z + dz, 0.f);
                        const float4 q0 = reinterpret_cast<const float4*>(xq + 8 * (int64_t)i)[0];
                        const float2 q1 = reinterpret_cast<const float2*>(xq + 8 * (int64_t)i)[2];
                        Sq[threadIdx.x][0] = q0.x; Sq[threadIdx.x][1] = q0.y; Sq[threadIdx.x][2] = q0.z;
                        Sq[threadIdx.x][3] = q0.w; Sq[threadIdx.x][4] = q1.x; Sq[threadIdx.x][5] = q1.y;
                    }
                    __syncthreads();
                    if (act) {
                        for (int j = half; j < sn; j += 2) {
                            const float4 sp = Sp[j];
                            const float ddx = tp.x - sp.x, ddy = tp.y - sp.y, ddz = tp.z - sp.z;
                            const float r2 = ddx * ddx + ddy * ddy + ddz * ddz;
                            const float ri = r2 > 0.f ? rsqrtf(r2) : 0.f;
#pragma unroll
                            for (int r = 0; r < 6; ++r) far[r] += Sq[j][r] * ri;
                        }
                    }
                }
            }
        }
        if (do_near && act) {
            for (int64_t j = nptr[ti] + half; j < nptr[ti + 1]; j += 2) {
                const float v = nval[j];
                const int64_t c = ncol[j];
                const float4 q0 = reinterpret_cast<const float4*>(xq + 8 * c)[0];
                const float2 q1 = reinterpret_cast<const float2*>(xq + 8 * c)[2];
                nr[0] += v * q0.x; nr[1] += v * q0.y; nr[2] += v * q0.z;
                nr[3] += v * q0.w; nr[4] += v * q1.x; nr[5] += v * q1.y;
            }
        }
        __syncthreads();
        if (half == 1) {
#pragma unroll
            for (int r = 0; r < 6; ++r) { Red[lane][r] = far[r]; Red[lane][6 + r] = nr[r]; }
        }
        __syncthreads();
        if (half == 0 && act) {
            float tot[6];
#pragma unroll
            for (int r = 0; r < 6; ++r) tot[r] = (far[r] + Red[lane][r]) * invW + (nr[r] + Red[lane][6 + r]);
            y[ti] = make_float2(tot[0], tot[1]);
            y[n + ti] = make_float2(tot[2], tot[3]);
            y[2 * n + ti] = make_float2(tot[4], tot[5]);
        }
    }
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
    for (int i = 0; i < 343; ++i) ctx->ops.m2l_index[i] = ops.m2l_index[i];
    XRL_CUDA(cudaFuncSetAttribute(k_m2l, cudaFuncAttributeMaxDynamicSharedMemorySize, kM2LSmem));
}

}  // namespace xrl

static void mvm_triple(xrl_tree t, xrl_near nr, const float2* x, float2* y, uint32_t flags)
{
    xrl_ctx ctx = t->ctx;
    cudaStream_t st = ctx->stream;
    const int64_t n = t->n;
    const bool do_far = flags != XRL_MVM_NEAR_ONLY;
    const bool do_near = flags != XRL_MVM_FAR_ONLY;
    cudaEvent_t ev;

    phase_begin(ctx, PH_PACK, &ev);
    k_pack<<<nblk(n, 256), 256, 0, st>>>(n, x, t->xq.p);
    XRL_LAUNCH_CHECK();
    ctx->launches += 1;
    phase_end(ctx, PH_PACK, ev);

    if (do_far && t->nlevel > 1) {
        phase_begin(ctx, PH_P2M, &ev);
        k_p2m<<<t->nleaf, 128, 0, st>>>(t->leaves.p, t->bpb.p, t->bpe.p, t->blevel.p, t->loc.p, t->xq.p, t->mu.p);
        XRL_LAUNCH_CHECK();
        ctx->launches += 1;
        phase_end(ctx, PH_P2M, ev);

        phase_begin(ctx, PH_M2M, &ev);
        for (int l = t->nlevel - 2; l >= 2; --l) {
            const int np = t->par_start[l + 1] - t->par_start[l];
            if (np == 0) continue;
            k_m2m<<<np, 128, 0, st>>>(t->parents.p + t->par_start[l], t->bchild.p, t->bnchild.p, t->bix.p, t->biy.p,
                                      t->biz.p, ctx->ops.m2m.p, t->mu.p);
            XRL_LAUNCH_CHECK();
            ctx->launches += 1;
        }
        phase_end(ctx, PH_M2M, ev);

        phase_begin(ctx, PH_M2L, &ev);
        XRL_CUDA(cudaMemsetAsync(t->ell.p, 0, t->ell.bytes(), st));
        if (t->n_m2l_tiles > 0) {
            k_m2l<<<t->n_m2l_tiles, 256, kM2LSmem, st>>>(t->m2l_tiles.p, t->m2l_tgt.p, t->m2l_srcb.p, ctx->ops.m2l.p,
                                                         t->mu.p, t->ell.p);
            XRL_LAUNCH_CHECK();
            ctx->launches += 1;
        }
        phase_end(ctx, PH_M2L, ev);

        phase_begin(ctx, PH_P2L, &ev);
        if (t->n_x_targets > 0) {
            k_p2l<<<t->n_x_targets, 128, 0, st>>>(t->x_targets.p, t->x_ptr.p, t->x_src.p, t->blevel.p, t->bix.p,
                                                  t->biy.p, t->biz.p, t->bpb.p, t->bpe.p, t->loc.p, t->xq.p, t->ell.p);
            XRL_LAUNCH_CHECK();
            ctx->launches += 1;
        }
        phase_end(ctx, PH_P2L, ev);

        phase_begin(ctx, PH_L2L, &ev);
        for (int l = 3; l < t->nlevel; ++l) {
            const int b0 = t->lvl_start[l], nb = t->lvl_start[l + 1] - b0;
            k_l2l<<<nb, 128, 0, st>>>(b0, t->bparent.p, t->bix.p, t->biy.p, t->biz.p, ctx->ops.l2l.p, t->ell.p);
            XRL_LAUNCH_CHECK();
            ctx->launches += 1;
        }
        phase_end(ctx, PH_L2L, ev);
    } else if (do_far) {
        XRL_CUDA(cudaMemsetAsync(t->ell.p, 0, t->ell.bytes(), st));
    }

    phase_begin(ctx, PH_LEAF, &ev);
    k_leaf<<<t->nleaf, 128, 0, st>>>(t->leaves.p, t->blevel.p, t->bix.p, t->biy.p, t->biz.p, t->bpb.p, t->bpe.p,
                                     t->u_ptr.p, t->u_src.p, t->w_ptr.p, t->w_src.p, t->loc.p, t->xq.p, t->mu.p,
                                     t->ell.p, nr->row_ptr.p, nr->col.p, nr->val.p, (float)(1.0 / t->W),
                                     do_far ? 1 : 0, do_near ? 1 : 0, n, y);
    XRL_LAUNCH_CHECK();
    ctx->launches += 1;
    phase_end(ctx, PH_LEAF, ev);
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
        for (int v = 0; v < nvec; v += 3)
            mvm_triple(t, nr, (const float2*)x + (size_t)v * t->n, (float2*)y + (size_t)v * t->n, flags);
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
