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
//   k_pack       complex64 [3][n] -> float [n][8] charges          (HBM, 48 B/panel)
//   k_near_rg<1> near correction N x, row-group format (side stream)      (HBM / L1 gathers)
//   k_p2p        U-list direct sum, packed f32x2 (side stream)     (FP32 pipe)
//   k_p2p12, k_near_rg<2>   the same for two triples in one pass (xrl_mvm nvec = 6k)
//   k_p2m        leaf multipoles mu = sum q Rt(u)                   (per leaf)
//   (M2M)        child -> parent per level on the tensor-core translation kernel (k_m2l_tc)
//   k_m2l_tc     V-list translations on tcgen05 (3xTF32, warp-specialised)
//   k_p2l        X-list particle -> local
//   (L2L)        parent -> child per level on k_m2l_tc
//   k_l2p_leaf   per owned leaf: ell to shared memory, L2P of its panels
//   k_m2p        W-list M2P (leaves with a W list), completes y
#include <cuda_fp16.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "tcgen05.h"
#include "xrl_internal.h"

using namespace xrl;

__constant__ RecTables<float> c_tab;

namespace {



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
// One CTA (128 threads) per owned leaf, panels in chunks of 128: (1) thread t evaluates the 121 regular solid
// harmonics of panel t of the chunk into H^T[k][t] (row stride 132: the float4 reads below are conflict-free)
// and stages its 6 charges; (2) mu[k][r] += sum_p H^T[k][p] q[p][r] as a register-blocked product: thread
// (lane l, warp g) owns coefficients k = l, l + 32, l + 64, l + 96 and the panels p = 32 g .. 32 g + 31, four
// at a time (one float4 of H^T per coefficient, the 4 panels' charges broadcast: 96 FMAs per 12 shared loads);
// (3) the 4 warps' partial sums are added through shared memory.
constexpr int kChunk = 128;       // panels per P2M pass (one per thread)
constexpr int kP2MLd = 132;       // H^T row stride (floats): 132 = 4 mod 32
constexpr int kP2MSmem = (kNC * kP2MLd + kChunk * 8) * 4;

__global__ void __launch_bounds__(128) k_p2m(const int32_t* __restrict__ leaves, const int32_t* __restrict__ pb,
                                             const int32_t* __restrict__ pe, const int32_t* __restrict__ level,
                                             const float4* __restrict__ loc, const float* __restrict__ xq,
                                             float* __restrict__ mu)
{
    static_assert(4 * 32 >= kNC && kNC * kP2MLd >= 4 * 128 * 6, "P2M shape");
    extern __shared__ __align__(16) float p2m_sm[];
    float* HT = p2m_sm;                                                 // [kNC][kP2MLd]
    float(*Q)[8] = reinterpret_cast<float(*)[8]>(p2m_sm + kNC * kP2MLd);  // [kChunk][8]
    const int b = leaves[blockIdx.x];
    const int s = pb[b], e = pe[b];
    const float inv_s = ldexpf(1.f, level[b]);
    const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
    float acc[4][6];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int r = 0; r < 6; ++r) acc[i][r] = 0.f;
    for (int c0 = s; c0 < e; c0 += kChunk) {
        const int cn = min(kChunk, e - c0);
        {
            const int t = threadIdx.x;
            if (t < cn) {
                const int i = c0 + t;
                const float4 p = loc[i];
                regular_harmonics_visit<kP>(p.x * inv_s, p.y * inv_s, p.z * inv_s, c_tab,
                                            [&](int kk, float v) { HT[kk * kP2MLd + t] = v; });
                const float4 q0 = *reinterpret_cast<const float4*>(xq + 8 * (int64_t)i);
                const float2 q1 = *reinterpret_cast<const float2*>(xq + 8 * (int64_t)i + 4);
                *reinterpret_cast<float4*>(Q[t]) = q0;
                *reinterpret_cast<float4*>(Q[t] + 4) = make_float4(q1.x, q1.y, 0.f, 0.f);
            } else {  // padding panels: zero charge (their harmonics column is never read with weight != 0)
#pragma unroll
                for (int kk = 0; kk < kNC; ++kk) HT[kk * kP2MLd + t] = 0.f;
                *reinterpret_cast<float4*>(Q[t]) = make_float4(0.f, 0.f, 0.f, 0.f);
                *reinterpret_cast<float4*>(Q[t] + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        __syncthreads();
        const int p_end = min(32 * g + 32, cn);
        for (int p = 32 * g; p < p_end; p += 4) {
            float4 h[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int k = lane + 32 * i;
                h[i] = k < kNC ? *reinterpret_cast<const float4*>(HT + k * kP2MLd + p) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float4 qa = *reinterpret_cast<const float4*>(Q[p + u]);
                const float2 qb = *reinterpret_cast<const float2*>(Q[p + u] + 4);
                const float q[6] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float hv = u == 0 ? h[i].x : (u == 1 ? h[i].y : (u == 2 ? h[i].z : h[i].w));
#pragma unroll
                    for (int r = 0; r < 6; ++r) acc[i][r] = fmaf(hv, q[r], acc[i][r]);
                }
            }
        }
        __syncthreads();
    }
    // partial sums of the 4 warps -> mu[r][k] (k >= 121 zero); HT is free now
    float* red = p2m_sm;  // [4 warps][6][128]
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int r = 0; r < 6; ++r) red[(g * 6 + r) * 128 + lane + 32 * i] = acc[i][r];
    __syncthreads();
    float* out = mu + (size_t)b * kMuStride;
    for (int j = threadIdx.x; j < 6 * 128; j += blockDim.x) {
        const int r = j >> 7, k = j & 127;
        const float v = red[(0 * 6 + r) * 128 + k] + red[(1 * 6 + r) * 128 + k] + red[(2 * 6 + r) * 128 + k] +
                        red[(3 * 6 + r) * 128 + k];
        out[r * 128 + k] = k < kNC ? v : 0.f;
    }
}

// degree n of real coefficient index i = n*n + j
__device__ __forceinline__ int degree_of(int i)
{
    int n = 0;
    while ((n + 1) * (n + 1) <= i) ++n;
    return n;
}

// ------------------------------------------------------------------ M2L on tcgen05
// Tensor-core M2L (V list) on tcgen05.mma: 3xFP16 (kind::f16, the default for the M2L) or 3xTF32
// (kind::tf32: the M2M / L2L passes, and the M2L with XRL_M2L_TF32=1).  Pairs (target t, source s) sharing one
// offset o are cut into tiles of <= 21 pairs; a tile is one 128 x 128 x 128 product
//     D[(p, r)][i] = sum_k A[(p, r)][k] B[i][k],   A = mu_s(p)[r][k], B = T_o[i][k]
// with row (p, r) = 6 p + r (126 rows used), i.e. the 6 RHS of 21 source multipoles against one operator.
// Roles (warp-specialised, one persistent CTA per SM):
//   warps 0-7 (loaders, kTcLdW; two per TMEM lane quarter, one per K-half; thread = TMEM lane (p, r)): LDG
//     the FP32 multipole row (r-major image, 512 B), split it into hi/lo parts (FP16 on power-of-2 scaled
//     values, or TF32) and tcgen05.st them into TMEM (A_hi, A_lo), one tile of prefetch lead;
//   warps 8-11 (drain, thread = TMEM lane): tcgen05.ld the 121 coefficients of row (p, r) into a
//     shared-memory stage and reduce it into ell[t(p)][r][0..123] (r-major) with one TMA bulk reduction
//     (cp.reduce.async.bulk .add.f32) per row;
//   warp kTcMmaW (MMA issuer, one elected thread): per K-half 3 MMAs per K-step (A_lo B_hi, A_hi B_lo, A_hi
//     B_hi; f16: 4 K16 steps, tf32: 8 K8 steps) into one of two TMEM accumulators; the operator hi/lo
//     (canonical K-major layout) stays in shared memory for a block of tiles with the same offset
//     (cp.async.bulk);
//   warps after it (kTcFuseW, fused P2P): P2P target-leaf tasks from the counter shared with k_p2p.
// mbarriers: a_full/a_free per K-half (A), d_full/d_free per accumulator, op_full.
// Blocks (runs of tiles with one (chunk, offset)) are dealt to the CTAs by the LPT schedule of tree.cu, so all
// CTAs work inside one L2-resident target chunk.
constexpr int kTcPairs = 21;                        // pairs per tile (126 of 128 TMEM lanes)
#ifndef XRL_FUSE_WARPS
#define XRL_FUSE_WARPS 3
#endif
constexpr int kTcLdW = 8;                           // loader warps (two per TMEM lane quarter, one per K-half)
constexpr int kTcMmaW = kTcLdW + 4;                 // the MMA warp (after 4 drain warps)
constexpr int kTcFuseW = XRL_FUSE_WARPS;            // fused-P2P warps (group 1, beside the MMA warp)
// A second fused-P2P group of 4 warps (one warpgroup after the MMA warp's) runs in the 3xFP16 M2L, staging in the
// half of the operator buffer the FP16 operator leaves free.  Registers are moved to the P2P warpgroups with
// setmaxnreg: loaders kTcRegLd, drain kTcRegDr, MMA + P2P warpgroups kTcRegP2P (launched at 96 per thread).
#ifndef XRL_FUSE2_WARPS
#define XRL_FUSE2_WARPS 4
#endif
constexpr int kTcFuse2W = XRL_FUSE2_WARPS;
static_assert(kTcFuse2W == 0 || (kTcFuse2W == 4 && kTcMmaW % 4 == 0 && kTcFuseW == 3), "warpgroup-aligned roles");
#ifndef XRL_TC_REGS_LD
#define XRL_TC_REGS_LD 104
#endif
#ifndef XRL_TC_REGS_DR
#define XRL_TC_REGS_DR 48
#endif
#ifndef XRL_TC_REGS_WG4
#define XRL_TC_REGS_WG4 112
#endif
#ifndef XRL_TC_REGS_WG3
#define XRL_TC_REGS_WG3 112
#endif
constexpr int kTcDrCols = XRL_FUSE2_WARPS ? 16 : 32;  // drain: accumulator columns per tcgen05.ld
constexpr int kTcRegLd = XRL_TC_REGS_LD, kTcRegDr = XRL_TC_REGS_DR, kTcRegP2P = XRL_TC_REGS_WG3,
              kTcRegP2P2 = XRL_TC_REGS_WG4;
constexpr int kTcThreads = 32 * (kTcMmaW + 1 + kTcFuseW + kTcFuse2W);
constexpr int kTcRegLaunch = 96;  // per-thread registers at launch (__maxnreg__) when kTcFuse2W > 0
// this warpgroup's register count: setmaxnreg.inc above the launch count, .dec below it
template <int kRegs>
__device__ __forceinline__ void set_max_regs()
{
    if constexpr (kRegs > kTcRegLaunch) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegs));
    else if constexpr (kRegs < kTcRegLaunch) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegs));
}
static_assert(kTcFuse2W == 0 || 32 * (8 * kTcRegLd + 4 * kTcRegDr + 4 * kTcRegP2P + 4 * kTcRegP2P2) <= kTcRegLaunch * kTcThreads,
              "setmaxnreg budget: the CTA's registers at launch (96 per thread)");
constexpr int kTcOpBytes = 128 * 128 * 4;           // one operator part (hi or lo): 64 KB
constexpr int kTcStageLd = 132;                     // drain stage row stride (floats; conflict-free STS.128)
constexpr int kTcSmem = 2 * kTcOpBytes + 128 * kTcStageLd * 4 + 1024 + 512 * 12 * 4;  // operator hi + lo, drain stage (+ align), fused-P2P staging
constexpr uint32_t kTcColAh = 0, kTcColAl = 128, kTcColD = 256;  // D buffers at 256 and 384

__device__ __forceinline__ void mbar_arrive(uint64_t* bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     tc::smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
                 : "memory");
}

// Bulk (TMA) reduction smem -> global, f32 add; bulk-group completion.
__device__ __forceinline__ void bulk_red_add_f32(float* dst, const float* src, uint32_t bytes)
{
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
                 "r"(tc::smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// 32-byte (whole sector) read-only load, no L1 allocation
__device__ __forceinline__ void ldg256(const float* p, float* v)
{
    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p));
}

__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t phase)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(tc::smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
// whole-warp wait with a warp-uniform exit condition (keeps the warp converged)
__device__ __forceinline__ void mbar_wait_warp(uint64_t* bar, uint32_t phase)
{
    while (!__all_sync(0xffffffffu, mbar_try(bar, phase))) {
    }
}


// ---------------------------------------------------------------- P2P tasks (shared with k_m2l_tc)
constexpr int kUWin = 64;
// Shared-memory scratch of one P2P leaf task (window of U-list leaves).
struct P2PWin {
    int Uoff[kUWin + 1], Uid[kUWin], Upb[kUWin];
    float3 Ud[kUWin];
    int wsum[2];
};

template <int kNT, int kChunk, int kBar>
__device__ void p2p_leaf(int b, int tb, int te, int tid, float* smraw, P2PWin& W, const int32_t* __restrict__ level,
                         const int32_t* __restrict__ ix, const int32_t* __restrict__ iy, const int32_t* __restrict__ iz,
                         const int32_t* __restrict__ pb, const int32_t* __restrict__ pe,
                         const int64_t* __restrict__ uptr, const int32_t* __restrict__ usrc,
                         const float4* __restrict__ loc, const float* __restrict__ xq, float invW, int accumulate,
                         int64_t n, int64_t p0, float2* __restrict__ y);

// P2P leaf tasks handed to the M2L kernel's fused P2P warps (3 warps, plus a 4-warp group in the 3xFP16 M2L;
// tasks[counter++] while the M2L runs; the
// standalone k_p2p takes the rest from the same counter).  leaves == nullptr: no fused P2P.
struct P2PTasks {
    const int4* tasks;  // (leaf, first target panel, #targets, -)
    int ntasks;
    int* counter;
    const int32_t *level, *ix, *iy, *iz, *pb, *pe;
    const int64_t* uptr;
    const int32_t* usrc;
    const float4* loc;
    const float* xq;
    float invW;
    int64_t n, p0;
    float2* y;
    int accumulate;  // 1: y already holds the near part (near-first side stream), the P2P adds to it
};
constexpr int kFuseChunk = 512;                          // sources staged per chunk by the fused P2P warps
constexpr int kFuseSmem = kFuseChunk * 12 * 4;           // their staging / reduction buffer (bytes)
constexpr int kFuse2Chunk = 1024;                        // the second group: 48 KB in the free operator half

// This CTA's tile sequence: blocks blockIdx.x, blockIdx.x + gridDim.x, ...; all tiles of each block.  In a
// multi-level launch (lvr != nullptr) `lev` is the level of the current block: level v owns the block rows
// [lvr[v], lvr[v+1]) (row = block index / gridDim.x).
struct TileSeq {
    int bi, ti, tend, lev;
    bool ok;
    __device__ void find(const int4* __restrict__ blocks, int nblocks, const int* __restrict__ lvr)
    {
        ok = false;
        for (; bi < nblocks; bi += gridDim.x) {
            const int4 bk = __ldg(blocks + bi);
            if (bk.y > 0) { ti = bk.x; tend = bk.x + bk.y; ok = true; break; }
        }
        if (ok && lvr) {
            const int row = bi / gridDim.x;
            while (row >= __ldg(lvr + lev + 1)) ++lev;
        }
    }
    __device__ TileSeq(const int4* __restrict__ blocks, int nblocks, const int* __restrict__ lvr = nullptr)
        : bi(blockIdx.x), ti(0), tend(0), lev(0), ok(false)
    {
        find(blocks, nblocks, lvr);
    }
    __device__ void advance(const int4* __restrict__ blocks, int nblocks, const int* __restrict__ lvr = nullptr)
    {
        if (++ti < tend) return;
        bi += gridDim.x;
        find(blocks, nblocks, lvr);
    }
};

// Grid barrier of a multi-level launch: the loaders of every CTA wait until all CTAs have drained level
// lv - 1 (done[lv - 1] == gridDim.x; one CTA per SM, all resident).  A watchdog traps instead of hanging.
__device__ __forceinline__ void wait_level(const int* done, int lv)
{
    if (!done || lv <= 0) return;
    long long spins = 0;
    for (;;) {
        int v;
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(done + lv - 1) : "memory");
        if (v >= (int)gridDim.x) break;
        __nanosleep(64);
        if (++spins > (1ll << 26)) asm volatile("trap;");
    }
}

// 32-byte load through L2 (coherent: data written earlier in the same launch by other CTAs)
__device__ __forceinline__ void ldg256_coherent(const float* p, float* v)
{
    asm volatile("ld.global.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p)
                 : "memory");
}

// blocks[j] = {first tile, #tiles, offset, chunk}; tiles[t] = {offset, first pair, #pairs, chunk}
// Scale exponent e of the multipoles for the 3xFP16 M2L: the largest |mu| times 2^e lies in [2^14, 2^15)
// (clamped to [-90, 90]: the drain's 2^-(e + opexp) stays a normal float; 0 when every multipole is zero).
__device__ __forceinline__ int mu_scale_exp(const unsigned* mumax)
{
    const unsigned bits = *mumax;  // written by k_mu_max before this launch (stream order)
    if (bits == 0u) return 0;
    return max(-90, min(90, 14 - ((int)(bits >> 23) - 127)));
}

// kH = false: 3xTF32 (kind::tf32, K = 8); the M2M / L2L passes.  kH = true: 3xFP16 (kind::f16, K = 16, twice
// the tensor rate at the same 11-bit significand per part) on power-of-2 scaled operands: every multipole times
// 2^e, e = 14 - exponent of the largest |mu| of the MVM (*mumax, k_mu_max), every operator times 2^opexp (host,
// largest |T| in [2^14, 2^15)); the drain multiplies by 2^-(e + opexp).  Used for the M2L.
template <bool kH>
#if XRL_FUSE2_WARPS
#define XRL_TC_REGS __maxnreg__(96)  /* kTcRegLaunch */
#else
#define XRL_TC_REGS __launch_bounds__(kTcThreads, 1)
#endif
__global__ void XRL_TC_REGS k_m2l_tc(const int4* __restrict__ blocks, int nblocks,
                                                          const int4* __restrict__ tiles,
                                                          const int32_t* __restrict__ tgt,
                                                          const int32_t* __restrict__ srcb,
                                                          const void* __restrict__ opimg,
                                                          const float* __restrict__ bimg, float* __restrict__ ell,
                                                          int dbg, P2PTasks p2p, const int* __restrict__ lvr,
                                                          int* __restrict__ lv_done, int nlv,
                                                          const unsigned* __restrict__ mumax, int opexp)
{
    constexpr uint32_t kOpPart = kH ? 128 * 128 * 2 : kTcOpBytes;  // bytes of one operator part (hi or lo)
    constexpr uint32_t kColAl = kH ? 64 : kTcColAl;
    extern __shared__ uint8_t tsm_raw[];
    uint8_t* opsm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
    float* stage = reinterpret_cast<float*>(opsm + 2 * kTcOpBytes);  // [128 rows][kTcStageLd]
    float* p2p_sm = stage + 128 * kTcStageLd;                          // fused P2P staging (kFuseSmem)
    __shared__ uint64_t a_full[2], a_free[2], d_full[2], d_free[2], op_full;
    __shared__ uint32_t tbase;
    __shared__ int m2l_live, p2p_task, p2p_task2;
    __shared__ P2PWin p2p_win, p2p_win2;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) m2l_live = kTcMmaW + 1;  // warps of the translation roles still running
    if (tid == 0) {
        for (int h = 0; h < 2; ++h) {
            tc::mbar_init(&a_full[h], 4);
            tc::mbar_init(&a_free[h], 1);
            tc::mbar_init(&d_full[h], 1);
            tc::mbar_init(&d_free[h], 4);
        }
        tc::mbar_init(&op_full, 1);
    }
    if (warp == kTcMmaW) tc::tmem_alloc<512>(&tbase);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tm = tbase;
    // roles by warpgroup (setmaxnreg is warpgroup-wide: each role branch starts with its own, so ptxas
    // allocates the branch within it): 0-7 loaders, 8-11 drain, 12 MMA, 13-15 fused P2P 1, 16-19 fused P2P 2
    if (warp >= kTcMmaW + 1 + kTcFuseW) {
        if (kTcFuse2W > 0) set_max_regs<kTcRegP2P2>();
        {
            // ---------------- fused P2P, second group (3xFP16 M2L only): staging in the free operator half
            if (kH && p2p.tasks) {
                const int tp = tid - 32 * (kTcMmaW + 1 + kTcFuseW);
                float* sm2 = reinterpret_cast<float*>(opsm + 2 * kOpPart);
                for (;;) {
                    if (tp == 0) p2p_task2 = *(volatile int*)&m2l_live > 0 ? atomicAdd(p2p.counter, 1) : INT_MAX;
                    asm volatile("bar.sync 3, %0;" ::"n"(32 * kTcFuse2W) : "memory");
                    const int task = p2p_task2;
                    if (task >= p2p.ntasks) break;
                    const int4 tk = p2p.tasks[task];
                    p2p_leaf<32 * kTcFuse2W, kFuse2Chunk, 3>(tk.x, tk.y, tk.y + tk.z, tp, sm2, p2p_win2, p2p.level, p2p.ix,
                                                             p2p.iy, p2p.iz, p2p.pb, p2p.pe, p2p.uptr, p2p.usrc, p2p.loc,
                                                             p2p.xq, p2p.invW, p2p.accumulate, p2p.n, p2p.p0, p2p.y);
                }
            }
        }
    } else if (warp >= kTcMmaW) {
        if (kTcFuse2W > 0) set_max_regs<kTcRegP2P>();
        if (warp > kTcMmaW) {
            // ---------------- fused P2P: three warps take target-leaf tasks from the shared counter while the
            // translation roles run (the M2L is bound by L2 traffic and leaves the FP32 pipes idle)
            if (p2p.tasks) {
                const int tp = tid - 32 * (kTcMmaW + 1);
                for (;;) {
                    if (tp == 0) p2p_task = *(volatile int*)&m2l_live > 0 ? atomicAdd(p2p.counter, 1) : INT_MAX;
                    asm volatile("bar.sync 1, %0;" ::"n"(32 * kTcFuseW) : "memory");
                    const int task = p2p_task;
                    if (task >= p2p.ntasks) break;
                    const int4 tk = p2p.tasks[task];
                    p2p_leaf<32 * kTcFuseW, kFuseChunk, 1>(tk.x, tk.y, tk.y + tk.z, tp, p2p_sm, p2p_win, p2p.level, p2p.ix, p2p.iy, p2p.iz,
                                                p2p.pb, p2p.pe, p2p.uptr, p2p.usrc, p2p.loc, p2p.xq, p2p.invW, p2p.accumulate, p2p.n,
                                                p2p.p0, p2p.y);
                }
            }
        } else {
            // ---------------- MMA issuer: the whole warp runs the loop with warp-uniform control
            // (block descriptors through shared memory, barrier waits voted with __all_sync) so the
            // descriptors stay in uniform registers and lane 0 issues back-to-back UTCHMMAs
            // (uniform bases recomputed here so they live in uniform registers)
            const uint32_t tmu = tbase;
            const uint32_t oph = (tc::smem_u32(tsm_raw) + 1023u) & ~1023u, opl = oph + kOpPart;
            const uint32_t idesc = kH ? tc::idesc_f16(128, 128) : tc::idesc_tf32(128, 128);
            int j = 0, nb = 0;
            for (int bi = blockIdx.x; bi < nblocks; bi += gridDim.x, ++nb) {
                int4 bk = __ldg(blocks + bi);
                bk.y = __shfl_sync(0xffffffffu, bk.y, 0);  // warp-uniform (keeps the MMA operands in uniform registers)
                bk.z = __shfl_sync(0xffffffffu, bk.z, 0);
                if (bk.y <= 0) { --nb; continue; }  // padding block of the balanced order: no operator load
                if (j > 0) {  // every MMA reading the previous operator must be complete
                    mbar_wait_warp(&d_full[(j - 1) & 1], ((j - 1) >> 1) & 1);
                    tc::fence_after();
                }
                if (lane == 0) {
                    mbar_expect_tx(&op_full, 2 * kOpPart);
                    const uint8_t* src = reinterpret_cast<const uint8_t*>(opimg) + (size_t)bk.z * 2 * kOpPart;
                    for (uint32_t c = 0; c < 2 * kOpPart / 32768; ++c)
                        bulk_g2s(opsm + c * 32768, src + c * 32768, 32768, &op_full);
                }
                mbar_wait_warp(&op_full, nb & 1);
                for (int ti = 0; ti < bk.y; ++ti, ++j) {
                    const int d = j & 1;
                    mbar_wait_warp(&d_free[d], ((j >> 1) & 1) ^ 1);
                    tc::fence_after();
                    const uint32_t dst = tmu + kTcColD + 128 * d;
    #pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        mbar_wait_warp(&a_full[h], j & 1);
                        tc::fence_after();
                        if (kH && tc::elect_one()) {
    #pragma unroll
                            for (int s = 4 * h; s < 4 * h + 4; ++s) {
                                // B element (i, k) at half ((i/8)*16 + k/8)*64 + (i%8)*8 + k%8: LBO 128, SBO 2048 bytes
                                const uint64_t bh = tc::smem_desc(oph + 256 * s, 128, 2048);
                                const uint64_t bl = tc::smem_desc(opl + 256 * s, 128, 2048);
                                tc::mma_f16_ts(dst, tmu + kColAl + 8 * s, bh, idesc, s > 0);
                                tc::mma_f16_ts(dst, tmu + kTcColAh + 8 * s, bl, idesc, 1);
                                tc::mma_f16_ts(dst, tmu + kTcColAh + 8 * s, bh, idesc, 1);
                            }
                            tc::commit(&a_free[h]);
                            if (h == 1) tc::commit(&d_full[d]);
                        } else if (!kH && tc::elect_one()) {
    #pragma unroll
                            for (int s = 8 * h; s < 8 * h + 8; ++s) {
                                // B (operator) element (i, k) at ((i/8)*32 + k/4)*128 + (i%8)*16 + (k%4)*4: LBO 128, SBO 4096
                                const uint64_t bh = tc::smem_desc(oph + 256 * s, 128, 4096);
                                const uint64_t bl = tc::smem_desc(opl + 256 * s, 128, 4096);
                                tc::mma_tf32_ts(dst, tmu + kTcColAl + 8 * s, bh, idesc, s > 0);
                                tc::mma_tf32_ts(dst, tmu + kTcColAh + 8 * s, bl, idesc, 1);
                                tc::mma_tf32_ts(dst, tmu + kTcColAh + 8 * s, bh, idesc, 1);
                            }
                            tc::commit(&a_free[h]);
                            if (h == 1) tc::commit(&d_full[d]);
                        }
                        __syncwarp();
                    }
                }
            }
        }
    } else if (warp < kTcLdW) {
        if (kTcFuse2W > 0) set_max_regs<kTcRegLd>();
        // ---------------- loaders: thread = TMEM lane L = (p, r); warps w and w + 4 share lane quarter w % 4,
        // warps 0-3 convert K-half 0 of their rows and warps 4-7 K-half 1.  Each thread's half row (64 floats,
        // 8 x 256-bit loads: whole 32-byte sectors) of the next tile is loaded right after the current one is
        // handed to the MMA, so the gathers have a whole tile period to arrive.
        const int L = tid & 127, p = L / 6, r = L % 6, h = warp >> 2;
        const bool lane_ok = L < 6 * kTcPairs;
        const uint32_t ta = tm + ((uint32_t)(32 * (warp & 3)) << 16);
        auto row_of = [&](const int4& tl, bool ok) -> const float* {
            if (!ok || !lane_ok || p >= tl.z || (dbg & 2)) return nullptr;
            return bimg + (size_t)__ldg(srcb + tl.y + p) * kMuStride + r * 128;
        };
        const float sc0 = kH ? __int_as_float((127 + mu_scale_exp(mumax)) << 23) : 1.f;  // the multipoles' 2^e
        float x[64];
        auto load_half = [&](const float* row) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                if (row) {
                    if (lvr) ldg256_coherent(row + 64 * h + 8 * c, x + 8 * c);  // written in this launch
                    else ldg256(row + 64 * h + 8 * c, x + 8 * c);
                } else {
#pragma unroll
                    for (int q = 0; q < 8; ++q) x[8 * c + q] = 0.f;
                }
            }
        };
        auto level_gate = [&](int lv) {  // the previous level is complete in every CTA
            if (lane == 0) wait_level(lv_done, lv);
            __syncwarp();
        };
        TileSeq s0(blocks, nblocks, lvr);
        if (s0.ok) level_gate(s0.lev);
        load_half(row_of(s0.ok ? __ldg(tiles + s0.ti) : make_int4(0, 0, 0, 0), s0.ok));
        for (int j = 0; s0.ok; ++j) {
            TileSeq s1 = s0;
            s1.advance(blocks, nblocks, lvr);
            const int4 tl1 = s1.ok ? __ldg(tiles + s1.ti) : make_int4(0, 0, 0, 0);
            // the MMAs of the previous tile must be done with this K-half of A
            tc::mbar_wait(&a_free[h], (j & 1) ^ 1);
            tc::fence_after();
            if constexpr (kH) {
#pragma unroll
                for (int c2 = 0; c2 < 4; ++c2) {  // 16 coefficients = 8 columns of packed f16 pairs at a time
                    uint32_t hi[8], lo[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const float a = x[16 * c2 + 2 * q] * sc0, b = x[16 * c2 + 2 * q + 1] * sc0;
                        const __half2 hh = __floats2half2_rn(a, b);  // .x (low half) = a: the lower k
                        const float2 hf = __half22float2(hh);
                        const __half2 ll = __floats2half2_rn(a - hf.x, b - hf.y);
                        hi[q] = *reinterpret_cast<const uint32_t*>(&hh);
                        lo[q] = *reinterpret_cast<const uint32_t*>(&ll);
                    }
                    tc::tmem_st8u(ta + kTcColAh + 32 * h + 8 * c2, hi);
                    tc::tmem_st8u(ta + kColAl + 32 * h + 8 * c2, lo);
                }
            } else {
#pragma unroll
                for (int c2 = 0; c2 < 8; ++c2) {  // 8 columns at a time
                    float hi[8], lo[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        hi[q] = tc::tf32_rna(x[8 * c2 + q]);
                        lo[q] = x[8 * c2 + q] - hi[q];
                    }
                    tc::tmem_st8(ta + kTcColAh + 64 * h + 8 * c2, hi);
                    tc::tmem_st8(ta + kTcColAl + 64 * h + 8 * c2, lo);
                }
            }
            tc::tmem_st_wait();
            tc::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&a_full[h]);
            if (s1.ok) {
                // a tile of the next level is read only after the grid barrier (this tile is already handed over)
                if (s1.lev != s0.lev) level_gate(s1.lev);
                load_half(row_of(tl1, true));
            }
            s0 = s1;
        }
    } else {
        if (kTcFuse2W > 0) set_max_regs<kTcRegDr>();
        // ---------------- drain: thread = TMEM lane L = (p, r) reads its accumulator row into a
        // shared-memory stage; then each thread reduces its whole row into ell with one TMA bulk
        // reduction (asynchronous: frees the drain warps; tools/ubench_red.cu measured the variants)
        const int L = tid - 32 * kTcLdW, p = L / 6, r = L % 6;
        const bool lane_ok = L < 6 * kTcPairs;
        const int qd = warp & 3;  // lane quarter (warp % 4)
        // multi-level launch: after its last tile of a level, every drain thread waits for its bulk reductions
        // to complete and fences them; then one thread marks the level (and any level this CTA had no tile
        // in) done for the other CTAs' loaders
        int signaled = 0;
        auto signal_upto = [&](int lv) {  // levels [signaled, lv) are complete in this CTA
            if (!lv_done || lv <= signaled) return;
            bulk_wait0();
            asm volatile("fence.proxy.async.global;" ::: "memory");
            __threadfence();
            asm volatile("bar.sync 2, 128;" ::: "memory");
            if (L == 0)
                for (int v = signaled; v < lv; ++v) atomicAdd(lv_done + v, 1);
            signaled = lv;
        };
        const float unscale = kH ? __int_as_float((127 - mu_scale_exp(mumax) - opexp) << 23) : 1.f;
        TileSeq sq(blocks, nblocks, lvr);
        if (sq.ok) signal_upto(sq.lev);
        int4 cur = sq.ok ? __ldg(tiles + sq.ti) : make_int4(0, 0, 0, 0);
        int cur_t = (sq.ok && lane_ok && p < cur.z) ? __ldg(tgt + cur.y + p) : -1;
        for (int j = 0; sq.ok; ++j) {
            TileSeq nx = sq;
            nx.advance(blocks, nblocks, lvr);
            int nxt_t = -1;
            int4 nxt = make_int4(0, 0, 0, 0);
            if (nx.ok) {
                nxt = __ldg(tiles + nx.ti);
                if (lane_ok && p < nxt.z) nxt_t = __ldg(tgt + nxt.y + p);
            }
            const int d = j & 1;
            tc::mbar_wait(&d_full[d], (j >> 1) & 1);
            tc::fence_after();
            const uint32_t ta = tm + ((uint32_t)(32 * qd) << 16) + kTcColD + 128 * d;
            float* srow = stage + L * kTcStageLd;
            bulk_wait_read0();  // this thread's previous bulk reduction has finished reading its stage row
#pragma unroll
            for (int c = 0; c < 128 / kTcDrCols; ++c) {  // kTcDrCols columns per tcgen05.ld (registers: see kTcRegDr)
                float v[kTcDrCols];
                if (dbg & 4) {
                    for (int q = 0; q < kTcDrCols; ++q) v[q] = 0.f;
                } else {
                    if (kTcDrCols == 32) tc::tmem_ld32(ta + kTcDrCols * c, v);
                    else tc::tmem_ld16(ta + kTcDrCols * c, v);
                    if (kH) {
#pragma unroll
                        for (int q = 0; q < kTcDrCols; ++q) v[q] *= unscale;
                    }
                }
#pragma unroll
                for (int q = 0; q < kTcDrCols / 4; ++q)
                    *reinterpret_cast<float4*>(srow + kTcDrCols * c + 4 * q) =
                        make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            }
            tc::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&d_free[d]);  // accumulator d may be overwritten
            if (cur_t >= 0 && !(dbg & 1)) {
                // row (p, r) -> ell[t][r][0..123] with one bulk reduction (TMA, whole lines in L2)
                tc::fence_proxy_async();
                bulk_red_add_f32(ell + (size_t)cur_t * kEllStride + r * 128, srow, 124 * 4);
                bulk_commit();
            }
            if (nx.ok && nx.lev != sq.lev) signal_upto(nx.lev);
            sq = nx;
            cur = nxt;
            cur_t = nxt_t;
        }
        if (lvr) signal_upto(nlv);
        bulk_wait0();
    }
    if (warp <= kTcMmaW && lane == 0) atomicSub(&m2l_live, 1);
    tc::fence_before();
    __syncthreads();
    if (warp == kTcMmaW) tc::tmem_dealloc<512>(tbase);
}

// Largest |mu| of the MVM for the 3xFP16 M2L scale: *mumax = max over the boxes' multipole coefficients (as the
// bits of a non-negative float, so an unsigned atomicMax orders them); one warp per box, 6 rows of 124 floats.
__global__ void __launch_bounds__(256) k_mu_max(int nbox, const float* __restrict__ mu, unsigned* __restrict__ mumax)
{
    const int b = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    float m = 0.f;
    if (b < nbox && lane < 31) {
#pragma unroll
        for (int r = 0; r < 6; ++r) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(mu + (size_t)b * kMuStride + r * 128) + lane);
            m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, d));
    __shared__ float wm[8];
    if (lane == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) m = fmaxf(m, wm[w]);
        atomicMax(mumax, __float_as_uint(m));
    }
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
    float* out = ell + (size_t)b * kEllStride;
#pragma unroll
    for (int jj = 0; jj < 6; ++jj) {
        const int o = threadIdx.x + 128 * jj;
        if (o < kNC * 6) atomicAdd(out + (o % 6) * 128 + o / 6, acc[jj]);  // may run beside the M2L's reductions
    }
}

// ------------------------------------------------------------------ near-field SpMV
// y += N x for the 6 real RHS (N: the near correction and the self terms) over the
// row-group format of near.cu (build_near_groups): 8 lanes per segment, 4 segments per warp.  Per union column
// of a group of 4 rows a lane gathers one 32-byte charge record (L1-cached: neighbouring groups share their
// near columns) and applies the float4 of the 4 rows' values to it (24 FMAs).  A lane's next four column
// offsets (one u64) are loaded one chunk ahead, so the offset -> gather chain of one chunk overlaps the
// previous chunk; the 8 lanes reduce-scatter the 4 x 6 sums with 24 shuffles and add them into y with vector
// L2 reductions (a group with several segments adds several times; the L2P / M2P add concurrently).

// 32-byte read-only load through L1 (the charge records are re-read by neighbouring rows)
__device__ __forceinline__ void ldg256_l1(const float* p, float* v)
{
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p));
}

// y += (a, b) as one vector L2 reduction (the L2P and the near SpMV may run concurrently into y)
__device__ __forceinline__ void red_add2(float2* p, float a, float b)
{
    asm volatile("red.global.add.v2.f32 [%0], {%1,%2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}

// streaming loads of the near entries: read once per MVM, so no L1 allocation and L2 evict-first (the
// 1.2 GB stream must not evict the 61 MB of charge records the gathers re-read from L2)
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ float4 ldg_stream4(const float* p, uint64_t pol)
{
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint2 ldg_stream_u64(const uint16_t* p, uint64_t pol)
{
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
    return v;
}
// 32-byte charge-record gather through L1, L2 evict-last
__device__ __forceinline__ void ldg256_l1_keep(const float* p, float* v, uint64_t pol)
{
    asm volatile("ld.global.nc.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p), "l"(pol));
}

__device__ __forceinline__ float4 ldg_stream4v(const float4* p, uint64_t pol)
{
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}

// a[j * 6 + r] (row j of the group, RHS r) summed over the 8 lanes of a team; lane l8 ends with the sums of row
// 2 (l8 >> 2 & 1) + (l8 >> 1 & 1) in c[0..5] (xor 4 halves the rows, xor 2 halves them again, xor 1 all-reduces)
__device__ __forceinline__ void rg_reduce(const float (&a)[24], int l8, float (&c)[6])
{
    const unsigned m = 0xffu << (threadIdx.x & 24);  // the team's lanes (teams of a warp may leave the loop apart)
    const bool h2 = l8 & 4, h1 = l8 & 2;
    float b[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) {
        const float send = h2 ? a[k] : a[12 + k], keep = h2 ? a[12 + k] : a[k];
        b[k] = keep + __shfl_xor_sync(m, send, 4);
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const float send = h1 ? b[k] : b[6 + k], keep = h1 ? b[6 + k] : b[k];
        c[k] = keep + __shfl_xor_sync(m, send, 2);
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) c[k] += __shfl_xor_sync(m, c[k], 1);
}

// NT = 1: one triple (xq -> y); NT = 2: two triples in one pass over the format (xq -> y, xq2 -> y2).
// Each CTA owns a contiguous, slot-balanced range of segments (consecutive groups share most of their columns,
// so the CTA's charge gathers hit L1 again); its 32 teams take the range's segments round-robin.
#ifndef XRL_NEAR_MINB
#define XRL_NEAR_MINB 2
#endif
#ifndef XRL_NEAR_PFW
#define XRL_NEAR_PFW 0
#endif
constexpr bool kNearPfw = XRL_NEAR_PFW;
#ifndef XRL_NEAR_G6
#define XRL_NEAR_G6 0
#endif
// charge record gather: one 32-byte load (8 registers), or XRL_NEAR_G6 16 + 8 bytes (6 registers, 2 requests)
constexpr int kNearQ = XRL_NEAR_G6 ? 6 : 8;
__device__ __forceinline__ void ldg_rec_keep(const float* p, float* v, uint64_t pol)
{
    if (XRL_NEAR_G6) {
        asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "l"(p), "l"(pol));
        asm volatile("ld.global.nc.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;" : "=f"(v[4]), "=f"(v[5]) : "l"(p + 4), "l"(pol));
    } else {
        ldg256_l1_keep(p, v, pol);
    }
}
#ifndef XRL_NEAR_NT
#define XRL_NEAR_NT 256
#endif
template <int NT>
__global__ void __launch_bounds__(XRL_NEAR_NT, NT == 1 ? XRL_NEAR_MINB : 512 / XRL_NEAR_NT) k_near_rg(int64_t nseg, const int32_t* __restrict__ seg_grp,
                                                  const int32_t* __restrict__ seg_base,
                                                  const int64_t* __restrict__ seg_off, const float4* __restrict__ gval,
                                                  const uint16_t* __restrict__ eoff, const float* __restrict__ xq,
                                                  const float* __restrict__ xq2, int64_t nl, float2* __restrict__ y,
                                                  float2* __restrict__ y2)
{
    __shared__ int64_t rng[2];
    if (threadIdx.x < 2) {
        const int64_t E = __ldg(seg_off + nseg);
        const int64_t target = (E * (int64_t)(blockIdx.x + threadIdx.x)) / gridDim.x;
        int64_t lo = 0, hi = nseg;  // first segment whose start is >= target
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (__ldg(seg_off + mid) < target) lo = mid + 1; else hi = mid;
        }
        rng[threadIdx.x] = (blockIdx.x + threadIdx.x == gridDim.x) ? nseg : lo;
    }
    __syncthreads();
    const int64_t s_end = rng[1];
    const int64_t nteams = blockDim.x >> 3;
    const int l8 = threadIdx.x & 7;
    const uint64_t pol_stream = policy_evict_first(), pol_keep = policy_evict_last();
    int64_t s = rng[0] + (threadIdx.x >> 3);
    int64_t b0 = 0, b1 = 0;  // slot range of segment s
    int32_t base = 0;
    if (s < s_end) { b0 = __ldg(seg_off + s); b1 = __ldg(seg_off + s + 1); base = __ldg(seg_base + s); }
    uint2 o = make_uint2(0u, 0u);
    if (s < s_end && b0 + 4 * l8 < b1) o = ldg_stream_u64(eoff + b0 + 4 * l8, pol_stream);
    // values of the chunk at block start `bs` of a segment ending at `be` (the lane's u-th value at u nc + l8)
    auto load_w = [&](int64_t bs, int64_t be, float4 (&w)[4]) {
        const int nc = (int)(be - bs < 32 ? be - bs : 32) >> 2;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            w[u] = l8 < nc ? ldg_stream4v(gval + bs + u * nc + l8, pol_stream) : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    float4 pw[4];  // XRL_NEAR_PFW: the next chunk's values, loaded one chunk ahead like the offsets
    if (kNearPfw) {
        if (s < s_end) load_w(b0, b1, pw);
        else for (int u = 0; u < 4; ++u) pw[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    while (s < s_end) {
        const int64_t sn = s + nteams;
        int64_t n0 = 0, n1 = 0;
        int32_t nbase = 0;
        if (sn < s_end) { n0 = __ldg(seg_off + sn); n1 = __ldg(seg_off + sn + 1); nbase = __ldg(seg_base + sn); }
        const int64_t grp = __ldg(seg_grp + s);
        float a[NT][24];
#pragma unroll
        for (int v = 0; v < NT; ++v)
#pragma unroll
            for (int k = 0; k < 24; ++k) a[v][k] = 0.f;
        const int nit = (int)((b1 - b0 + 31) >> 5);  // chunk rounds of the team (uniform over its 8 lanes)
        for (int it = 0; it < nit; ++it) {
            const int64_t blk = b0 + 32 * it;
            const int nc = (int)(b1 - blk < 32 ? b1 - blk : 32) >> 2;  // lanes with a chunk in this block
            const bool act = l8 < nc;
            // a lane without a chunk gathers record `base` with weight 0 (no branches around the gathers)
            const uint32_t c0 = act ? o.x & 0xffff : 0u, c1 = act ? o.x >> 16 : 0u;
            const uint32_t c2 = act ? o.y & 0xffff : 0u, c3 = act ? o.y >> 16 : 0u;
            // the next chunk's offsets: this segment's, else the next segment's first
            const int64_t np = it + 1 < nit ? blk + 32 + 4 * l8 : n0 + 4 * l8;
            const int64_t ne = it + 1 < nit ? b1 : n1;
            if ((it + 1 < nit || sn < s_end) && np < ne) o = ldg_stream_u64(eoff + np, pol_stream);
            float4 w[4];
            if (kNearPfw) {
#pragma unroll
                for (int u = 0; u < 4; ++u) w[u] = pw[u];
                if (it + 1 < nit) load_w(blk + 32, b1, pw);
                else if (sn < s_end) load_w(n0, n1, pw);
            } else {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    w[u] = act ? ldg_stream4v(gval + blk + u * nc + l8, pol_stream) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int v = 0; v < NT; ++v) {
                const float* xb = (v == 0 ? xq : xq2) + 8 * (int64_t)base;
                float q[4][kNearQ];
                ldg_rec_keep(xb + 8 * c0, q[0], pol_keep);
                ldg_rec_keep(xb + 8 * c1, q[1], pol_keep);
                ldg_rec_keep(xb + 8 * c2, q[2], pol_keep);
                ldg_rec_keep(xb + 8 * c3, q[3], pol_keep);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float wj[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
#pragma unroll
                    for (int j = 0; j < 4; ++j)
#pragma unroll
                        for (int r = 0; r < 6; ++r) a[v][j * 6 + r] = fmaf(wj[j], q[u][r], a[v][j * 6 + r]);
                }
            }
        }
#pragma unroll
        for (int v = 0; v < NT; ++v) {
            float c[6];
            rg_reduce(a[v], l8, c);
            const int64_t row = kNearG * grp + 2 * ((l8 >> 2) & 1) + ((l8 >> 1) & 1);
            float2* yv = v == 0 ? y : y2;
            if (row < nl) {
                if (l8 & 1) red_add2(yv + 2 * nl + row, c[4], c[5]);
                else { red_add2(yv + row, c[0], c[1]); red_add2(yv + nl + row, c[2], c[3]); }
            }
        }
        s = sn;
        b0 = n0;
        b1 = n1;
        base = nbase;
    }
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
#ifndef XRL_P2P_CHUNK
#define XRL_P2P_CHUNK 1024
#endif
constexpr int kSrcChunk = XRL_P2P_CHUNK;
constexpr int kP2PSmem = (kSrcChunk * 12 > 128 * (4 * 6 + 1) * 2 ? kSrcChunk * 12 : 128 * (4 * 6 + 1) * 2) * 4;
#ifndef XRL_P2P_TPT
#define XRL_P2P_TPT 8
#endif
#ifndef XRL_P2P_UNROLL
#define XRL_P2P_UNROLL 2
#endif
constexpr int kTPT = XRL_P2P_TPT;
constexpr int kP2PUnroll = XRL_P2P_UNROLL;
constexpr int kTP2 = kTPT / 2;  // packed target pairs per thread

// Packed FP32 pairs (sm_100 FFMA2/FADD2/FMUL2): two targets per instruction.
// A scalar operand is broadcast to both halves by ptxas (".F32" operand form).
using f2x = unsigned long long;
__device__ __forceinline__ f2x pk2(float a, float b)
{
    f2x r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float2 upk2(f2x v)
{
    float2 r;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ f2x fma2(f2x a, f2x b, f2x c)
{
    f2x d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ void fma2_acc(f2x& acc, f2x a, f2x b)
{
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}
__device__ __forceinline__ f2x sub2(f2x a, f2x b)
{
    f2x d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2x mul2(f2x a, f2x b)
{
    f2x d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2x ld_shared_u64(const void* p)
{
    f2x v;
    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
    return v;
}
__device__ __forceinline__ void st_shared_u64(void* p, f2x v)
{
    asm volatile("st.shared.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "l"(v) : "memory");
}
// MUFU.RSQ without the denormal fix-up (FTZ, R8: r^2 is O(1e-12) or larger in W units)
__device__ __forceinline__ float rsqrt_ftz(float x)
{
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// one source j against the thread's kTP2 target pairs
template <bool kSelf>
__device__ __forceinline__ void p2p_one(int j, const float4* __restrict__ Sp, const float4 (*__restrict__ Sq)[2],
                                        const f2x* tx, const f2x* ty, const f2x* tz, f2x (*acc)[6])
{
    const float4 sp = Sp[j];
    const float4 q0 = Sq[j][0], q1 = Sq[j][1];
    const f2x sx = pk2(sp.x, sp.x), sy = pk2(sp.y, sp.y), sz = pk2(sp.z, sp.z);
    const f2x c0 = pk2(q0.x, q0.x), c1 = pk2(q0.y, q0.y), c2 = pk2(q0.z, q0.z);
    const f2x c3 = pk2(q0.w, q0.w), c4 = pk2(q1.x, q1.x), c5 = pk2(q1.y, q1.y);
#pragma unroll
    for (int q = 0; q < kTP2; ++q) {
        const f2x dx = sub2(tx[q], sx), dy = sub2(ty[q], sy), dz = sub2(tz[q], sz);
        const float2 r2 = upk2(fma2(dx, dx, fma2(dy, dy, mul2(dz, dz))));
        float ra = rsqrt_ftz(r2.x), rb = rsqrt_ftz(r2.y);
        if (kSelf) {
            ra = r2.x > 0.f ? ra : 0.f;
            rb = r2.y > 0.f ? rb : 0.f;
        }
        const f2x ri = pk2(ra, rb);
        fma2_acc(acc[q][0], c0, ri); fma2_acc(acc[q][1], c1, ri); fma2_acc(acc[q][2], c2, ri);
        fma2_acc(acc[q][3], c3, ri); fma2_acc(acc[q][4], c4, ri); fma2_acc(acc[q][5], c5, ri);
    }
}

// Per source: 3 FADD2 + FMUL2 + 2 FFMA2 + 2 MUFU + 6 FFMA2 per two targets (7 issue slots per pair).  The main
// loop takes kP2PUnroll sources per trip without guards, so ptxas interleaves one source's rsqrt chain with the
// other's charge FMAs; the remainder follows.
template <bool kSelf>
__device__ __forceinline__ void p2p_range(int j0, int j1, int S, const float4* __restrict__ Sp,
                                          const float4 (*__restrict__ Sq)[2], const f2x* tx, const f2x* ty,
                                          const f2x* tz, f2x (*acc)[6])
{
    int j = j0;
#pragma unroll 1
    for (; j + (kP2PUnroll - 1) * S < j1; j += kP2PUnroll * S) {
#pragma unroll
        for (int u = 0; u < kP2PUnroll; ++u) p2p_one<kSelf>(j + u * S, Sp, Sq, tx, ty, tz, acc);
    }
#pragma unroll 1
    for (; j < j1; j += S) p2p_one<kSelf>(j, Sp, Sq, tx, ty, tz, acc);
}

__device__ __forceinline__ int first_in_class(int lo, int sg, int S)
{
    // smallest j >= lo with j % S == sg
    const int r = lo % S;
    return lo + ((sg - r + S) % S);
}


// P2P of targets [tb, te) of leaf b by kNT threads (tid 0..kNT-1) synchronised with barrier kBar (0:
// __syncthreads, else a named barrier of kNT threads); smraw: kChunk * 12 floats of staging, also the
// reduction buffer (>= kNT * (kTP2 * 6 + 1) * 2 floats).
template <int kNT, int kChunk, int kBar>
__device__ void p2p_leaf(
    int b, int tb, int te, int tid, float* smraw, P2PWin& W, const int32_t* __restrict__ level, const int32_t* __restrict__ ix,
    const int32_t* __restrict__ iy, const int32_t* __restrict__ iz, const int32_t* __restrict__ pb,
    const int32_t* __restrict__ pe, const int64_t* __restrict__ uptr, const int32_t* __restrict__ usrc,
    const float4* __restrict__ loc, const float* __restrict__ xq, float invW, int accumulate, int64_t n,
    int64_t p0, float2* __restrict__ y)
{
    static_assert(kNT >= kUWin && kChunk * 12 >= kNT * (kTP2 * 6 + 1) * 2, "P2P task shape");
    // n, p0: owned panel range [p0, p0+n), y local [3][n]
    // the source staging buffers and the final reduction share one buffer (smraw)
    float4* Sp = reinterpret_cast<float4*>(smraw);
    float4(*Sq)[2] = reinterpret_cast<float4(*)[2]>(smraw + 4 * kChunk);
    f2x(*Red)[kTP2 * 6 + 1] = reinterpret_cast<f2x(*)[kTP2 * 6 + 1]>(smraw);  // packed target pairs
    int* Uoff = W.Uoff;
    int* Uid = W.Uid;
    int* Upb = W.Upb;
    float3* Ud = W.Ud;
    int* wsum = W.wsum;
    const float3 cb = box_center(level[b], ix[b], iy[b], iz[b]);
    const int lane = tid & 31, warp = tid >> 5;
    auto sync = [&]() {
        if (kBar == 0) __syncthreads();
        else asm volatile("bar.sync %0, %1;" ::"r"(kBar), "r"(kNT) : "memory");
    };
    for (int t0 = tb; t0 < te; t0 += kNT * kTPT) {
        const int T = min(kNT * kTPT, te - t0);
        const int NG = (T + kTPT - 1) / kTPT;
        const int S = max(1, kNT / NG);
        const int tg = tid % NG, sg = tid / NG;
        const bool act = sg < S;
        f2x tx[kTP2], ty[kTP2], tz[kTP2];
        f2x acc[kTP2][6];  // acc[q][r] = (y of target 2q, y of target 2q+1), RHS r
#pragma unroll
        for (int q = 0; q < kTP2; ++q) {
            float4 p[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int ti = tg * kTPT + 2 * q + h;
                p[h] = make_float4(1e18f, 1e18f, 1e18f, 0.f);  // padding target: far away, discarded
                if (act && ti < T) p[h] = loc[t0 + ti];
            }
            // round trip through shared memory so each packed pair is defined by one 64-bit load
            // (ptxas otherwise keeps the halves in unrelated registers and re-pairs them per use)
            float2* tp = reinterpret_cast<float2*>(smraw) + (tid * kTP2 + q) * 3;
            tp[0] = make_float2(p[0].x, p[1].x);
            tp[1] = make_float2(p[0].y, p[1].y);
            tp[2] = make_float2(p[0].z, p[1].z);
            tx[q] = ld_shared_u64(tp);
            ty[q] = ld_shared_u64(tp + 1);
            tz[q] = ld_shared_u64(tp + 2);
#pragma unroll
            for (int r = 0; r < 6; ++r) acc[q][r] = 0ull;
        }
        for (int64_t u0 = uptr[b]; u0 < uptr[b + 1]; u0 += kUWin) {
            const int nu = (int)min((int64_t)kUWin, uptr[b + 1] - u0);
            sync();
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
            sync();
            if (tid >= 32 && tid < kUWin) Uoff[tid + 1] += wsum[0];
            if (tid == 0) Uoff[0] = 0;
            sync();
            const int total = Uoff[nu];
            // the target leaf's own panels in the flattened window (needs the r = 0 guard)
            int self_lo = 0, self_hi = 0;
            for (int i = 0; i < nu; ++i)
                if (Uid[i] == b) { self_lo = Uoff[i]; self_hi = Uoff[i + 1]; }
            for (int s0 = 0; s0 < total; s0 += kChunk) {
                const int sn = min(kChunk, total - s0);
                if (s0 > 0) sync();
                // staging: a thread's sources j, j + kNT, ... ascend, so its window leaf is searched once and then
                // advanced; two sources per round with all six loads issued before the stores
                int li = tid < sn ? find_seg(Uoff, nu, s0 + tid) : 0;
#ifdef XRL_P2P_DBG_NOSTAGE  // timing ablation only (WRONG RESULTS): stage the first chunk of the first window
                if (s0 > 0 || u0 > uptr[b]) li = -1;
#endif
                for (int j = tid; li >= 0 && j < sn; j += 2 * kNT) {
                    const int f0 = s0 + j, f1 = f0 + kNT;
                    const bool two = j + kNT < sn;
                    while (Uoff[li + 1] <= f0) ++li;
                    const int i0 = Upb[li] + (f0 - Uoff[li]);
                    const float3 d0 = Ud[li];
                    if (two)
                        while (Uoff[li + 1] <= f1) ++li;
                    const int i1 = two ? Upb[li] + (f1 - Uoff[li]) : i0;
                    const float3 d1 = Ud[li];
                    const float4 p0 = loc[i0], p1 = loc[i1];
                    const float4* q0 = reinterpret_cast<const float4*>(xq + 8 * (int64_t)i0);
                    const float4* q1 = reinterpret_cast<const float4*>(xq + 8 * (int64_t)i1);
                    const float4 a0 = q0[0], b0 = q0[1], a1 = q1[0], b1 = q1[1];
                    Sp[j] = make_float4(p0.x + d0.x, p0.y + d0.y, p0.z + d0.z, 0.f);
                    Sq[j][0] = a0;
                    Sq[j][1] = b0;
                    if (two) {
                        Sp[j + kNT] = make_float4(p1.x + d1.x, p1.y + d1.y, p1.z + d1.z, 0.f);
                        Sq[j + kNT][0] = a1;
                        Sq[j + kNT][1] = b1;
                    }
                }
                sync();
                if (act) {
                    const int a0 = max(0, min(sn, self_lo - s0)), a1 = max(0, min(sn, self_hi - s0));
                    p2p_range<false>(first_in_class(0, sg, S), a0, S, Sp, Sq, tx, ty, tz, acc);
                    p2p_range<true>(first_in_class(a0, sg, S), a1, S, Sp, Sq, tx, ty, tz, acc);
                    p2p_range<false>(first_in_class(a1, sg, S), sn, S, Sp, Sq, tx, ty, tz, acc);
                }
            }
        }
        sync();
#pragma unroll
        for (int q = 0; q < kTP2; ++q)
#pragma unroll
            for (int r = 0; r < 6; ++r) st_shared_u64(&Red[tid][q * 6 + r], acc[q][r]);
        sync();
        // reduce over the S source groups: thread handles target index ti = tid, tid + 128, ...
        for (int ti = tid; ti < T; ti += kNT) {
            const int g0 = ti / kTPT, q = (ti % kTPT) >> 1, h = ti & 1;
            float tot[6];
#pragma unroll
            for (int r = 0; r < 6; ++r) {
                float f = 0.f;
                for (int gg = 0; gg < S; ++gg) f += reinterpret_cast<const float*>(&Red[g0 + gg * NG][q * 6 + r])[h];
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
        sync();
    }
}

// Standalone P2P: one CTA (128 threads) per leaf task; tasks are taken from a global counter shared with
// the P2P warps fused into the M2L kernel (leaves[counter++]), so every owned leaf is done exactly once.
__global__ void __launch_bounds__(128) k_p2p(
    const int4* __restrict__ tasks, int ntasks, int* __restrict__ counter, const int32_t* __restrict__ level,
    const int32_t* __restrict__ ix, const int32_t* __restrict__ iy, const int32_t* __restrict__ iz,
    const int32_t* __restrict__ pb, const int32_t* __restrict__ pe, const int64_t* __restrict__ uptr,
    const int32_t* __restrict__ usrc, const float4* __restrict__ loc, const float* __restrict__ xq, float invW,
    int accumulate, int64_t n, int64_t p0, float2* __restrict__ y)
{
    extern __shared__ __align__(16) float smraw[];  // kP2PSmem: source staging, then the reduction
    __shared__ P2PWin W;
    __shared__ int task;
    if (threadIdx.x == 0) task = atomicAdd(counter, 1);
    __syncthreads();
    if (task >= ntasks) return;
    const int4 tk = tasks[task];
    p2p_leaf<128, kSrcChunk, 0>(tk.x, tk.y, tk.y + tk.z, threadIdx.x, smraw, W, level, ix, iy, iz, pb, pe, uptr, usrc, loc, xq,
                                invW, accumulate, n, p0, y);
}

// ------------------------------------------------------------------ two triples in one P2P / near pass
// xrl_mvm with nvec = 6k runs the triples in pairs: the P2P computes r and 1/r once per pair for 12 right-hand
// sides (per pair 3 FADD2/2 + FMUL2/2 + FFMA2 + 6 FFMA2 per target pair instead of twice 3 + 3: 25 % fewer
// FP32-pipe instructions per right-hand side) and the near SpMV streams its 6-byte entries once for both.
// The second triple's charges are packed into xq2; 4 targets per thread keep the accumulators at 48 registers.
constexpr int kTPT12 = 8;
constexpr int kTP212 = kTPT12 / 2;
constexpr int kSrcChunk12 = 512;
constexpr int kP2PSmem12 = (kSrcChunk12 * 20 > 128 * (kTP212 * 12 + 1) * 2 ? kSrcChunk12 * 20 : 128 * (kTP212 * 12 + 1) * 2) * 4;

template <bool kSelf>
__device__ __forceinline__ void p2p_range12(int j0, int j1, int S, const float4* __restrict__ Sp,
                                            const float4 (*__restrict__ Sq)[4], const f2x* tx, const f2x* ty,
                                            const f2x* tz, f2x (*acc)[12])
{
#pragma unroll 2
    for (int j = j0; j < j1; j += S) {
        const float4 sp = Sp[j];
        const float4 q0 = Sq[j][0], q1 = Sq[j][1], q2 = Sq[j][2], q3 = Sq[j][3];
        const f2x sx = pk2(sp.x, sp.x), sy = pk2(sp.y, sp.y), sz = pk2(sp.z, sp.z);
        const float c[12] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q2.x, q2.y, q2.z, q2.w, q3.x, q3.y};
#pragma unroll
        for (int q = 0; q < kTP212; ++q) {
            const f2x dx = sub2(tx[q], sx), dy = sub2(ty[q], sy), dz = sub2(tz[q], sz);
            const float2 r2 = upk2(fma2(dx, dx, fma2(dy, dy, mul2(dz, dz))));
            float ra = rsqrt_ftz(r2.x), rb = rsqrt_ftz(r2.y);
            if (kSelf) {
                ra = r2.x > 0.f ? ra : 0.f;
                rb = r2.y > 0.f ? rb : 0.f;
            }
            const f2x ri = pk2(ra, rb);
#pragma unroll
            for (int r = 0; r < 12; ++r) fma2_acc(acc[q][r], pk2(c[r], c[r]), ri);
        }
    }
}

// p2p_leaf for two triples: targets [tb, te) of leaf b, charges xq (triple 1) and xq2 (triple 2), results
// stored into y and y2 (each [3][n], accumulate as p2p_leaf).  128 threads, __syncthreads.
__device__ void p2p_leaf12(int b, int tb, int te, int tid, float* smraw, P2PWin& W, const int32_t* __restrict__ level,
                           const int32_t* __restrict__ ix, const int32_t* __restrict__ iy, const int32_t* __restrict__ iz,
                           const int32_t* __restrict__ pb, const int32_t* __restrict__ pe,
                           const int64_t* __restrict__ uptr, const int32_t* __restrict__ usrc,
                           const float4* __restrict__ loc, const float* __restrict__ xq, const float* __restrict__ xq2,
                           float invW, int accumulate, int64_t n, int64_t p0, float2* __restrict__ y,
                           float2* __restrict__ y2)
{
    constexpr int kNT = 128, kChunk = kSrcChunk12;
    float4* Sp = reinterpret_cast<float4*>(smraw);
    float4(*Sq)[4] = reinterpret_cast<float4(*)[4]>(smraw + 4 * kChunk);
    f2x(*Red)[kTP212 * 12 + 1] = reinterpret_cast<f2x(*)[kTP212 * 12 + 1]>(smraw);
    int* Uoff = W.Uoff;
    int* Uid = W.Uid;
    int* Upb = W.Upb;
    float3* Ud = W.Ud;
    int* wsum = W.wsum;
    const float3 cb = box_center(level[b], ix[b], iy[b], iz[b]);
    const int lane = tid & 31, warp = tid >> 5;
    for (int t0 = tb; t0 < te; t0 += kNT * kTPT12) {
        const int T = min(kNT * kTPT12, te - t0);
        const int NG = (T + kTPT12 - 1) / kTPT12;
        const int S = max(1, kNT / NG);
        const int tg = tid % NG, sg = tid / NG;
        const bool act = sg < S;
        f2x tx[kTP212], ty[kTP212], tz[kTP212];
        f2x acc[kTP212][12];
#pragma unroll
        for (int q = 0; q < kTP212; ++q) {
            float4 p[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int ti = tg * kTPT12 + 2 * q + h;
                p[h] = make_float4(1e18f, 1e18f, 1e18f, 0.f);
                if (act && ti < T) p[h] = loc[t0 + ti];
            }
            float2* tp = reinterpret_cast<float2*>(smraw) + (tid * kTP212 + q) * 3;
            tp[0] = make_float2(p[0].x, p[1].x);
            tp[1] = make_float2(p[0].y, p[1].y);
            tp[2] = make_float2(p[0].z, p[1].z);
            tx[q] = ld_shared_u64(tp);
            ty[q] = ld_shared_u64(tp + 1);
            tz[q] = ld_shared_u64(tp + 2);
#pragma unroll
            for (int r = 0; r < 12; ++r) acc[q][r] = 0ull;
        }
        for (int64_t u0 = uptr[b]; u0 < uptr[b + 1]; u0 += kUWin) {
            const int nu = (int)min((int64_t)kUWin, uptr[b + 1] - u0);
            __syncthreads();
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
                Uoff[tid + 1] = inc;
            }
            __syncthreads();
            if (tid >= 32 && tid < kUWin) Uoff[tid + 1] += wsum[0];
            if (tid == 0) Uoff[0] = 0;
            __syncthreads();
            const int total = Uoff[nu];
            int self_lo = 0, self_hi = 0;
            for (int i = 0; i < nu; ++i)
                if (Uid[i] == b) { self_lo = Uoff[i]; self_hi = Uoff[i + 1]; }
            for (int s0 = 0; s0 < total; s0 += kChunk) {
                const int sn = min(kChunk, total - s0);
                if (s0 > 0) __syncthreads();
                for (int j = tid; j < sn; j += kNT) {
                    const int f = s0 + j;
                    const int li = find_seg(Uoff, nu, f);
                    const int i = Upb[li] + (f - Uoff[li]);
                    const float3 d = Ud[li];
                    const float4 p = loc[i];
                    Sp[j] = make_float4(p.x + d.x, p.y + d.y, p.z + d.z, 0.f);
                    const float4* qa = reinterpret_cast<const float4*>(xq + 8 * (int64_t)i);
                    const float4* qb = reinterpret_cast<const float4*>(xq2 + 8 * (int64_t)i);
                    Sq[j][0] = qa[0];
                    Sq[j][1] = qa[1];
                    Sq[j][2] = qb[0];
                    Sq[j][3] = qb[1];
                }
                __syncthreads();
                if (act) {
                    const int a0 = max(0, min(sn, self_lo - s0)), a1 = max(0, min(sn, self_hi - s0));
                    p2p_range12<false>(first_in_class(0, sg, S), a0, S, Sp, Sq, tx, ty, tz, acc);
                    p2p_range12<true>(first_in_class(a0, sg, S), a1, S, Sp, Sq, tx, ty, tz, acc);
                    p2p_range12<false>(first_in_class(a1, sg, S), sn, S, Sp, Sq, tx, ty, tz, acc);
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kTP212; ++q)
#pragma unroll
            for (int r = 0; r < 12; ++r) st_shared_u64(&Red[tid][q * 12 + r], acc[q][r]);
        __syncthreads();
        for (int ti = tid; ti < T; ti += kNT) {
            const int g0 = ti / kTPT12, q = (ti % kTPT12) >> 1, h = ti & 1;
            float tot[12];
#pragma unroll
            for (int r = 0; r < 12; ++r) {
                float f = 0.f;
                for (int gg = 0; gg < S; ++gg) f += reinterpret_cast<const float*>(&Red[g0 + gg * NG][q * 12 + r])[h];
                tot[r] = f * invW;
            }
            const int64_t k = t0 + ti - p0;
            if (accumulate) {
                const float2 a = y[k], c = y[n + k], d = y[2 * n + k];
                const float2 a2 = y2[k], c2 = y2[n + k], d2 = y2[2 * n + k];
                tot[0] += a.x; tot[1] += a.y; tot[2] += c.x; tot[3] += c.y; tot[4] += d.x; tot[5] += d.y;
                tot[6] += a2.x; tot[7] += a2.y; tot[8] += c2.x; tot[9] += c2.y; tot[10] += d2.x; tot[11] += d2.y;
            }
            y[k] = make_float2(tot[0], tot[1]);
            y[n + k] = make_float2(tot[2], tot[3]);
            y[2 * n + k] = make_float2(tot[4], tot[5]);
            y2[k] = make_float2(tot[6], tot[7]);
            y2[n + k] = make_float2(tot[8], tot[9]);
            y2[2 * n + k] = make_float2(tot[10], tot[11]);
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(128) k_p2p12(
    const int4* __restrict__ tasks, int ntasks, int* __restrict__ counter, const int32_t* __restrict__ level,
    const int32_t* __restrict__ ix, const int32_t* __restrict__ iy, const int32_t* __restrict__ iz,
    const int32_t* __restrict__ pb, const int32_t* __restrict__ pe, const int64_t* __restrict__ uptr,
    const int32_t* __restrict__ usrc, const float4* __restrict__ loc, const float* __restrict__ xq,
    const float* __restrict__ xq2, float invW, int64_t n, int64_t p0, float2* __restrict__ y, float2* __restrict__ y2)
{
    extern __shared__ __align__(16) float smraw[];
    __shared__ P2PWin W;
    __shared__ int task;
    if (threadIdx.x == 0) task = atomicAdd(counter, 1);
    __syncthreads();
    if (task >= ntasks) return;
    const int4 tk = tasks[task];
    p2p_leaf12(tk.x, tk.y, tk.y + tk.z, threadIdx.x, smraw, W, level, ix, iy, iz, pb, pe, uptr, usrc, loc, xq, xq2,
               invW, 0, n, p0, y, y2);
}

// ------------------------------------------------------------------ L2P (+ M2P below)
// L2P per owned leaf (one CTA of 128 threads): the leaf's local expansion ell[r][k] (r-major) is transposed
// into shared memory as [k][8] once, then each thread evaluates panels pb + tid, pb + tid + 128, ... with
// broadcast shared-memory reads per coefficient (the panel-per-thread k_l2p re-read the k-major copy through
// L1 and was latency-bound on it: 45 % L1 hits, 0.23 ms on config 4).
__global__ void __launch_bounds__(128) k_l2p_leaf(const int32_t* __restrict__ leaves,
                                                  const int32_t* __restrict__ pb, const int32_t* __restrict__ pe,
                                                  const int32_t* __restrict__ level, const float4* __restrict__ loc,
                                                  const float* __restrict__ ell, int64_t p0, int64_t n, float invW,
                                                  float2* __restrict__ y)
{
    __shared__ __align__(16) float sl[kNC * 8];
    const int b = leaves[blockIdx.x];
    const float* src = ell + (size_t)b * kEllStride;
    for (int j = threadIdx.x; j < kNC * 8; j += blockDim.x) {
        const int k = j >> 3, r = j & 7;
        sl[j] = r < 6 ? src[r * 128 + k] : 0.f;
    }
    __syncthreads();
    const float inv_sb = ldexpf(1.f, level[b]);
    const float sc = inv_sb * invW;
    for (int64_t i = pb[b] + threadIdx.x; i < pe[b]; i += blockDim.x) {
        const float4 tp = loc[i];
        float far[6] = {0, 0, 0, 0, 0, 0};
        regular_harmonics_visit<kP>(tp.x * inv_sb, tp.y * inv_sb, tp.z * inv_sb, c_tab, [&](int k, float v) {
            const float4 a = *reinterpret_cast<const float4*>(sl + 8 * k);
            const float2 c = *reinterpret_cast<const float2*>(sl + 8 * k + 4);
            far[0] = fmaf(a.x, v, far[0]);
            far[1] = fmaf(a.y, v, far[1]);
            far[2] = fmaf(a.z, v, far[2]);
            far[3] = fmaf(a.w, v, far[3]);
            far[4] = fmaf(c.x, v, far[4]);
            far[5] = fmaf(c.y, v, far[5]);
        });
        const int64_t li = i - p0;
        red_add2(y + li, far[0] * sc, far[1] * sc);
        red_add2(y + n + li, far[2] * sc, far[3] * sc);
        red_add2(y + 2 * n + li, far[4] * sc, far[5] * sc);
    }
}

__device__ __forceinline__ void red_add_v2(float* p, float a, float b)
{
    asm volatile("red.global.add.v2.f32 [%0], {%1,%2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}

// M2P (W list, adaptive): one CTA per (owned leaf b, W box w) pair, thread per panel of b;
// y += (1/W) (1/s_w) sum_k c_k mu_w[k] It_k(u_w), accumulated with red.global.add (pairs of one leaf
// run concurrently).
__global__ void __launch_bounds__(128) k_m2p(const int2* __restrict__ wpairs, int64_t p0, int64_t n,
                                             const int32_t* __restrict__ pb, const int32_t* __restrict__ pe,
                                             const int32_t* __restrict__ level, const int32_t* __restrict__ ix,
                                             const int32_t* __restrict__ iy, const int32_t* __restrict__ iz,
                                             const float4* __restrict__ loc, const float* __restrict__ mu, float invW,
                                             float2* __restrict__ y)
{
    const int2 pr = wpairs[blockIdx.x];
    const int b = pr.x, w = pr.y;
    const float3 cb = box_center(level[b], ix[b], iy[b], iz[b]);
    const int lw = level[w];
    const float3 cw = box_center(lw, ix[w], iy[w], iz[w]);
    const float inv_sw = ldexpf(1.f, lw);
    const float* M = mu + (size_t)w * kMuStride;  // mu[r][k]
    for (int i = pb[b] + threadIdx.x; i < pe[b]; i += blockDim.x) {
        const float4 tp = loc[i];
        float a[6] = {0, 0, 0, 0, 0, 0};
        irregular_harmonics_visit<kP>((tp.x + cb.x - cw.x) * inv_sw, (tp.y + cb.y - cw.y) * inv_sw,
                                      (tp.z + cb.z - cw.z) * inv_sw, c_tab, [&](int k, float v) {
            const float hk = (degree_of(k) * degree_of(k) == k) ? v : 2.f * v;
#pragma unroll
            for (int r = 0; r < 6; ++r) a[r] = fmaf(__ldg(M + r * 128 + k), hk, a[r]);
        });
        const float sc = inv_sw * invW;
        const int64_t li = i - p0;
        red_add_v2(reinterpret_cast<float*>(y + li), a[0] * sc, a[1] * sc);
        red_add_v2(reinterpret_cast<float*>(y + n + li), a[2] * sc, a[3] * sc);
        red_add_v2(reinterpret_cast<float*>(y + 2 * n + li), a[4] * sc, a[5] * sc);
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

// zero the 768-float expansion records of the listed boxes (one CTA of 192 threads, float4 stores, per box)
__global__ void k_zero_boxes(const int32_t* __restrict__ ids, float* __restrict__ e)
{
    reinterpret_cast<float4*>(e + (size_t)ids[blockIdx.x] * kMuStride)[threadIdx.x] = make_float4(0.f, 0.f, 0.f, 0.f);
}
static void zero_boxes(xrl_ctx ctx, const xrl::DBuf<int32_t>& ids, int n, int nbox, xrl::DBuf<float>& e, cudaStream_t st)
{
    if (n == nbox) {
        XRL_CUDA(cudaMemsetAsync(e.p, 0, e.bytes(), st));
    } else if (n > 0) {
        k_zero_boxes<<<n, kMuStride / 4, 0, st>>>(ids.p, e.p);
        XRL_LAUNCH_CHECK();
        ctx->launches += 1;
    }
}

// Operators are built once per process in FP64 on the host.
const HostOperators& host_ops()
{
    static HostOperators ops;
    static std::once_flag once;
    std::call_once(once, [] { build_operators(ops); });
    return ops;
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
// T[i][k] (i, k < 121, zero padded to 128) in the tcgen05 canonical K-major
// (no swizzle) layout of a 128 (N = i) x 128 (K = k) B operand: element (i, k)
// at float ((i/8)*32 + k/4)*32 + (i%8)*4 + k%4 of its part; [offset][hi|lo][16384].
void upload_tc_images(DBuf<float>& dst, const HostOperators& ops)
{
    const size_t img = 128 * 128;
    std::vector<float> h((size_t)kNOpImg * 2 * img, 0.f);
    for (int m = 0; m < kNOpImg; ++m)
        for (int i = 0; i < kNC; ++i)
            for (int k = 0; k < kNC; ++k) {
                // images 0..315 M2L offsets, 316..323 M2M octants, 324..331 L2L octants (T[i][k], FP64)
                const double* T = m < kOpM2M ? &ops.m2l[(size_t)m * kNC * kNC]
                                : m < kOpL2L ? &ops.m2m[(size_t)(m - kOpM2M) * kNC * kNC]
                                             : &ops.l2l[(size_t)(m - kOpL2L) * kNC * kNC];
                const float a = (float)T[(size_t)i * kNC + k];
                const float hi = tf32_host(a);
                const size_t e = ((size_t)(i / 8) * 32 + k / 4) * 32 + (i % 8) * 4 + k % 4;
                h[(size_t)m * 2 * img + e] = hi;
                h[(size_t)m * 2 * img + img + e] = a - hi;
            }
    dst.alloc(h.size());
    XRL_CUDA(cudaMemcpy(dst.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
}

// M2L operator images for k_m2l_tc<true> (3xFP16): per offset o, T[i][k] * 2^opexp (one exponent for all
// offsets: the largest |entry| in [2^14, 2^15)) split into FP16 hi = rn(a), lo = rn(a - hi), in the canonical K-major layout of a 128 x 128
// 16-bit B operand: element (i, k) at half ((i/8)*16 + k/8)*64 + (i%8)*8 + k%8; [offset][hi|lo][16384].
void upload_h16_images(DBuf<uint16_t>& dst, int& opexp, const HostOperators& ops)
{
    const size_t img = 128 * 128;
    std::vector<uint16_t> h((size_t)kNM2L * 2 * img, 0);
    double mx = 0;
    for (size_t i = 0; i < (size_t)kNM2L * kNC * kNC; ++i) mx = std::max(mx, std::fabs(ops.m2l[i]));
    int e2;
    std::frexp(mx, &e2);  // mx in [2^(e2-1), 2^e2)
    opexp = 15 - e2;
    for (int m = 0; m < kNM2L; ++m) {
        const double* T = &ops.m2l[(size_t)m * kNC * kNC];
        for (int i = 0; i < kNC; ++i)
            for (int k = 0; k < kNC; ++k) {
                const double a = std::ldexp(T[(size_t)i * kNC + k], opexp);
                const __half hi = __double2half(a);
                const __half lo = __double2half(a - (double)__half2float(hi));
                const size_t e = ((size_t)(i / 8) * 16 + k / 8) * 64 + (i % 8) * 8 + k % 8;
                h[(size_t)m * 2 * img + e] = __half_as_ushort(hi);
                h[(size_t)m * 2 * img + img + e] = __half_as_ushort(lo);
            }
    }
    dst.alloc(h.size());
    XRL_CUDA(cudaMemcpy(dst.p, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
}

}  // namespace

namespace xrl {

void upload_constants(xrl_ctx ctx)
{
    RecTables<float> tab;
    fill_recurrence_tables(tab);
    XRL_CUDA(cudaMemcpyToSymbol(c_tab, &tab, sizeof(tab)));
    const HostOperators& ops = host_ops();
    upload_tc_images(ctx->ops.m2l_tc, ops);
    upload_h16_images(ctx->ops.m2l_h16, ctx->ops.m2l_hexp, ops);
    XRL_CUDA(cudaFuncSetAttribute(k_m2l_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem));
    XRL_CUDA(cudaFuncSetAttribute(k_m2l_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem));
    XRL_CUDA(cudaFuncSetAttribute(k_p2p, cudaFuncAttributeMaxDynamicSharedMemorySize, kP2PSmem));
    XRL_CUDA(cudaFuncSetAttribute(k_p2p12, cudaFuncAttributeMaxDynamicSharedMemorySize, kP2PSmem12));
    XRL_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device));
    for (int i = 0; i < 343; ++i) ctx->ops.m2l_index[i] = ops.m2l_index[i];
    XRL_CUDA(cudaFuncSetAttribute(k_p2l, cudaFuncAttributeMaxDynamicSharedMemorySize, kP2LSmem));
    XRL_CUDA(cudaFuncSetAttribute(k_p2m, cudaFuncAttributeMaxDynamicSharedMemorySize, kP2MSmem));
}

}  // namespace xrl

// All M2M levels (bottom-up) or all L2L levels (top-down) in one launch of the tensor-core translation
// kernel: the pass's blocks are balanced per level over one persistent grid and the CTAs meet at a grid
// barrier between levels (TransPass, tree.cu); src/dst are r-major expansion arrays.
static void translate_pass(xrl_tree t, xrl::TransPass& P, const float* src, float* dst, cudaStream_t st)
{
    if (P.nblocks <= 0 || P.nlev <= 0) return;
    xrl_ctx ctx = t->ctx;
    XRL_CUDA(cudaMemsetAsync(P.done.p, 0, sizeof(int) * P.nlev, st));
    k_m2l_tc<false><<<P.grid, kTcThreads, kTcSmem, st>>>(t->tr_blocks.p + P.first, P.nblocks, t->tr_tiles.p,
                                                         t->tr_tgt.p, t->tr_src.p, ctx->ops.m2l_tc.p, src, dst, 0,
                                                         P2PTasks{}, P.rows.p, P.done.p, P.nlev, nullptr, 0);
    XRL_LAUNCH_CHECK();
    ctx->launches += 1;
}

// ------------------------------------------------------------------ the MVM, phase by phase
// One triple (6 real RHS) through the tree.  Phases (each enqueued, none blocking):
//   begin  -> pack the owned charges -> [halo of x]                            (work stream)
//   side   -> P2P, then the near SpMV unless it waits for the fused P2P       (side stream)
//   up     -> P2M (own leaves), M2M -> [shared-box all-reduce, LET]          (work stream)
//   down   -> M2L (+ fused P2P warps), near, P2L, L2L, L2P, M2P, join       (work stream)
// [..]: only on a partitioned tree; the exchanges run over NCCL (xrl_mvm) or as device copies between
// the trees of one process (xrl_mvm_vranks).  Single-rank trees own every panel and exchange nothing.
struct Mvm {
    xrl_tree t;
    xrl_near nr;
    float2* y;
    uint32_t flags;
    int sched;
    cudaStream_t st, side;
    bool do_far, do_near, chain, fuse, side_done;
    bool near_first = false;  // side stream: near SpMV (into zeroed y) before the P2P, which then accumulates
    int64_t nl, p0;
    float invW;
    cudaEvent_t halo = nullptr;  // multi-rank, overlapped halo: the P2P / P2L wait for it
    bool p2l_early = false;      // the P2L ran on the comm stream during the up pass (L2L waits for ev_p2l)
    float* xq = nullptr;         // this triple's packed charges (t->xq, or t->xq2 for the second of a pair)
    const float* xq2 = nullptr;  // pair mode (first triple): the second triple's charges; the side stream's
    float2* y2 = nullptr;        //   P2P / near SpMV serve both triples and also write y2
};

static Mvm mvm_make(xrl_tree t, xrl_near nr, float2* y, uint32_t flags, int sched)
{
    xrl_ctx ctx = t->ctx;
    Mvm M;
    M.t = t;
    M.nr = nr;
    M.y = y;
    M.flags = flags;
    M.sched = sched;
    M.st = sched ? ctx->work : ctx->stream;
    M.side = sched ? ctx->side : ctx->stream;
    M.do_far = flags != XRL_MVM_NEAR_ONLY;
    M.do_near = flags != XRL_MVM_FAR_ONLY;
    M.chain = M.do_far && t->nlevel > 1;
    // the fused P2P warps pay off when the M2L is long and L2-bound (whole meshes, 2-way shards); on a rank's
    // share of an 8-way partition the M2L is short and the warps only stretch it (projection: 5.77x fused vs
    // 5.9x unfused at 8 ranks of config 4)
    static const int fuse_max_world = [] {  // XRL_FUSE_MAXWORLD (tuning): largest partition that fuses
        const char* e = std::getenv("XRL_FUSE_MAXWORLD");
        return e ? std::atoi(e) : 2;
    }();
    M.fuse = sched != 0 && ctx->fuse_p2p && M.chain && t->n_m2l_tiles > 0 && t->n_own_leaves > 0 &&
             t->part_world <= fuse_max_world;
    M.side_done = false;
    static const bool near_first_env = [] {  // XRL_NEAR_FIRST=1 (schedule experiment)
        const char* e = std::getenv("XRL_NEAR_FIRST");
        return e && e[0] == '1';
    }();
    M.near_first = near_first_env && sched != 0 && M.do_far && M.do_near;
    M.nl = t->p1 - t->p0;
    M.p0 = t->p0;
    M.invW = (float)(1.0 / t->W);
    M.xq = t->xq.p;
    return M;
}

// x: this rank's slice [3][n_local] (the whole vector on a single-rank tree)
static void mvm_begin(Mvm& M, const float2* x)
{
    xrl_tree t = M.t;
    xrl_ctx ctx = t->ctx;
    if (M.sched) {
        XRL_CUDA(cudaEventRecord(ctx->ev_work, ctx->stream));
        XRL_CUDA(cudaStreamWaitEvent(M.st, ctx->ev_work, 0));
    }
    cudaEvent_t ev;
    phase_begin(ctx, PH_PACK, &ev, M.st);
    if (M.nl > 0) {
        k_pack<<<nblk(M.nl, 256), 256, 0, M.st>>>(M.nl, x, M.xq + 8 * M.p0);
        XRL_LAUNCH_CHECK();
        ctx->launches += 1;
    }
    phase_end(ctx, PH_PACK, ev, M.st);
    XRL_CUDA(cudaMemsetAsync(t->p2p_counter.p, 0, sizeof(int), M.st));  // P2P leaf tasks (before the fork)
}

// halo of x, step 1: pack the records peers read (work stream unless given)
static void halo_pack(Mvm& M, cudaStream_t st = nullptr)
{
    xrl_near N = M.nr;
    gather_records(N->halo_soff.back(), 8, N->halo_sidx.p, M.t->xq.p, N->halo_sbuf.p, st ? st : M.st);
    M.t->ctx->launches += N->halo_soff.back() > 0;
}
// step 3 (after the transport): scatter the received records into the charges
static void halo_unpack(Mvm& M, cudaStream_t st = nullptr)
{
    xrl_near N = M.nr;
    scatter_records(N->halo_roff.back(), 8, N->halo_ridx.p, N->halo_rbuf.p, M.t->xq.p, st ? st : M.st);
    M.t->ctx->launches += N->halo_roff.back() > 0;
}

static void launch_near(Mvm& M)
{
    xrl_tree t = M.t;
    xrl_ctx ctx = t->ctx;
    xrl_near nr = M.nr;
    cudaEvent_t ev;
    if (M.do_near) {
        phase_begin(ctx, PH_NEAR, &ev, M.side);
        // the SpMV adds into y: in the near-only mode it starts from zero
        if (!M.do_far && M.nl > 0) XRL_CUDA(cudaMemsetAsync(M.y, 0, sizeof(float2) * 3 * (size_t)M.nl, M.side));
        if (!M.do_far && M.nl > 0 && M.y2) XRL_CUDA(cudaMemsetAsync(M.y2, 0, sizeof(float2) * 3 * (size_t)M.nl, M.side));
        if (nr->n_segs > 0) {
            // persistent: XRL_NEAR_MINB (2) CTAs of 256 per SM, each a slot-balanced range of segments
            const int grid = (int)std::min<int64_t>(nblk(8 * nr->n_segs, XRL_NEAR_NT),
                                                    (M.xq2 ? 512 / XRL_NEAR_NT : XRL_NEAR_MINB) * ctx->num_sms);
            if (M.xq2)
                k_near_rg<2><<<grid, XRL_NEAR_NT, 0, M.side>>>(nr->n_segs, nr->seg_grp.p, nr->seg_base.p, nr->seg_off.p,
                                                              nr->gval.p, nr->eoff.p, M.xq, M.xq2, M.nl, M.y, M.y2);
            else
                k_near_rg<1><<<grid, XRL_NEAR_NT, 0, M.side>>>(nr->n_segs, nr->seg_grp.p, nr->seg_base.p, nr->seg_off.p,
                                                              nr->gval.p, nr->eoff.p, t->xq.p, nullptr, M.nl, M.y, nullptr);
            XRL_LAUNCH_CHECK();
            ctx->launches += 1;
        }
        phase_end(ctx, PH_NEAR, ev, M.side);
    }
    XRL_CUDA(cudaEventRecord(ctx->ev_join, M.side));
}

// fork the side stream: the P2P (FP32-bound; shares SMs well with the tensor-core M2L), then the near
// SpMV unless it must wait for the P2P tasks fused into the M2L kernel
static void mvm_side(Mvm& M)
{
    xrl_tree t = M.t;
    xrl_ctx ctx = t->ctx;
    cudaEvent_t ev;
    M.side_done = true;
    XRL_CUDA(cudaEventRecord(ctx->ev_fork, M.st));
    XRL_CUDA(cudaStreamWaitEvent(M.side, ctx->ev_fork, 0));
    if (M.halo) XRL_CUDA(cudaStreamWaitEvent(M.side, M.halo, 0));  // the P2P reads remote charges
    const bool nf = M.near_first && !M.xq2;
    if (nf) {  // y = 0, y += N x, then the P2P adds its part
        if (M.nl > 0) XRL_CUDA(cudaMemsetAsync(M.y, 0, sizeof(float2) * 3 * (size_t)M.nl, M.side));
        launch_near(M);
        XRL_CUDA(cudaEventRecord(ctx->ev_near, M.side));
    }
    if (M.do_far) {
        phase_begin(ctx, PH_P2P, &ev, M.side);
        if (t->n_own_leaves > 0 && M.xq2) {
            k_p2p12<<<t->n_p2p_tasks, 128, kP2PSmem12, M.side>>>(t->p2p_tasks.p, t->n_p2p_tasks, t->p2p_counter.p,
                                                                t->blevel.p, t->bix.p, t->biy.p, t->biz.p, t->bpb.p,
                                                                t->bpe.p, t->u_ptr.p, t->u_src.p, t->loc.p, M.xq,
                                                                M.xq2, M.invW, M.nl, M.p0, M.y, M.y2);
            XRL_LAUNCH_CHECK();
            ctx->launches += 1;
        } else if (t->n_own_leaves > 0) {
            k_p2p<<<t->n_p2p_tasks, 128, kP2PSmem, M.side>>>(t->p2p_tasks.p, t->n_p2p_tasks, t->p2p_counter.p,
                                                            t->blevel.p, t->bix.p, t->biy.p, t->biz.p, t->bpb.p,
                                                            t->bpe.p, t->u_ptr.p, t->u_src.p, t->loc.p, M.xq,
                                                            M.invW, nf ? 1 : 0, M.nl, M.p0, M.y);
            XRL_LAUNCH_CHECK();
            ctx->launches += 1;
        }
        phase_end(ctx, PH_P2P, ev, M.side);
    }
    XRL_CUDA(cudaEventRecord(ctx->ev_p2p, M.side));  // y holds the P2P part: the L2P may add to it
    if (nf) XRL_CUDA(cudaEventRecord(ctx->ev_join, M.side));
    else if (!M.fuse) launch_near(M);
}

static void launch_p2l(Mvm& M, cudaStream_t st)
{
    xrl_tree t = M.t;
    xrl_ctx ctx = t->ctx;
    cudaEvent_t ev;
    phase_begin(ctx, PH_P2L, &ev, st);
    if (t->n_x_targets > 0) {
        k_p2l<<<t->n_x_targets, 128, kP2LSmem, st>>>(t->x_targets.p, t->x_ptr.p, t->x_src.p, t->blevel.p, t->bix.p,
                                                     t->biy.p, t->biz.p, t->bpb.p, t->bpe.p, t->loc.p, M.xq, t->ell.p);
        XRL_LAUNCH_CHECK();
        ctx->launches += 1;
    }
    phase_end(ctx, PH_P2L, ev, st);
}

// upward pass: P2M of the own leaves, M2M of the relevant boxes.  In the forked schedules the local
// expansions are zeroed here and the P2L (X list: a few, latency-bound CTAs) runs on the comm stream beside the
// up pass instead of between the M2L and the L2L; it adds into ell atomically, the L2L waits for it.
static void mvm_up(Mvm& M)
{
    xrl_tree t = M.t;
    xrl_ctx ctx = t->ctx;
    if (!M.chain) return;
    cudaEvent_t ev;
    if (M.sched != XRL_SCHED_SERIAL && ctx->comm && ctx->ev_p2l) {
        zero_boxes(ctx, t->ell_zero, t->n_ell_zero, t->nbox, t->ell, M.st);
        XRL_CUDA(cudaEventRecord(ctx->ev_p2l, M.st));
        XRL_CUDA(cudaStreamWaitEvent(ctx->comm, ctx->ev_p2l, 0));  // (the halo, if any, is already on comm)
        launch_p2l(M, ctx->comm);
        XRL_CUDA(cudaEventRecord(ctx->ev_p2l, ctx->comm));
        M.p2l_early = true;
    }
    phase_begin(ctx, PH_P2M, &ev, M.st);
    zero_boxes(ctx, t->mu_zero, t->n_mu_zero, t->nbox, t->mu, M.st);  // parents accumulate the M2M reductions
    if (t->n_own_leaves > 0) {
        k_p2m<<<t->n_own_leaves, 128, kP2MSmem, M.st>>>(t->own_leaves.p, t->bpb.p, t->bpe.p, t->blevel.p, t->loc.p,
                                                         M.xq, t->mu.p);
        XRL_LAUNCH_CHECK();
        ctx->launches += 1;
    }
    phase_end(ctx, PH_P2M, ev, M.st);
    phase_begin(ctx, PH_M2M, &ev, M.st);
    translate_pass(t, t->m2m_pass, t->mu.p, t->mu.p, M.st);
    phase_end(ctx, PH_M2M, ev, M.st);
}

// multipole exchange, step 1: pack the shared boxes' partial multipoles and the LET boxes peers need
static void mu_pack(Mvm& M)
{
    xrl_tree t = M.t;
    gather_records((int64_t)t->shared_boxes.size(), kMuStride, t->sh_idx.p, t->mu.p, t->sh_buf.p, M.st);
    t->ctx->launches += !t->shared_boxes.empty();
}
// step 2 (after the shared all-reduce): full multipoles of the shared boxes back into mu; pack the LET
static void mu_shared_unpack_let_pack(Mvm& M)
{
    xrl_tree t = M.t;
    scatter_records((int64_t)t->shared_boxes.size(), kMuStride, t->sh_idx.p, t->sh_buf.p, t->mu.p, M.st);
    gather_records(t->let_soff.back(), kMuStride, t->let_sidx.p, t->mu.p, t->let_sbuf.p, M.st);
    t->ctx->launches += !t->shared_boxes.empty() + (t->let_soff.back() > 0);
}
// step 3 (after the LET transport): the received multipoles into mu
static void let_unpack(Mvm& M)
{
    xrl_tree t = M.t;
    scatter_records(t->let_roff.back(), kMuStride, t->let_ridx.p, t->let_rbuf.p, t->mu.p, M.st);
    t->ctx->launches += t->let_roff.back() > 0;
}

// downward pass and the join
static void mvm_down(Mvm& M)
{
    xrl_tree t = M.t;
    xrl_ctx ctx = t->ctx;
    cudaEvent_t ev;
#ifdef XRL_PROFILING_ABLATION
    // XRL_M2L_DBG (profiling ablations, WRONG RESULTS; only in a library built with
    // -DXRL_PROFILING_ABLATION): 1 skip reductions, 2 skip A loads, 4 skip D reads
    static const int m2l_dbg = [] {
        const char* e = getenv("XRL_M2L_DBG");
        const int v = e ? atoi(e) : 0;
        if (v) fprintf(stderr, "xrl: XRL_M2L_DBG=%d -- M2L ablation active, MVM results are wrong\n", v);
        return v;
    }();
#else
    constexpr int m2l_dbg = 0;  // the shipped library has no ablation switch
#endif
    if (M.chain) {
        if (!M.p2l_early) zero_boxes(ctx, t->ell_zero, t->n_ell_zero, t->nbox, t->ell, M.st);
        if (!M.side_done) mvm_side(M);  // XRL_SCHED_LATE, or the virtual-rank driver
        phase_begin(ctx, PH_M2L, &ev, M.st);
        if (t->n_m2l_tiles > 0) {
            const int grid = t->m2l_grid;  // the grid the block order was balanced for (tree.cu)
            P2PTasks tasks{};
            if (M.fuse && M.near_first && !M.xq2)  // the fused warps add to y after the near SpMV
                XRL_CUDA(cudaStreamWaitEvent(M.st, ctx->ev_near, 0));
            if (M.fuse)
                tasks = P2PTasks{t->p2p_tasks.p, t->n_p2p_tasks, t->p2p_counter.p, t->blevel.p, t->bix.p, t->biy.p,
                                 t->biz.p, t->bpb.p, t->bpe.p, t->u_ptr.p, t->u_src.p, t->loc.p, M.xq, M.invW, M.nl,
                                 M.p0, M.y, M.near_first ? 1 : 0};
            if (ctx->m2l_h16) {  // 3xFP16 (default): the multipole row exponents first
                if (t->mu_max.n < 1) t->mu_max.alloc(1);
                XRL_CUDA(cudaMemsetAsync(t->mu_max.p, 0, sizeof(unsigned), M.st));
                k_mu_max<<<(t->nbox + 7) / 8, 256, 0, M.st>>>(t->nbox, t->mu.p, t->mu_max.p);
                XRL_LAUNCH_CHECK();
                k_m2l_tc<true><<<grid, kTcThreads, kTcSmem, M.st>>>(t->m2l_blocks.p, t->n_m2l_blocks, t->m2l_tiles.p,
                                                                    t->m2l_tgt.p, t->m2l_srcb.p, ctx->ops.m2l_h16.p,
                                                                    t->mu.p, t->ell.p, m2l_dbg, tasks, nullptr, nullptr,
                                                                    0, t->mu_max.p, ctx->ops.m2l_hexp);
                XRL_LAUNCH_CHECK();
                ctx->launches += 2;
            } else {
                k_m2l_tc<false><<<grid, kTcThreads, kTcSmem, M.st>>>(t->m2l_blocks.p, t->n_m2l_blocks, t->m2l_tiles.p,
                                                                     t->m2l_tgt.p, t->m2l_srcb.p, ctx->ops.m2l_tc.p,
                                                                     t->mu.p, t->ell.p, m2l_dbg, tasks, nullptr,
                                                                     nullptr, 0, nullptr, 0);
                XRL_LAUNCH_CHECK();
                ctx->launches += 1;
            }
        }
        phase_end(ctx, PH_M2L, ev, M.st);
        if (M.fuse && !(M.near_first && !M.xq2)) {
            XRL_CUDA(cudaEventRecord(ctx->ev_m2l, M.st));
            XRL_CUDA(cudaStreamWaitEvent(M.side, ctx->ev_m2l, 0));  // fused P2P tasks done
            launch_near(M);
        }
        if (M.p2l_early) {
            XRL_CUDA(cudaStreamWaitEvent(M.st, ctx->ev_p2l, 0));
        } else {
            if (M.halo) XRL_CUDA(cudaStreamWaitEvent(M.st, M.halo, 0));  // the P2L reads remote leaves' charges
            launch_p2l(M, M.st);
        }
        phase_begin(ctx, PH_L2L, &ev, M.st);
        translate_pass(t, t->l2l_pass, t->ell.p, t->ell.p, M.st);
        phase_end(ctx, PH_L2L, ev, M.st);
    } else if (!M.side_done) {
        mvm_side(M);
    }
    // after the P2P wrote y, the local-expansion / W-list evaluation adds to it (vector L2 reductions, so it
    // may overlap the near SpMV, which adds the same way); join the side stream at the end
    if (M.sched) XRL_CUDA(cudaStreamWaitEvent(M.st, ctx->ev_p2p, 0));
    if (M.chain && M.nl > 0) {
        phase_begin(ctx, PH_L2P, &ev, M.st);
        if (t->n_own_leaves > 0) {
            k_l2p_leaf<<<t->n_own_leaves, 128, 0, M.st>>>(t->own_leaves.p, t->bpb.p, t->bpe.p, t->blevel.p, t->loc.p,
                                                        t->ell.p, M.p0, M.nl, M.invW, M.y);
            XRL_LAUNCH_CHECK();
            ctx->launches += 1;
        }
        if (t->n_w_targets > 0) {
            k_m2p<<<t->n_w_targets, 128, 0, M.st>>>(t->w_targets.p, M.p0, M.nl, t->bpb.p, t->bpe.p, t->blevel.p,
                                                    t->bix.p, t->biy.p, t->biz.p, t->loc.p, t->mu.p, M.invW, M.y);
            XRL_LAUNCH_CHECK();
            ctx->launches += 1;
        }
        phase_end(ctx, PH_L2P, ev, M.st);
    }
    if (M.sched) {  // join the side stream, then the work stream back into the caller's stream
        XRL_CUDA(cudaStreamWaitEvent(M.st, ctx->ev_join, 0));
        XRL_CUDA(cudaEventRecord(ctx->ev_work, M.st));
        XRL_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_work, 0));
    }
}

// One triple on this process's tree: x this rank's slice [3][n_local], y the same.  On a partitioned
// multi-rank tree the exchanges run over NCCL between the phases.  transports = false (the virtual-rank
// timing pass): the same phases, streams and overlap with the three transports left out.
static xrl_status mvm_triple(xrl_tree t, xrl_near nr, const float2* x, float2* y, uint32_t flags,
                             bool transports = true)
{
    xrl_ctx ctx = t->ctx;
    Mvm M = mvm_make(t, nr, y, flags, ctx->sched);
    const bool dist = t->part_world > 1;
    mvm_begin(M, x);
    // the NCCL exchanges run on the library's comm stream (one stream, so every rank issues them in the same
    // order): the halo of x overlaps the up pass, which reads only the rank's own charges
    const bool overlap = dist && M.sched != XRL_SCHED_SERIAL && ctx->comm;
    cudaStream_t cs = overlap ? ctx->comm : M.st;
    if (dist) {
        if (overlap) {
            XRL_CUDA(cudaEventRecord(ctx->ev_comm, M.st));
            XRL_CUDA(cudaStreamWaitEvent(cs, ctx->ev_comm, 0));
        }
        halo_pack(M, cs);
        if (transports) {
            xrl_status s = nccl_exchange(ctx, nr->halo_sbuf.p, nr->halo_soff, nr->halo_rbuf.p, nr->halo_roff, 8, cs);
            if (s) return s;
        }
        halo_unpack(M, cs);
        if (overlap) {
            XRL_CUDA(cudaEventRecord(ctx->ev_halo, cs));
            M.halo = ctx->ev_halo;
        }
    }
    if (M.sched != XRL_SCHED_LATE || !M.chain) mvm_side(M);
    mvm_up(M);
    if (dist && M.chain) {
        mu_pack(M);
        if (overlap) {
            XRL_CUDA(cudaEventRecord(ctx->ev_comm, M.st));
            XRL_CUDA(cudaStreamWaitEvent(cs, ctx->ev_comm, 0));
        }
        if (transports) {
            xrl_status s = nccl_allreduce_sum(ctx, t->sh_buf.p, t->shared_boxes.size() * (size_t)kMuStride, cs);
            if (s) return s;
        }
        if (overlap) {
            XRL_CUDA(cudaEventRecord(ctx->ev_comm, cs));
            XRL_CUDA(cudaStreamWaitEvent(M.st, ctx->ev_comm, 0));
        }
        mu_shared_unpack_let_pack(M);
        if (overlap) {
            XRL_CUDA(cudaEventRecord(ctx->ev_comm, M.st));
            XRL_CUDA(cudaStreamWaitEvent(cs, ctx->ev_comm, 0));
        }
        if (transports) {
            xrl_status s = nccl_exchange(ctx, t->let_sbuf.p, t->let_soff, t->let_rbuf.p, t->let_roff, kMuStride, cs);
            if (s) return s;
        }
        if (overlap) {
            XRL_CUDA(cudaEventRecord(ctx->ev_comm, cs));
            XRL_CUDA(cudaStreamWaitEvent(M.st, ctx->ev_comm, 0));
        }
        let_unpack(M);
    }
    mvm_down(M);
    if (overlap) XRL_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_halo, 0));  // (already implied; explicit join)
    return XRL_OK;
}

// Two triples of a single-rank tree: the side stream's P2P and near SpMV serve both (k_p2p12, k_near_rg<2>:
// one pass over the U lists and the near entries for 12 right-hand sides); the FMM expansions (mu, ell: one
// triple's worth of tree scratch) run for the first triple, then for the second, on the work stream.
static void mvm_pair(xrl_tree t, xrl_near nr, const float2* xa, float2* ya, const float2* xb, float2* yb,
                     uint32_t flags)
{
    xrl_ctx ctx = t->ctx;
    if (t->xq2.n < t->xq.n) {
        t->xq2.alloc(t->xq.n);
        XRL_CUDA(cudaMemsetAsync(t->xq2.p, 0, t->xq2.bytes(), ctx->stream));
    }
    Mvm A = mvm_make(t, nr, ya, flags, ctx->sched);
    A.xq2 = t->xq2.p;
    A.y2 = yb;
    A.fuse = false;
    mvm_begin(A, xa);
    if (A.nl > 0) {
        k_pack<<<nblk(A.nl, 256), 256, 0, A.st>>>(A.nl, xb, t->xq2.p + 8 * A.p0);
        XRL_LAUNCH_CHECK();
        ctx->launches += 1;
    }
    if (A.sched != XRL_SCHED_LATE || !A.chain) mvm_side(A);
    mvm_up(A);
    mvm_down(A);
    Mvm B = mvm_make(t, nr, yb, flags, ctx->sched);
    B.xq = t->xq2.p;
    B.fuse = false;
    B.side_done = true;  // its P2P / near ran with A's (ev_p2p, ev_join still mark them)
    if (B.sched) {
        XRL_CUDA(cudaEventRecord(ctx->ev_work, ctx->stream));
        XRL_CUDA(cudaStreamWaitEvent(B.st, ctx->ev_work, 0));
    }
    mvm_up(B);
    mvm_down(B);
}

static bool pair_enabled()
{
    static const bool on = [] {
        const char* e = std::getenv("XRL_PAIR");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Per-rank device times of the virtual-rank driver (events on the context stream, serial schedule).
struct VTimer {
    xrl_ctx ctx;
    bool on;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;  // (slot, (begin, end))
    cudaEvent_t b = nullptr;
    void begin()
    {
        if (!on) return;
        XRL_CUDA(cudaEventCreate(&b));
        XRL_CUDA(cudaEventRecord(b, ctx->stream));
    }
    void end(int slot)
    {
        if (!on) return;
        cudaEvent_t e;
        XRL_CUDA(cudaEventCreate(&e));
        XRL_CUDA(cudaEventRecord(e, ctx->stream));
        ev.push_back({slot, {b, e}});
    }
    void collect(double* ms)
    {
        if (!on) return;
        XRL_CUDA(cudaStreamSynchronize(ctx->stream));
        for (auto& p : ev) {
            float v = 0.f;
            XRL_CUDA(cudaEventElapsedTime(&v, p.second.first, p.second.second));
            ms[p.first] += v;
            cudaEventDestroy(p.second.first);
            cudaEventDestroy(p.second.second);
        }
        ev.clear();
    }
};

// Device-copy transport of one exchange between the k trees of a virtual-rank run: rank q's send
// segment for r -> rank r's receive segment from q.
template <typename SOff, typename ROff, typename SBuf, typename RBuf>
static xrl_status vcopy(int k, const std::vector<Mvm>& Ms, SOff soff, ROff roff, SBuf sbuf, RBuf rbuf, int w,
                        cudaStream_t st)
{
    for (int r = 0; r < k; ++r)
        for (int q = 0; q < k; ++q) {
            if (q == r) continue;
            const std::vector<int64_t>& so = soff(Ms[q]);
            const std::vector<int64_t>& ro = roff(Ms[r]);
            const int64_t cnt = so[r + 1] - so[r];
            if (cnt != ro[q + 1] - ro[q]) {
                set_error("xrl_mvm_vranks: exchange plans of ranks %d and %d disagree", q, r);
                return XRL_EINVAL;
            }
            if (cnt > 0)
                XRL_CUDA(cudaMemcpyAsync(rbuf(Ms[r]) + ro[q] * w, sbuf(Ms[q]) + so[r] * w, sizeof(float) * cnt * w,
                                         cudaMemcpyDeviceToDevice, st));
        }
    return XRL_OK;
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
    if (t->part_world > 1 && t->ctx->world == 1) {
        set_error("xrl_mvm: a partitioned tree on a single-rank context (virtual rank) runs through xrl_mvm_vranks");
        return XRL_EUNSUPPORTED;
    }
    try {
        XRL_CUDA(cudaSetDevice(t->ctx->device));
        const int64_t nl = t->p1 - t->p0;
        for (int v = 0; v < nvec;) {
            const float2* xv = (const float2*)x + (size_t)v * nl;
            float2* yv = (float2*)y + (size_t)v * nl;
            if (nvec - v >= 6 && t->part_world == 1 && pair_enabled()) {
                mvm_pair(t, nr, xv, yv, xv + 3 * nl, yv + 3 * nl, flags);
                v += 6;
                continue;
            }
            xrl_status s = mvm_triple(t, nr, xv, yv, flags);
            if (s) return s;
            v += 3;
        }
        return XRL_OK;
    } catch (const CudaError& e) {
        return e.code;
    }
}

xrl_status xrl_mvm_vranks(int32_t k, const xrl_tree* trees, const xrl_near* nears, const void* const* x,
                          void* const* y, int32_t nvec, uint32_t flags, double* rank_ms, double* exch_ms)
{
    if (k < 1 || !trees || !nears || !x || !y) { set_error("xrl_mvm_vranks: bad argument"); return XRL_EINVAL; }
    if (nvec < 3 || nvec % 3) { set_error("xrl_mvm_vranks: nvec=%d must be a positive multiple of 3", nvec); return XRL_EDIM; }
    if (flags > XRL_MVM_FAR_ONLY) { set_error("xrl_mvm_vranks: bad flags"); return XRL_EINVAL; }
    for (int r = 0; r < k; ++r) {
        if (!trees[r] || !nears[r] || !x[r] || !y[r]) { set_error("xrl_mvm_vranks: null handle or vector %d", r); return XRL_EINVAL; }
        if (nears[r]->tree != trees[r]) { set_error("xrl_mvm_vranks: near %d built from another tree", r); return XRL_EPROVENANCE; }
        if (trees[r]->ctx != trees[0]->ctx || trees[r]->ctx->world != 1) {
            set_error("xrl_mvm_vranks: all trees must share one single-rank context");
            return XRL_EPROVENANCE;
        }
        if (trees[r]->part_world != (k > 1 ? k : 1) || trees[r]->part_rank != (k > 1 ? r : 0) || trees[r]->n != trees[0]->n) {
            set_error("xrl_mvm_vranks: tree %d is not rank %d of a %d-way partition of one mesh", r, r, k);
            return XRL_EINVAL;
        }
        if (x[r] == y[r] || (((uintptr_t)x[r] | (uintptr_t)y[r]) & 15)) {
            set_error("xrl_mvm_vranks: vectors of rank %d alias or are not 16-byte aligned", r);
            return XRL_EINVAL;
        }
    }
    xrl_ctx ctx = trees[0]->ctx;
    try {
        XRL_CUDA(cudaSetDevice(ctx->device));
        if (rank_ms) for (int r = 0; r < k; ++r) rank_ms[r] = 0;
        if (exch_ms) *exch_ms = 0;
        // The ranks' phase groups run one after the other with the context's schedule (default: the forked /
        // fused one a real rank uses); each group forks from and joins back into the context stream, so its
        // events there bracket that rank's work alone on the GPU.  The exchanges are device copies on the
        // context stream between the groups.
        const int sched = ctx->sched;
        auto fork = [&]() {
            if (!sched) return;
            XRL_CUDA(cudaEventRecord(ctx->ev_work, ctx->stream));
            XRL_CUDA(cudaStreamWaitEvent(ctx->work, ctx->ev_work, 0));
        };
        auto join = [&]() {
            if (!sched) return;
            XRL_CUDA(cudaEventRecord(ctx->ev_work, ctx->work));
            XRL_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_work, 0));
        };
        VTimer tm{ctx, exch_ms != nullptr || (rank_ms && k == 1)};
        std::vector<double> ms(k + 1, 0.0);
        cudaStream_t st = ctx->stream;
        xrl_status s = XRL_OK;
        if (rank_ms && k > 1) {
            // timing pass (before the real one, whose results it does not touch): each rank's whole MVM alone on
            // the GPU in the production order -- pack, halo unpack, P2P forked early onto the side stream, up
            // pass, multipole unpack/pack, down pass -- with the three transports left out (their receive
            // buffers hold whatever the previous call left: the work is data-independent); the transports are
            // timed in the real pass (exch_ms) and modelled over NVLink by the projection
            VTimer rt{ctx, true};
            for (int r = 0; r < k; ++r) {
                rt.begin();
                s = mvm_triple(trees[r], nears[r], (const float2*)x[r], (float2*)y[r], flags, false);
                rt.end(r);
                if (s) return s;
            }
            std::vector<double> rms(k + 1, 0.0);
            rt.collect(rms.data());
            for (int r = 0; r < k; ++r) rank_ms[r] = rms[r] * (nvec / 3);
        }
        for (int v = 0; v < nvec && !s; v += 3) {
            std::vector<Mvm> Ms;
            for (int r = 0; r < k; ++r) {
                const int64_t nl = trees[r]->p1 - trees[r]->p0;
                Ms.push_back(mvm_make(trees[r], nears[r], (float2*)y[r] + (size_t)v * nl, flags,
                                      sched == XRL_SCHED_LATE ? XRL_SCHED_FORK : sched));
            }
            const bool dist = k > 1;
            for (int r = 0; r < k; ++r) {
                const int64_t nl = trees[r]->p1 - trees[r]->p0;
                tm.begin();
                mvm_begin(Ms[r], (const float2*)x[r] + (size_t)v * nl);  // (forks the work stream)
                if (dist) halo_pack(Ms[r]);
                join();
                tm.end(r);
            }
            if (dist) {
                tm.begin();
                s = vcopy(k, Ms, [](const Mvm& M) -> const std::vector<int64_t>& { return M.nr->halo_soff; },
                          [](const Mvm& M) -> const std::vector<int64_t>& { return M.nr->halo_roff; },
                          [](const Mvm& M) -> const float* { return M.nr->halo_sbuf.p; },
                          [](const Mvm& M) -> float* { return M.nr->halo_rbuf.p; }, 8, st);
                tm.end(k);
                if (s) break;
            }
            for (int r = 0; r < k; ++r) {
                tm.begin();
                fork();
                if (dist) halo_unpack(Ms[r]);
                mvm_up(Ms[r]);
                if (dist && Ms[r].chain) mu_pack(Ms[r]);
                join();
                tm.end(r);
            }
            if (dist && Ms[0].chain) {
                // all-reduce of the shared boxes: sum into rank 0's buffer, copy back to every rank
                tm.begin();
                const size_t cnt = trees[0]->shared_boxes.size() * (size_t)kMuStride;
                for (int r = 1; r < k; ++r) {
                    if (trees[r]->shared_boxes != trees[0]->shared_boxes) { set_error("xrl_mvm_vranks: shared boxes differ"); s = XRL_EINVAL; break; }
                    add_into((int64_t)cnt, trees[r]->sh_buf.p, trees[0]->sh_buf.p, st);
                }
                for (int r = 1; r < k && !s; ++r)
                    if (cnt) XRL_CUDA(cudaMemcpyAsync(trees[r]->sh_buf.p, trees[0]->sh_buf.p, 4 * cnt, cudaMemcpyDeviceToDevice, st));
                tm.end(k);
                if (s) break;
                for (int r = 0; r < k; ++r) {
                    tm.begin();
                    fork();
                    mu_shared_unpack_let_pack(Ms[r]);
                    join();
                    tm.end(r);
                }
                tm.begin();
                s = vcopy(k, Ms, [](const Mvm& M) -> const std::vector<int64_t>& { return M.t->let_soff; },
                          [](const Mvm& M) -> const std::vector<int64_t>& { return M.t->let_roff; },
                          [](const Mvm& M) -> const float* { return M.t->let_sbuf.p; },
                          [](const Mvm& M) -> float* { return M.t->let_rbuf.p; }, kMuStride, st);
                tm.end(k);
                if (s) break;
            }
            for (int r = 0; r < k; ++r) {
                tm.begin();
                fork();
                if (dist && Ms[r].chain) let_unpack(Ms[r]);
                mvm_down(Ms[r]);  // (joins the side and work streams back into the context stream)
                tm.end(r);
            }
        }
        tm.collect(ms.data());
        if (rank_ms && k == 1) rank_ms[0] = ms[0];
        if (exch_ms) *exch_ms = ms[k];
        return s;
    } catch (const CudaError& e) {
        return e.code;
    }
}

xrl_status xrl_exchange_info(xrl_tree t, xrl_near nr, int64_t* halo_send, int64_t* halo_recv, int64_t* let_send,
                             int64_t* let_recv, int64_t* shared)
{
    if (!t) { set_error("xrl_exchange_info: null tree"); return XRL_EINVAL; }
    const bool dist = t->part_world > 1;
    if (halo_send) *halo_send = dist && nr ? nr->halo_soff.back() : 0;
    if (halo_recv) *halo_recv = dist && nr ? nr->halo_roff.back() : 0;
    if (let_send) *let_send = dist ? t->let_soff.back() : 0;
    if (let_recv) *let_recv = dist ? t->let_roff.back() : 0;
    if (shared) *shared = dist ? (int64_t)t->shared_boxes.size() : 0;
    return XRL_OK;
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

xrl_status xrl_mvm_host_batch(xrl_tree t, xrl_near nr, const void* const* x_host, void* const* y_host, int32_t nvec,
                              int32_t nbatch, uint32_t flags)
{
    if (!t || !nr || !x_host || !y_host || nbatch < 1) { set_error("xrl_mvm_host_batch: bad argument"); return XRL_EINVAL; }
    if (nvec < 3 || nvec % 3) { set_error("xrl_mvm_host_batch: nvec must be a positive multiple of 3"); return XRL_EDIM; }
    for (int k = 0; k < nbatch; ++k)
        if (!x_host[k] || !y_host[k]) { set_error("xrl_mvm_host_batch: null buffer %d", k); return XRL_EINVAL; }
    if (t->part_world > 1 && t->ctx->world == 1) { set_error("xrl_mvm_host_batch: virtual partition not supported"); return XRL_EUNSUPPORTED; }
    struct Res {
        cudaStream_t cin = nullptr, cout = nullptr;
        cudaEvent_t in_done[2] = {}, in_free[2] = {}, out_ready[2] = {}, out_free[2] = {};
        ~Res()
        {
            for (int b = 0; b < 2; ++b) {
                if (in_done[b]) cudaEventDestroy(in_done[b]);
                if (in_free[b]) cudaEventDestroy(in_free[b]);
                if (out_ready[b]) cudaEventDestroy(out_ready[b]);
                if (out_free[b]) cudaEventDestroy(out_free[b]);
            }
            if (cin) cudaStreamDestroy(cin);
            if (cout) cudaStreamDestroy(cout);
        }
    } R;
    try {
        cudaStream_t st = t->ctx->stream;
        XRL_CUDA(cudaSetDevice(t->ctx->device));
        const bool sliced = t->part_world > 1;  // multi-rank: library-order slices, no reordering
        const size_t cnt = (size_t)nvec * (sliced ? (t->p1 - t->p0) : t->n);
        for (int b = 0; b < 2; ++b)
            if (t->xbuf[b].n < cnt) { t->xbuf[b].alloc(cnt); t->ybuf[b].alloc(cnt); }
        if (!sliced && t->xlib.n < cnt) { t->xtmp.alloc(cnt); t->ytmp.alloc(cnt); t->xlib.alloc(cnt); t->ylib.alloc(cnt); }
        XRL_CUDA(cudaStreamCreateWithFlags(&R.cin, cudaStreamNonBlocking));
        XRL_CUDA(cudaStreamCreateWithFlags(&R.cout, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            XRL_CUDA(cudaEventCreateWithFlags(&R.in_done[b], cudaEventDisableTiming));
            XRL_CUDA(cudaEventCreateWithFlags(&R.in_free[b], cudaEventDisableTiming));
            XRL_CUDA(cudaEventCreateWithFlags(&R.out_ready[b], cudaEventDisableTiming));
            XRL_CUDA(cudaEventCreateWithFlags(&R.out_free[b], cudaEventDisableTiming));
        }
        // the copy streams start after the work already queued on the context stream
        XRL_CUDA(cudaEventRecord(R.in_free[0], st));
        XRL_CUDA(cudaStreamWaitEvent(R.cin, R.in_free[0], 0));
        XRL_CUDA(cudaStreamWaitEvent(R.cout, R.in_free[0], 0));
        for (int k = 0; k < nbatch; ++k) {
            const int b = k & 1;
            // H2D of step k (buffer b is free once step k-2 has consumed it)
            if (k >= 2) XRL_CUDA(cudaStreamWaitEvent(R.cin, R.in_free[b], 0));
            XRL_CUDA(cudaMemcpyAsync(t->xbuf[b].p, x_host[k], cnt * 8, cudaMemcpyHostToDevice, R.cin));
            XRL_CUDA(cudaEventRecord(R.in_done[b], R.cin));
            // compute on the context stream
            XRL_CUDA(cudaStreamWaitEvent(st, R.in_done[b], 0));
            if (k >= 2) XRL_CUDA(cudaStreamWaitEvent(st, R.out_free[b], 0));  // D2H of step k-2 done with ybuf[b]
            xrl_status s;
            if (sliced) {
                s = xrl_mvm(t, nr, t->xbuf[b].p, t->ybuf[b].p, nvec, flags);
                if (s) return s;
                XRL_CUDA(cudaEventRecord(R.in_free[b], st));
            } else {
                s = xrl_to_library_order(t, t->xbuf[b].p, t->xlib.p, nvec);
                if (s) return s;
                XRL_CUDA(cudaEventRecord(R.in_free[b], st));
                s = xrl_mvm(t, nr, t->xlib.p, t->ylib.p, nvec, flags);
                if (s) return s;
                s = xrl_from_library_order(t, t->ylib.p, t->ybuf[b].p, nvec);
                if (s) return s;
            }
            XRL_CUDA(cudaEventRecord(R.out_ready[b], st));
            // D2H of step k
            XRL_CUDA(cudaStreamWaitEvent(R.cout, R.out_ready[b], 0));
            XRL_CUDA(cudaMemcpyAsync(y_host[k], t->ybuf[b].p, cnt * 8, cudaMemcpyDeviceToHost, R.cout));
            XRL_CUDA(cudaEventRecord(R.out_free[b], R.cout));
        }
        XRL_CUDA(cudaStreamSynchronize(R.cout));
        XRL_CUDA(cudaStreamSynchronize(st));
        return XRL_OK;
    } catch (const CudaError& e) {
        return e.code;
    }
}

}  // extern "C"
