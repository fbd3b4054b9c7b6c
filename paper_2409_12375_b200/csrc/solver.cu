// Loop-space operator, diagonal-of-P block preconditioner, GMRES and port
// excitation (Eq. 8-11).
#include <algorithm>
#include <climits>
#include <cmath>
#include <complex>
#include <functional>

#include "xrl_internal.h"

using namespace xrl;

namespace {

constexpr double kMu0 = 4e-7 * M_PI;

inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }


// u[(3r+t)][k] = sum_{l} C_t(l,k) v[r][l]   (u_t = A_t^T M^T v, panel rows)
__global__ void k_loops_to_panels(int64_t n, int64_t nl, int nrhs, const int64_t* __restrict__ ptr,
                                  const int32_t* __restrict__ col, const float* __restrict__ val,
                                  const float2* __restrict__ v, float2* __restrict__ u)
{
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    for (int r = 0; r < nrhs; ++r) {
        float2 a0 = {0, 0}, a1 = {0, 0}, a2 = {0, 0};
        for (int64_t q = ptr[k]; q < ptr[k + 1]; ++q) {
            const float2 x = v[(int64_t)r * nl + col[q]];
            const float c0 = val[3 * q], c1 = val[3 * q + 1], c2 = val[3 * q + 2];
            a0.x += c0 * x.x; a0.y += c0 * x.y;
            a1.x += c1 * x.x; a1.y += c1 * x.y;
            a2.x += c2 * x.x; a2.y += c2 * x.y;
        }
        u[(int64_t)(3 * r + 0) * n + k] = a0;
        u[(int64_t)(3 * r + 1) * n + k] = a1;
        u[(int64_t)(3 * r + 2) * n + k] = a2;
    }
}

// w[r][l] = sum_t sum_k C_t(l,k) ( zsa_k u_t[k] + j alpha_im pu_t[k] )
constexpr int kLongRow = 64;  // loop rows longer than this (handle / fundamental loops) get a CTA each

__device__ __forceinline__ float2 panel_y(const float2* __restrict__ zsa, float alpha_im, const float2* __restrict__ u,
                                          const float2* __restrict__ pu, int64_t n, int r, int t, int k)
{
    const float2 z = zsa[k];
    const float2 uu = u[(int64_t)(3 * r + t) * n + k];
    const float2 pp = pu[(int64_t)(3 * r + t) * n + k];
    return make_float2(z.x * uu.x - z.y * uu.y - alpha_im * pp.y, z.x * uu.y + z.y * uu.x + alpha_im * pp.x);
}

__global__ void __launch_bounds__(256) k_panels_to_loops_long(int64_t n, int64_t nl, int nrhs,
                                                              const int32_t* __restrict__ rows,
                                                              const int64_t* __restrict__ ptr,
                                                              const int32_t* __restrict__ col,
                                                              const float* __restrict__ val,
                                                              const float2* __restrict__ zsa, float alpha_im,
                                                              const float2* __restrict__ u,
                                                              const float2* __restrict__ pu, float2* __restrict__ w)
{
    const int l = rows[blockIdx.x];
    __shared__ float2 red[256];
    for (int r = 0; r < nrhs; ++r) {
        float2 acc = {0, 0};
        for (int64_t q = ptr[l] + threadIdx.x; q < ptr[l + 1]; q += blockDim.x) {
            const int k = col[q];
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                const float2 y = panel_y(zsa, alpha_im, u, pu, n, r, t, k);
                const float c = val[3 * q + t];
                acc.x += c * y.x;
                acc.y += c * y.y;
            }
        }
        red[threadIdx.x] = acc;
        __syncthreads();
        for (int st = 128; st > 0; st >>= 1) {
            if (threadIdx.x < st) { red[threadIdx.x].x += red[threadIdx.x + st].x; red[threadIdx.x].y += red[threadIdx.x + st].y; }
            __syncthreads();
        }
        if (threadIdx.x == 0) w[(int64_t)r * nl + l] = red[0];
        __syncthreads();
    }
}

__global__ void k_panels_to_loops(int64_t n, int64_t nl, int nrhs, const int64_t* __restrict__ ptr,
                                  const int32_t* __restrict__ col, const float* __restrict__ val,
                                  const float2* __restrict__ zsa, float alpha_im, const float2* __restrict__ u,
                                  const float2* __restrict__ pu, float2* __restrict__ w)
{
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= nl) return;
    if (ptr[l + 1] - ptr[l] > kLongRow) return;  // done by k_panels_to_loops_long
    for (int r = 0; r < nrhs; ++r) {
        float2 acc = {0, 0};
        for (int64_t q = ptr[l]; q < ptr[l + 1]; ++q) {
            const int k = col[q];
            const float2 z = zsa[k];
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                const float2 uu = u[(int64_t)(3 * r + t) * n + k];
                const float2 pp = pu[(int64_t)(3 * r + t) * n + k];
                const float2 y = make_float2(z.x * uu.x - z.y * uu.y - alpha_im * pp.y,
                                             z.x * uu.y + z.y * uu.x + alpha_im * pp.x);
                const float c = val[3 * q + t];
                acc.x += c * y.x;
                acc.y += c * y.y;
            }
        }
        w[(int64_t)r * nl + l] = acc;
    }
}

// ---------------------------------------------------------------- preconditioner
// d_k = Z_s/A_k + j alpha P_kk (P_kk = diagonal of the near CSR, FP64).
__global__ void k_diag_p(int64_t n, const int64_t* __restrict__ ptr, const int32_t* __restrict__ col,
                         const double* __restrict__ val64, double* pkk)
{
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    double d = 0;
    for (int64_t q = ptr[k]; q < ptr[k + 1]; ++q)
        if (col[q] == k) d = val64[q];
    pkk[k] = d;
}

constexpr int kBS = 64;

// One CTA per block: assemble Q_BB = sum_k d_k c_a(k).c_b(k) (FP64 complex),
// invert in place by Gauss-Jordan with partial pivoting, store transposed.
// qdense != nullptr: the blocks come pre-assembled (FP64 complex, [block][kBS][kBS] row-major; any Q kind)
__global__ void __launch_bounds__(256) k_block_inverse(const int32_t* __restrict__ bptr, const int64_t* __restrict__ clp,
                                                       const int32_t* __restrict__ clc, const double* __restrict__ clv,
                                                       const int64_t* __restrict__ cpp, const int32_t* __restrict__ cpc,
                                                       const double* __restrict__ cpv,
                                                       const double2* __restrict__ dk, const double2* __restrict__ qdense,
                                                       float2* __restrict__ inv, int* singular)
{
    extern __shared__ double2 Qsm[];
    double2 (*Q)[kBS + 1] = reinterpret_cast<double2 (*)[kBS + 1]>(Qsm);
    __shared__ int piv[kBS];
    __shared__ double colmax[kBS];
    __shared__ int pivrow;
    __shared__ double qmax;
    const int blk = blockIdx.x;
    const int l0 = bptr[blk], m = bptr[blk + 1] - l0;
    const int tid = threadIdx.x;
    for (int i = tid; i < kBS * (kBS + 1); i += blockDim.x) (&Q[0][0])[i] = make_double2(0, 0);
    __syncthreads();
    if (qdense) {
        const double2* qb = qdense + (size_t)blk * kBS * kBS;
        for (int i = tid; i < m * m; i += blockDim.x) Q[i / m][i % m] = qb[(i / m) * kBS + i % m];
    }
    // assembly: thread per row a
    for (int a = tid; a < m && !qdense; a += blockDim.x) {
        const int la = l0 + a;
        for (int64_t q = clp[la]; q < clp[la + 1]; ++q) {
            const int k = clc[q];
            const double ca0 = clv[3 * q], ca1 = clv[3 * q + 1], ca2 = clv[3 * q + 2];
            const double2 d = dk[k];
            for (int64_t q2 = cpp[k]; q2 < cpp[k + 1]; ++q2) {
                const int lb = cpc[q2];
                if (lb < l0 || lb >= l0 + m) continue;
                // C value of (lb, k) from the panel row (was a search of lb's loop row: quadratic in the length
                // of the long fundamental loops, 1.1 s of block build on config 4)
                const double s = ca0 * cpv[3 * q2] + ca1 * cpv[3 * q2 + 1] + ca2 * cpv[3 * q2 + 2];
                Q[a][lb - l0].x += d.x * s;
                Q[a][lb - l0].y += d.y * s;
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        double mx = 0;
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < m; ++j) mx = fmax(mx, hypot(Q[i][j].x, Q[i][j].y));
        qmax = mx;
    }
    __syncthreads();
    // Gauss-Jordan in place
    for (int k = 0; k < m; ++k) {
        if (tid < m) colmax[tid] = (tid >= k) ? hypot(Q[tid][k].x, Q[tid][k].y) : -1.0;
        __syncthreads();
        if (tid == 0) {
            int p = k;
            for (int i = k + 1; i < m; ++i)
                if (colmax[i] > colmax[p]) p = i;
            pivrow = p;
            piv[k] = p;
            if (!(colmax[p] > 1e-13 * qmax)) atomicMax(singular, blk + 1);
        }
        __syncthreads();
        const int p = pivrow;
        if (p != k)
            for (int j = tid; j < m; j += blockDim.x) { double2 t = Q[k][j]; Q[k][j] = Q[p][j]; Q[p][j] = t; }
        __syncthreads();
        const double2 pv = Q[k][k];
        const double den = pv.x * pv.x + pv.y * pv.y;
        const double2 ip = make_double2(pv.x / den, -pv.y / den);
        __syncthreads();
        // scale row k (with Q[k][k] := 1 before scaling -> becomes 1/pivot)
        for (int j = tid; j < m; j += blockDim.x) {
            const double2 v = (j == k) ? make_double2(1, 0) : Q[k][j];
            Q[k][j] = make_double2(v.x * ip.x - v.y * ip.y, v.x * ip.y + v.y * ip.x);
        }
        __syncthreads();
        // eliminate column k from the other rows
        for (int idx = tid; idx < m * m; idx += blockDim.x) {
            const int i = idx / m, j = idx % m;
            if (i == k) continue;
            const double2 f = Q[i][k];
            if (j == k) continue;
            const double2 r = Q[k][j];
            Q[i][j].x -= f.x * r.x - f.y * r.y;
            Q[i][j].y -= f.x * r.y + f.y * r.x;
        }
        __syncthreads();
        for (int i = tid; i < m; i += blockDim.x) {
            if (i == k) continue;
            const double2 f = Q[i][k];
            Q[i][k] = make_double2(-(f.x * ip.x - f.y * ip.y), -(f.x * ip.y + f.y * ip.x));
        }
        __syncthreads();
    }
    // undo the row interchanges as column interchanges, in reverse order
    for (int k = m - 1; k >= 0; --k) {
        const int p = piv[k];
        if (p != k)
            for (int i = tid; i < m; i += blockDim.x) { double2 t = Q[i][k]; Q[i][k] = Q[i][p]; Q[i][p] = t; }
        __syncthreads();
    }
    // store transposed: inv[blk][b][a] = Q^-1[a][b]
    float2* out = inv + (size_t)blk * kBS * kBS;
    for (int idx = tid; idx < kBS * kBS; idx += blockDim.x) {
        const int b = idx / kBS, a = idx % kBS;
        out[idx] = (a < m && b < m) ? make_float2((float)Q[a][b].x, (float)Q[a][b].y) : make_float2(0.f, 0.f);
    }
}

// z_B = inv_B v_B, thread per row, inverse stored column-major.
__global__ void k_block_apply(int nl, int nrhs, const int32_t* __restrict__ bptr, const float2* __restrict__ inv,
                              const float2* __restrict__ v, float2* __restrict__ z)
{
    __shared__ float2 vs[kBS];
    const int blk = blockIdx.x;
    const int l0 = bptr[blk], m = bptr[blk + 1] - l0;
    const int a = threadIdx.x;
    const float2* B = inv + (size_t)blk * kBS * kBS;
    for (int r = 0; r < nrhs; ++r) {
        __syncthreads();
        if (a < m) vs[a] = v[(int64_t)r * nl + l0 + a];
        __syncthreads();
        if (a < m) {
            float2 acc = {0, 0};
            for (int b = 0; b < m; ++b) {
                const float2 q = B[b * kBS + a];
                acc.x += q.x * vs[b].x - q.y * vs[b].y;
                acc.y += q.x * vs[b].y + q.y * vs[b].x;
            }
            z[(int64_t)r * nl + l0 + a] = acc;
        }
    }
}

// ---------------------------------------------------------------- GMRES BLAS
// h[r][i] += sum_x conj(V[r][i][x]) w[r][x], i < ni   (grid (ni, nrhs, chunks), FP64
// accumulation, h zeroed by the caller, one double atomic per block)
constexpr int64_t kDotChunk = 16384;

__global__ void k_gdots(int64_t nl, int ldv, const float2* __restrict__ V, const float2* __restrict__ w,
                        double2* __restrict__ h, int ni)
{
    const int i = blockIdx.x, r = blockIdx.y;
    const float2* vi = V + ((int64_t)r * ldv + i) * nl;
    const float2* wr = w + (int64_t)r * nl;
    double sx = 0, sy = 0;
    const int64_t x0 = (int64_t)blockIdx.z * kDotChunk, x1 = min(nl, x0 + kDotChunk);
    for (int64_t x = x0 + threadIdx.x; x < x1; x += blockDim.x) {
        const float2 a = vi[x], b = wr[x];
        sx += (double)a.x * b.x + (double)a.y * b.y;
        sy += (double)a.x * b.y - (double)a.y * b.x;
    }
    __shared__ double rx[256], ry[256];
    rx[threadIdx.x] = sx;
    ry[threadIdx.x] = sy;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) { rx[threadIdx.x] += rx[threadIdx.x + s]; ry[threadIdx.x] += ry[threadIdx.x + s]; }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        atomicAdd(&h[(int64_t)r * ni + i].x, rx[0]);
        atomicAdd(&h[(int64_t)r * ni + i].y, ry[0]);
    }
}

// w[r][x] += sgn * sum_{i<ni} V[r][i][x] h[r][i]
__global__ void k_gupdate(int64_t nl, int ldv, int nrhs, const float2* __restrict__ V, const double2* __restrict__ h,
                          int ni, float sgn, float2* __restrict__ w)
{
    const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (x >= nl) return;
    for (int r = 0; r < nrhs; ++r) {
        float ax = 0, ay = 0;
        for (int i = 0; i < ni; ++i) {
            const float2 v = V[((int64_t)r * ldv + i) * nl + x];
            const double2 c = h[(int64_t)r * ni + i];
            ax += v.x * (float)c.x - v.y * (float)c.y;
            ay += v.x * (float)c.y + v.y * (float)c.x;
        }
        float2 o = w[(int64_t)r * nl + x];
        o.x += sgn * ax;
        o.y += sgn * ay;
        w[(int64_t)r * nl + x] = o;
    }
}

// out[r][x] = a[r][x] * s[r] (complex-real scale), s in FP64
__global__ void k_gscale(int64_t nl, int nrhs, const float2* __restrict__ a, int64_t a_stride,
                         const double* __restrict__ s, float2* __restrict__ out, int64_t o_stride)
{
    const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (x >= nl) return;
    for (int r = 0; r < nrhs; ++r) {
        const float2 v = a[r * a_stride + x];
        out[r * o_stride + x] = make_float2((float)(v.x * s[r]), (float)(v.y * s[r]));
    }
}

// out = a - b
__global__ void k_gaxpy(int64_t cnt, const float2* __restrict__ a, float2* __restrict__ x)  // x += a
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < cnt) { const float2 v = a[i]; x[i].x += v.x; x[i].y += v.y; }
}

__global__ void k_gsub(int64_t cnt, const float2* __restrict__ a, const float2* __restrict__ b, float2* __restrict__ out)
{
    const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (x >= cnt) return;
    out[x] = make_float2(a[x].x - b[x].x, a[x].y - b[x].y);
}

// ---- loop-space sharding (partitioned operators)
// y[(3r+t)][k] = zsa_k u_t[k] + j alpha_im pu_t[k] for the rank's panels (ystride: slot stride of y)
__global__ void k_panel_y(int64_t np, int nrhs, const float2* __restrict__ zsa, float alpha_im,
                          const float2* __restrict__ u, const float2* __restrict__ pu, float2* __restrict__ y,
                          int64_t ystride)
{
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= np) return;
    const float2 z = zsa[k];
    for (int c = 0; c < 3 * nrhs; ++c) {
        const float2 uu = u[(int64_t)c * np + k], pp = pu[(int64_t)c * np + k];
        y[(int64_t)c * ystride + k] = make_float2(z.x * uu.x - z.y * uu.y - alpha_im * pp.y,
                                                  z.x * uu.y + z.y * uu.x + alpha_im * pp.x);
    }
}

// w[r][l] = sum_q sum_t val[3q+t] y[(3r+t)][col[q]] for the rank's loops (rows longer than kLongRow: below)
__global__ void k_loops_from_y(int64_t nl, int nrhs, const int64_t* __restrict__ ptr, const int32_t* __restrict__ col,
                               const float* __restrict__ val, const float2* __restrict__ y, int64_t ystride,
                               float2* __restrict__ w)
{
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= nl) return;
    if (ptr[l + 1] - ptr[l] > kLongRow) return;
    for (int r = 0; r < nrhs; ++r) {
        float2 acc = {0, 0};
        for (int64_t q = ptr[l]; q < ptr[l + 1]; ++q)
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                const float2 v = y[(int64_t)(3 * r + t) * ystride + col[q]];
                const float c = val[3 * q + t];
                acc.x += c * v.x;
                acc.y += c * v.y;
            }
        w[(int64_t)r * nl + l] = acc;
    }
}

__global__ void __launch_bounds__(256) k_loops_from_y_long(int64_t nl, int nrhs, const int32_t* __restrict__ rows,
                                                           const int64_t* __restrict__ ptr,
                                                           const int32_t* __restrict__ col,
                                                           const float* __restrict__ val, const float2* __restrict__ y,
                                                           int64_t ystride, float2* __restrict__ w)
{
    const int l = rows[blockIdx.x];
    __shared__ float2 red[256];
    for (int r = 0; r < nrhs; ++r) {
        float2 acc = {0, 0};
        for (int64_t q = ptr[l] + threadIdx.x; q < ptr[l + 1]; q += blockDim.x)
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                const float2 v = y[(int64_t)(3 * r + t) * ystride + col[q]];
                const float c = val[3 * q + t];
                acc.x += c * v.x;
                acc.y += c * v.y;
            }
        red[threadIdx.x] = acc;
        __syncthreads();
        for (int st = 128; st > 0; st >>= 1) {
            if (threadIdx.x < st) { red[threadIdx.x].x += red[threadIdx.x + st].x; red[threadIdx.x].y += red[threadIdx.x + st].y; }
            __syncthreads();
        }
        if (threadIdx.x == 0) w[(int64_t)r * nl + l] = red[0];
        __syncthreads();
    }
}

// dst[i][c] = src[c][idx[i]]  (records of R complex values for the exchanges)
__global__ void k_pack_cols(int64_t cnt, int R, const int32_t* __restrict__ idx, const float2* __restrict__ src,
                            int64_t sstride, float2* __restrict__ dst)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= cnt * R) return;
    const int64_t i = t / R;
    const int c = (int)(t - i * R);
    dst[t] = src[(int64_t)c * sstride + idx[i]];
}
// dst[c][base + i] = src[i][c]
__global__ void k_unpack_cols(int64_t cnt, int R, const float2* __restrict__ src, float2* __restrict__ dst,
                              int64_t dstride, int64_t base)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= cnt * R) return;
    const int64_t i = t / R;
    const int c = (int)(t - i * R);
    dst[(int64_t)c * dstride + base + i] = src[t];
}

}  // namespace

// ====================================================================== host
using cd = std::complex<double>;

static void esi_eval(double sigma, double zeta, double f, double& re, double& im)
{
    const double rdc = 2.0 / (sigma * zeta);
    if (f <= 0) { re = rdc; im = 0; return; }
    const double rrf = std::sqrt(M_PI * kMu0 / sigma);
    const cd a = cd(1, 1) * rrf * std::sqrt(f);
    const cd x = a / rdc;
    cd z;
    if (std::abs(x) < 1e-4) z = rdc / (1.0 - x / 2.0 + x * x / 6.0 - x * x * x / 24.0);  // a/(1-e^-x) = rdc*x/(1-e^-x)
    else z = a / (1.0 - std::exp(-x));
    re = z.real();
    im = z.imag();
}

static void op_reserve(xrl_op op, int nrhs)
{
    if (op->cap_rhs >= nrhs) return;
    op->u.alloc((size_t)3 * nrhs * op->tree->n);
    op->pu.alloc((size_t)3 * nrhs * op->tree->n);
    op->cap_rhs = nrhs;
}

static xrl_status op_apply(xrl_op op, const float2* v, float2* w, int nrhs)
{
    xrl_tree t = op->tree;
    xrl_topo T = op->topo;
    cudaStream_t st = t->ctx->stream;
    const int64_t n = t->n, nl = T->n_loops;
    op_reserve(op, nrhs);
    k_loops_to_panels<<<nblk(n, 256), 256, 0, st>>>(n, nl, nrhs, T->cp_ptr.p, T->cp_col.p, T->cp_val.p, v, op->u.p);
    XRL_LAUNCH_CHECK();
    t->ctx->launches += 1;
    xrl_status s = xrl_mvm(t, op->near, op->u.p, op->pu.p, 3 * nrhs, XRL_MVM_FULL);
    if (s) return s;
    k_panels_to_loops<<<nblk(nl, 256), 256, 0, st>>>(n, nl, nrhs, T->cl_ptr.p, T->cl_col.p, T->cl_val.p, op->zsa.p,
                                                     (float)op->alpha_im, op->u.p, op->pu.p, w);
    XRL_LAUNCH_CHECK();
    t->ctx->launches += 1;
    if (T->n_long > 0) {
        k_panels_to_loops_long<<<T->n_long, 256, 0, st>>>(n, nl, nrhs, T->long_rows.p, T->cl_ptr.p, T->cl_col.p,
                                                          T->cl_val.p, op->zsa.p, (float)op->alpha_im, op->u.p,
                                                          op->pu.p, w);
        XRL_LAUNCH_CHECK();
        t->ctx->launches += 1;
    }
    return XRL_OK;
}

// ---------------------------------------------------------------- loop-space sharding
static int owner_in(const std::vector<int64_t>& cut, int64_t i)
{
    return (int)(std::upper_bound(cut.begin(), cut.end() - 1, i) - cut.begin()) - 1;
}

// Per-peer receive / send lists of rank me from need[r] (ascending ids; owner by `cut`).
static void split_by_owner(const std::vector<std::vector<int64_t>>& need, int me, const std::vector<int64_t>& cut,
                           std::vector<int64_t>& roff, std::vector<int64_t>& ridx, std::vector<int64_t>& soff,
                           std::vector<int64_t>& sidx)
{
    const int W = (int)cut.size() - 1;
    roff.assign(W + 1, 0);
    soff.assign(W + 1, 0);
    ridx.clear();
    sidx.clear();
    for (int q = 0; q < W; ++q) {
        roff[q] = (int64_t)ridx.size();
        if (q != me)
            for (int64_t v : need[me])
                if (owner_in(cut, v) == q) ridx.push_back(v);
        soff[q] = (int64_t)sidx.size();
        if (q != me)
            for (int64_t v : need[q])
                if (owner_in(cut, v) == me) sidx.push_back(v);
    }
    roff[W] = (int64_t)ridx.size();
    soff[W] = (int64_t)sidx.size();
}

// The loop-space shard of a partitioned operator (every rank derives every rank's lists from the shared
// topology, so the send list q -> r equals the receive list r <- q).
static void build_loop_partition(xrl_op op)
{
    xrl_tree t = op->tree;
    xrl_topo T = op->topo;
    cudaStream_t st = t->ctx->stream;
    const int W = t->part_world, me = t->part_rank;
    const int64_t nl = T->n_loops;
    std::vector<int64_t> pcut(t->part_cuts.begin(), t->part_cuts.end());
    const std::vector<int64_t>& cp = T->c_ptr_h;
    const std::vector<int32_t>& cc = T->c_col_h;
    const std::vector<double>& cv = T->c_val_h;
    auto P = std::make_unique<LoopPart>();
    // loop cuts: as many loops per rank as have their first (lowest) panel in the rank's panel range
    std::vector<int64_t> cnt(W + 1, 0);
    for (int64_t l = 0; l < nl; ++l) {
        int64_t mn = INT64_MAX;
        for (int64_t q = cp[l]; q < cp[l + 1]; ++q) mn = std::min<int64_t>(mn, cc[q]);
        cnt[mn == INT64_MAX ? W - 1 : owner_in(pcut, mn)]++;
    }
    P->lcut.assign(W + 1, 0);
    for (int r = 0; r < W; ++r) P->lcut[r + 1] = P->lcut[r] + cnt[r];
    P->L0 = P->lcut[me];
    P->L1 = P->lcut[me + 1];
    P->nlo = P->L1 - P->L0;
    P->npl = t->p1 - t->p0;
    // loop halo: loops a rank's panels read that another rank owns; panel halo: panels a rank's loops read
    std::vector<std::vector<int64_t>> lneed(W), pneed(W);
    std::vector<int64_t> seen(W, -1);
    std::vector<std::vector<uint8_t>> pmark(W, std::vector<uint8_t>(t->n, 0));
    for (int64_t l = 0; l < nl; ++l) {
        const int lo = owner_in(P->lcut, l);
        for (int64_t q = cp[l]; q < cp[l + 1]; ++q) {
            const int r = owner_in(pcut, cc[q]);
            if (r != lo && seen[r] != l) { seen[r] = l; lneed[r].push_back(l); }
            if (r != lo) pmark[lo][cc[q]] = 1;
        }
    }
    for (int r = 0; r < W; ++r) {
        for (int64_t k = 0; k < t->n; ++k)
            if (pmark[r][k]) pneed[r].push_back(k);
        std::vector<uint8_t>().swap(pmark[r]);
    }
    std::vector<int64_t> lr, ls, pr, ps;
    split_by_owner(lneed, me, P->lcut, P->lh_roff, lr, P->lh_soff, ls);
    split_by_owner(pneed, me, pcut, P->ph_roff, pr, P->ph_soff, ps);
    P->nlh = (int64_t)lr.size();
    P->nph = (int64_t)pr.size();
    auto up32 = [&](DBuf<int32_t>& d, const std::vector<int64_t>& h, int64_t base) {
        std::vector<int32_t> v(h.size());
        for (size_t i = 0; i < h.size(); ++i) v[i] = (int32_t)(h[i] - base);
        d.alloc(std::max<size_t>(1, v.size()));
        if (!v.empty()) XRL_CUDA(cudaMemcpyAsync(d.p, v.data(), 4 * v.size(), cudaMemcpyHostToDevice, st));
        XRL_CUDA(cudaStreamSynchronize(st));
    };
    up32(P->lh_sidx, ls, P->L0);
    up32(P->ph_sidx, ps, t->p0);
    // slots: owned loops [0, nlo) then the halo loops; owned panels [0, npl) then the halo panels
    auto slot_of = [](const std::vector<int64_t>& halo, int64_t id, int64_t lo, int64_t hi, int64_t nown) -> int32_t {
        if (id >= lo && id < hi) return (int32_t)(id - lo);
        return (int32_t)(nown + (std::lower_bound(halo.begin(), halo.end(), id) - halo.begin()));
    };
    // owned panel -> loop slots (transpose of C restricted to the owned panels)
    {
        std::vector<int64_t> ptr(P->npl + 1, 0);
        for (int64_t l = 0; l < nl; ++l)
            for (int64_t q = cp[l]; q < cp[l + 1]; ++q)
                if (cc[q] >= t->p0 && cc[q] < t->p1) ptr[cc[q] - t->p0 + 1]++;
        for (int64_t k = 0; k < P->npl; ++k) ptr[k + 1] += ptr[k];
        std::vector<int32_t> col(ptr[P->npl]);
        std::vector<float> val(3 * ptr[P->npl]);
        std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
        for (int64_t l = 0; l < nl; ++l)
            for (int64_t q = cp[l]; q < cp[l + 1]; ++q)
                if (cc[q] >= t->p0 && cc[q] < t->p1) {
                    const int64_t f = fill[cc[q] - t->p0]++;
                    col[f] = slot_of(lr, l, P->L0, P->L1, P->nlo);
                    for (int d = 0; d < 3; ++d) val[3 * f + d] = (float)cv[3 * q + d];
                }
        P->pl_ptr.alloc(ptr.size());
        P->pl_col.alloc(std::max<size_t>(1, col.size()));
        P->pl_val.alloc(std::max<size_t>(1, val.size()));
        XRL_CUDA(cudaMemcpyAsync(P->pl_ptr.p, ptr.data(), 8 * ptr.size(), cudaMemcpyHostToDevice, st));
        if (!col.empty()) {
            XRL_CUDA(cudaMemcpyAsync(P->pl_col.p, col.data(), 4 * col.size(), cudaMemcpyHostToDevice, st));
            XRL_CUDA(cudaMemcpyAsync(P->pl_val.p, val.data(), 4 * val.size(), cudaMemcpyHostToDevice, st));
        }
        XRL_CUDA(cudaStreamSynchronize(st));
    }
    // owned loop -> panel slots
    {
        std::vector<int64_t> ptr(P->nlo + 1, 0);
        std::vector<int32_t> col, lng;
        std::vector<float> val;
        for (int64_t l = P->L0; l < P->L1; ++l) {
            for (int64_t q = cp[l]; q < cp[l + 1]; ++q) {
                col.push_back(slot_of(pr, cc[q], t->p0, t->p1, P->npl));
                for (int d = 0; d < 3; ++d) val.push_back((float)cv[3 * q + d]);
            }
            ptr[l - P->L0 + 1] = (int64_t)col.size();
            if (cp[l + 1] - cp[l] > kLongRow) lng.push_back((int32_t)(l - P->L0));
        }
        P->lp_ptr.alloc(ptr.size());
        P->lp_col.alloc(std::max<size_t>(1, col.size()));
        P->lp_val.alloc(std::max<size_t>(1, val.size()));
        P->lp_long.alloc(std::max<size_t>(1, lng.size()));
        P->n_long = (int32_t)lng.size();
        XRL_CUDA(cudaMemcpyAsync(P->lp_ptr.p, ptr.data(), 8 * ptr.size(), cudaMemcpyHostToDevice, st));
        if (!col.empty()) {
            XRL_CUDA(cudaMemcpyAsync(P->lp_col.p, col.data(), 4 * col.size(), cudaMemcpyHostToDevice, st));
            XRL_CUDA(cudaMemcpyAsync(P->lp_val.p, val.data(), 4 * val.size(), cudaMemcpyHostToDevice, st));
        }
        if (!lng.empty()) XRL_CUDA(cudaMemcpyAsync(P->lp_long.p, lng.data(), 4 * lng.size(), cudaMemcpyHostToDevice, st));
        XRL_CUDA(cudaStreamSynchronize(st));
    }
    op->part = std::move(P);
}

static void part_reserve(LoopPart& P, int nrhs)
{
    if (P.cap >= nrhs) return;
    P.vext.alloc(std::max<int64_t>(1, (int64_t)nrhs * (P.nlo + P.nlh)));
    P.u.alloc(std::max<int64_t>(1, (int64_t)3 * nrhs * P.npl));
    P.pu.alloc(std::max<int64_t>(1, (int64_t)3 * nrhs * P.npl));
    P.yext.alloc(std::max<int64_t>(1, (int64_t)3 * nrhs * (P.npl + P.nph)));
    const int64_t recs = std::max({P.lh_soff.back(), P.lh_roff.back(), P.ph_soff.back(), P.ph_roff.back(), (int64_t)1});
    P.sbuf.alloc(recs * 3 * nrhs);
    P.rbuf.alloc(recs * 3 * nrhs);
    P.cap = nrhs;
}

// One exchange of the loop-space shard between k parts of one process (device copies) or over NCCL (k = 1).
static xrl_status part_exchange(const std::vector<xrl_op>& ops, bool loops, int rec, bool nccl, cudaStream_t st)
{
    const int k = (int)ops.size();
    if (nccl) {
        LoopPart& P = *ops[0]->part;
        return nccl_exchange(ops[0]->tree->ctx, (const float*)P.sbuf.p, loops ? P.lh_soff : P.ph_soff, (float*)P.rbuf.p,
                             loops ? P.lh_roff : P.ph_roff, 2 * rec, st);
    }
    for (int r = 0; r < k; ++r)
        for (int q = 0; q < k; ++q) {
            if (q == r) continue;
            LoopPart& S = *ops[q]->part;
            LoopPart& R = *ops[r]->part;
            const std::vector<int64_t>& so = loops ? S.lh_soff : S.ph_soff;
            const std::vector<int64_t>& ro = loops ? R.lh_roff : R.ph_roff;
            const int64_t cnt = so[r + 1] - so[r];
            if (cnt != ro[q + 1] - ro[q]) { set_error("loop-space exchange plans of ranks %d and %d disagree", q, r); return XRL_EINVAL; }
            if (cnt > 0)
                XRL_CUDA(cudaMemcpyAsync(R.rbuf.p + ro[q] * rec, S.sbuf.p + so[r] * rec, sizeof(float2) * cnt * rec,
                                         cudaMemcpyDeviceToDevice, st));
        }
    return XRL_OK;
}

// w = A v for the parts of a partitioned operator (all k ranks of a virtual run, or this rank over NCCL):
// loop halo -> u = C^T v on the owned panels -> P u by the sharded MVM -> y = Z_s/A u + j alpha P u ->
// panel halo -> w = C y on the owned loops.
static xrl_status op_apply_parts(const std::vector<xrl_op>& ops, const std::vector<const float2*>& v,
                                 const std::vector<float2*>& w, int nrhs, bool nccl)
{
    const int k = (int)ops.size();
    xrl_ctx ctx = ops[0]->tree->ctx;
    cudaStream_t st = ctx->stream;
    const int R = nrhs;
    for (int i = 0; i < k; ++i) {
        LoopPart& P = *ops[i]->part;
        part_reserve(P, nrhs);
        const int64_t ns = P.lh_soff.back();
        if (ns > 0) {
            k_pack_cols<<<nblk(ns * R, 256), 256, 0, st>>>(ns, R, P.lh_sidx.p, v[i], P.nlo, P.sbuf.p);
            XRL_LAUNCH_CHECK();
        }
    }
    xrl_status s = part_exchange(ops, true, R, nccl, st);
    if (s) return s;
    std::vector<float2*> u(k), pu(k);
    for (int i = 0; i < k; ++i) {
        xrl_op op = ops[i];
        LoopPart& P = *op->part;
        const int64_t nv = P.nlo + P.nlh;
        if (P.nlo > 0)
            XRL_CUDA(cudaMemcpy2DAsync(P.vext.p, 8 * nv, v[i], 8 * P.nlo, 8 * P.nlo, R, cudaMemcpyDeviceToDevice, st));
        if (P.nlh > 0) {
            k_unpack_cols<<<nblk(P.nlh * R, 256), 256, 0, st>>>(P.nlh, R, P.rbuf.p, P.vext.p, nv, P.nlo);
            XRL_LAUNCH_CHECK();
        }
        if (P.npl > 0) {
            k_loops_to_panels<<<nblk(P.npl, 256), 256, 0, st>>>(P.npl, nv, R, P.pl_ptr.p, P.pl_col.p, P.pl_val.p, P.vext.p,
                                                               P.u.p);
            XRL_LAUNCH_CHECK();
        }
        u[i] = P.u.p;
        pu[i] = P.pu.p;
        ctx->launches += 3;
    }
    // P u: the sharded MVM (NCCL collective, or the virtual-rank driver over the k trees)
    if (nccl) {
        s = xrl_mvm(ops[0]->tree, ops[0]->near, u[0], pu[0], 3 * R, XRL_MVM_FULL);
    } else {
        std::vector<xrl_tree> tr(k);
        std::vector<xrl_near> nr(k);
        std::vector<const void*> uv(k);
        std::vector<void*> pv(k);
        for (int i = 0; i < k; ++i) { tr[i] = ops[i]->tree; nr[i] = ops[i]->near; uv[i] = u[i]; pv[i] = pu[i]; }
        s = xrl_mvm_vranks(k, tr.data(), nr.data(), uv.data(), pv.data(), 3 * R, XRL_MVM_FULL, nullptr, nullptr);
    }
    if (s) return s;
    for (int i = 0; i < k; ++i) {
        xrl_op op = ops[i];
        LoopPart& P = *op->part;
        const int64_t ys = P.npl + P.nph;
        if (P.npl > 0) {
            k_panel_y<<<nblk(P.npl, 256), 256, 0, st>>>(P.npl, R, op->zsa.p + op->tree->p0, (float)op->alpha_im, P.u.p,
                                                       P.pu.p, P.yext.p, ys);
            XRL_LAUNCH_CHECK();
        }
        const int64_t ns = P.ph_soff.back();
        if (ns > 0) {
            k_pack_cols<<<nblk(ns * 3 * R, 256), 256, 0, st>>>(ns, 3 * R, P.ph_sidx.p, P.yext.p, ys, P.sbuf.p);
            XRL_LAUNCH_CHECK();
        }
    }
    s = part_exchange(ops, false, 3 * R, nccl, st);
    if (s) return s;
    for (int i = 0; i < k; ++i) {
        LoopPart& P = *ops[i]->part;
        const int64_t ys = P.npl + P.nph;
        if (P.nph > 0) {
            k_unpack_cols<<<nblk(P.nph * 3 * R, 256), 256, 0, st>>>(P.nph, 3 * R, P.rbuf.p, P.yext.p, ys, P.npl);
            XRL_LAUNCH_CHECK();
        }
        if (P.nlo > 0) {
            k_loops_from_y<<<nblk(P.nlo, 256), 256, 0, st>>>(P.nlo, R, P.lp_ptr.p, P.lp_col.p, P.lp_val.p, P.yext.p, ys,
                                                            w[i]);
            XRL_LAUNCH_CHECK();
        }
        if (P.n_long > 0) {
            k_loops_from_y_long<<<P.n_long, 256, 0, st>>>(P.nlo, R, P.lp_long.p, P.lp_ptr.p, P.lp_col.p, P.lp_val.p,
                                                          P.yext.p, ys, w[i]);
            XRL_LAUNCH_CHECK();
        }
        ctx->launches += 5;
    }
    return XRL_OK;
}

namespace xrl {
// Diagonal of the edge-edge matrix L = sum_t A_t P A_t^T (the diagonal-of-L baseline):
// for edge e between panels p < q with midpoint m, A(e, p) = m - c_p, A(e, q) = c_q - m (Alg. 1), so
// L_ee = |m - c_p|^2 P_pp + |c_q - m|^2 P_qq + 2 (m - c_p).(c_q - m) P_pq, with P_pq from the near CSR
// (edge-adjacent panels are always near).
__global__ void k_edge_ldiag(int64_t ne, const int32_t* __restrict__ ei, const int32_t* __restrict__ ej,
                             const double* __restrict__ mid, const double* __restrict__ cent,
                             const int64_t* __restrict__ ptr, const int32_t* __restrict__ col,
                             const double* __restrict__ val64, double* __restrict__ lee, int* missing)
{
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= ne) return;
    const int p = ei[e], q = ej[e];
    auto entry = [&](int r, int c) -> double {
        int64_t lo = ptr[r], hi = ptr[r + 1] - 1;
        while (lo < hi) {
            const int64_t md = (lo + hi) >> 1;
            if (col[md] < c) lo = md + 1; else hi = md;
        }
        if (lo < ptr[r + 1] && col[lo] == c) return val64[lo];
        atomicExch(missing, 1);
        return 0.0;
    };
    double ap = 0, aq = 0, apq = 0;
    for (int d = 0; d < 3; ++d) {
        const double a = mid[3 * e + d] - cent[3 * (int64_t)p + d], b = cent[3 * (int64_t)q + d] - mid[3 * e + d];
        ap += a * a;
        aq += b * b;
        apq += a * b;
    }
    lee[e] = ap * entry(p, p) + aq * entry(q, q) + 2.0 * apq * entry(p, q);
}

void precond_ldiag(xrl_op op, std::vector<double>& lee)
{
    xrl_tree t = op->tree;
    xrl_topo T = op->topo;
    cudaStream_t st = t->ctx->stream;
    const int64_t ne = T->n_edges;
    lee.assign(ne, 0.0);
    if (ne == 0) return;
    DBuf<int32_t> ei(ne), ej(ne);
    DBuf<double> mid(3 * ne), out(ne);
    DBuf<int> miss(1);
    XRL_CUDA(cudaMemcpyAsync(ei.p, T->edge_i.data(), 4 * ne, cudaMemcpyHostToDevice, st));
    XRL_CUDA(cudaMemcpyAsync(ej.p, T->edge_j.data(), 4 * ne, cudaMemcpyHostToDevice, st));
    XRL_CUDA(cudaMemcpyAsync(mid.p, T->edge_mid.data(), 24 * ne, cudaMemcpyHostToDevice, st));
    XRL_CUDA(cudaMemsetAsync(miss.p, 0, 4, st));
    k_edge_ldiag<<<nblk(ne, 256), 256, 0, st>>>(ne, ei.p, ej.p, mid.p, t->cent.p, op->near->row_ptr.p, op->near->col.p,
                                                op->near->val64.p, out.p, miss.p);
    XRL_LAUNCH_CHECK();
    int hm = 0;
    XRL_CUDA(cudaMemcpyAsync(lee.data(), out.p, 8 * ne, cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaMemcpyAsync(&hm, miss.p, 4, cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaStreamSynchronize(st));
    if (hm) {
        set_error("diag-of-L: an edge's panel pair is not in the near field (eta too small)");
        throw CudaError{XRL_EGEOM};
    }
}

void precond_diag(xrl_op op, std::vector<double2>& hd)
{
    xrl_tree t = op->tree;
    cudaStream_t st = t->ctx->stream;
    const int64_t n = t->n;
    DBuf<double> pkk(n);
    k_diag_p<<<nblk(n, 256), 256, 0, st>>>(n, op->near->row_ptr.p, op->near->col.p, op->near->val64.p, pkk.p);
    XRL_LAUNCH_CHECK();
    std::vector<double> hp(n);
    XRL_CUDA(cudaMemcpyAsync(hp.data(), pkk.p, 8 * n, cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaStreamSynchronize(st));
    hd.resize(n);
    for (int64_t i = 0; i < n; ++i) hd[i] = make_double2(op->zsa_h[2 * i], op->zsa_h[2 * i + 1] + op->alpha_im * hp[i]);
}
}  // namespace xrl

static void pc_apply(xrl_precond pc, const float2* v, float2* z, int nrhs)
{
    if (pc->kind == 1) {
        exact_apply(pc, v, z, nrhs);
        return;
    }
    xrl_tree t = pc->op->tree;
    const int nl = (int)pc->nl_loc;
    k_block_apply<<<pc->nblocks, kBS, 0, t->ctx->stream>>>(nl, nrhs, pc->bptr_loc.p, pc->inv.p, v, z);
    XRL_LAUNCH_CHECK();
    t->ctx->launches += 1;
}

void xrl::op_release(xrl_op op)
{
    if (!op->dead || op->refs > 0) return;
    xrl_tree t = op->tree;
    xrl_topo T = op->topo;
    cudaSetDevice(t->ctx->device);
    cudaStreamSynchronize(t->ctx->stream);
    xrl_near nr = op->near;
    delete op;
    --T->refs;
    topo_release(T);
    --nr->refs;
    near_release(nr);
    --t->refs;
    tree_release(t);
}

#define API_TRY try {
#define API_CATCH                                   \
    }                                               \
    catch (const CudaError& e) { return e.code; }   \
    catch (const std::bad_alloc&) {                 \
        set_error("host out of memory");            \
        return XRL_ENOMEM;                          \
    }

extern "C" {

xrl_status xrl_esi(double sigma, double zeta, double f, double* re, double* im)
{
    if (!(sigma > 0) || !(zeta > 0) || f < 0 || !re || !im) { set_error("xrl_esi: sigma, zeta > 0 and f >= 0 required"); return XRL_EINVAL; }
    esi_eval(sigma, zeta, f, *re, *im);
    return XRL_OK;
}

xrl_status xrl_operator_create(xrl_tree t, xrl_near nr, xrl_topo T, const double* zs, double sigma, double zeta,
                               double freq, xrl_op* out)
{
    if (!t || !nr || !T || !out) { set_error("xrl_operator_create: null argument"); return XRL_EINVAL; }
    *out = nullptr;
    if (nr->tree != t || T->tree != t) { set_error("xrl_operator_create: handles from different trees"); return XRL_EPROVENANCE; }
    if (freq < 0) { set_error("xrl_operator_create: negative frequency"); return XRL_EINVAL; }
    if (!zs && (!(sigma > 0) || !(zeta > 0))) { set_error("xrl_operator_create: need zs or sigma, zeta > 0"); return XRL_EINVAL; }
    API_TRY
        XRL_CUDA(cudaSetDevice(t->ctx->device));
        auto op = std::make_unique<xrl_op_s>();
        op->tree = t;
        op->near = nr;
        op->topo = T;
        op->freq = freq;
        op->omega = 2 * M_PI * freq;
        op->alpha_im = op->omega * kMu0 / (4 * M_PI);
        const int64_t n = t->n;
        std::vector<double> area(n);
        XRL_CUDA(cudaMemcpy(area.data(), t->area.p, 8 * n, cudaMemcpyDeviceToHost));
        op->zsa_h.resize(2 * n);
        std::vector<float2> zf(n);
        double zr = 0, zi = 0;
        if (!zs) esi_eval(sigma, zeta, freq, zr, zi);
        for (int64_t i = 0; i < n; ++i) {
            const int64_t k = T->perm[i];
            const double a = zs ? zs[2 * k] : zr, b = zs ? zs[2 * k + 1] : zi;
            op->zsa_h[2 * i] = a / area[i];
            op->zsa_h[2 * i + 1] = b / area[i];
            zf[i] = make_float2((float)(a / area[i]), (float)(b / area[i]));
        }
        op->zsa.alloc(n);
        XRL_CUDA(cudaMemcpy(op->zsa.p, zf.data(), 8 * n, cudaMemcpyHostToDevice));
        if (t->part_world > 1) build_loop_partition(op.get());  // loop-space shard of a partitioned tree
        ++T->refs;
        ++nr->refs;
        ++t->refs;
        *out = op.release();
        return XRL_OK;
    API_CATCH
}

void xrl_operator_destroy(xrl_op op)
{
    if (!op) return;
    op->dead = true;
    op_release(op);  // deferred while preconditioners built on it are alive
}

xrl_status xrl_operator_apply(xrl_op op, const void* v, void* w, int32_t nrhs)
{
    if (!op || !v || !w || nrhs < 1) { set_error("xrl_operator_apply: bad argument"); return XRL_EINVAL; }
    if (v == w) { set_error("xrl_operator_apply: v and w alias"); return XRL_EINVAL; }
    API_TRY
        XRL_CUDA(cudaSetDevice(op->tree->ctx->device));
        if (op->part) {
            if (op->tree->ctx->world == 1) {
                set_error("xrl_operator_apply: a virtual-rank operator runs through xrl_operator_apply_vranks");
                return XRL_EUNSUPPORTED;
            }
            return op_apply_parts({op}, {(const float2*)v}, {(float2*)w}, nrhs, true);
        }
        return op_apply(op, (const float2*)v, (float2*)w, nrhs);
    API_CATCH
}

static xrl_status check_vrank_ops(int32_t k, const xrl_op* ops, const char* who)
{
    if (k < 1 || !ops) { set_error("%s: bad argument", who); return XRL_EINVAL; }
    for (int r = 0; r < k; ++r) {
        if (!ops[r]) { set_error("%s: null operator %d", who, r); return XRL_EINVAL; }
        xrl_tree t = ops[r]->tree;
        const bool one = k == 1 && !ops[r]->part;
        if (!one && (!ops[r]->part || t->part_world != k || t->part_rank != r || t->ctx->world != 1 ||
                     t->ctx != ops[0]->tree->ctx || ops[r]->topo->n_loops != ops[0]->topo->n_loops)) {
            set_error("%s: operator %d is not rank %d of a %d-way partition on one single-rank context", who, r, r, k);
            return XRL_EINVAL;
        }
    }
    return XRL_OK;
}

xrl_status xrl_operator_info(xrl_op op, int64_t* loop_offset, int64_t* n_loops_local, int64_t* loop_halo,
                             int64_t* panel_halo)
{
    if (!op) { set_error("xrl_operator_info: null operator"); return XRL_EINVAL; }
    if (loop_offset) *loop_offset = op->part ? op->part->L0 : 0;
    if (n_loops_local) *n_loops_local = op->part ? op->part->nlo : op->topo->n_loops;
    if (loop_halo) *loop_halo = op->part ? op->part->lh_soff.back() + op->part->lh_roff.back() : 0;
    if (panel_halo) *panel_halo = op->part ? op->part->ph_soff.back() + op->part->ph_roff.back() : 0;
    return XRL_OK;
}

xrl_status xrl_operator_apply_vranks(int32_t k, const xrl_op* ops, const void* const* v, void* const* w, int32_t nrhs)
{
    xrl_status s = check_vrank_ops(k, ops, "xrl_operator_apply_vranks");
    if (s) return s;
    if (!v || !w || nrhs < 1) { set_error("xrl_operator_apply_vranks: bad argument"); return XRL_EINVAL; }
    API_TRY
        XRL_CUDA(cudaSetDevice(ops[0]->tree->ctx->device));
        if (k == 1 && !ops[0]->part) return op_apply(ops[0], (const float2*)v[0], (float2*)w[0], nrhs);
        std::vector<xrl_op> o(ops, ops + k);
        std::vector<const float2*> vv(k);
        std::vector<float2*> ww(k);
        for (int r = 0; r < k; ++r) { vv[r] = (const float2*)v[r]; ww[r] = (float2*)w[r]; }
        return op_apply_parts(o, vv, ww, nrhs, false);
    API_CATCH
}

static xrl_status precond_build_blocks(xrl_op op, int32_t qkind, int32_t block_size, xrl_precond* out)
{
    xrl_tree t = op->tree;
    xrl_topo T = op->topo;
    cudaStream_t st = t->ctx->stream;
    XRL_CUDA(cudaSetDevice(t->ctx->device));
    const int64_t n = t->n;
    // the blocks cover this rank's loops (all loops on a single-rank operator): no communication in the apply
    const int64_t L0 = op->part ? op->part->L0 : 0, L1 = op->part ? op->part->L1 : T->n_loops;
    auto pc = std::make_unique<xrl_precond_s>();
    pc->op = op;
    pc->qkind = qkind;
    pc->bs = block_size;
    for (int64_t l = L0; l < L1; l += block_size) pc->bptr_h.push_back((int32_t)l);
    pc->bptr_h.push_back((int32_t)L1);
    pc->nblocks = (int32_t)pc->bptr_h.size() - 1;
    pc->nl_loc = L1 - L0;
    pc->bptr.alloc(pc->bptr_h.size());
    pc->bptr_loc.alloc(pc->bptr_h.size());
    XRL_CUDA(cudaMemcpyAsync(pc->bptr.p, pc->bptr_h.data(), 4 * pc->bptr_h.size(), cudaMemcpyHostToDevice, st));
    {
        std::vector<int32_t> loc(pc->bptr_h.size());
        for (size_t i = 0; i < loc.size(); ++i) loc[i] = (int32_t)(pc->bptr_h[i] - L0);
        XRL_CUDA(cudaMemcpyAsync(pc->bptr_loc.p, loc.data(), 4 * loc.size(), cudaMemcpyHostToDevice, st));
        XRL_CUDA(cudaStreamSynchronize(st));
    }
    DBuf<double2> dk, qd;
    if (qkind == 0) {
        // d_k = Z_s/A + j alpha P_kk; the blocks are assembled on the GPU from C = M A_t
        std::vector<double2> hd;
        precond_diag(op, hd);
        dk.alloc(n);
        XRL_CUDA(cudaMemcpyAsync(dk.p, hd.data(), 16 * n, cudaMemcpyHostToDevice, st));
    } else {
        // any other Q (diag-of-L): assembled sparse on the host, its diagonal blocks uploaded dense
        std::vector<std::vector<int32_t>> rc;
        std::vector<std::vector<std::complex<double>>> rv;
        assemble_q(op, qkind, rc, rv);
        std::vector<double2> h((size_t)pc->nblocks * kBS * kBS, make_double2(0, 0));
        for (int b = 0; b < pc->nblocks; ++b) {
            const int l0 = pc->bptr_h[b], l1 = pc->bptr_h[b + 1];
            for (int a = l0; a < l1; ++a)
                for (size_t i = 0; i < rc[a].size(); ++i)
                    if (rc[a][i] >= l0 && rc[a][i] < l1)
                        h[((size_t)b * kBS + (a - l0)) * kBS + (rc[a][i] - l0)] =
                            make_double2(rv[a][i].real(), rv[a][i].imag());
        }
        qd.alloc(h.size());
        XRL_CUDA(cudaMemcpyAsync(qd.p, h.data(), 16 * h.size(), cudaMemcpyHostToDevice, st));
    }
    pc->inv.alloc((size_t)pc->nblocks * kBS * kBS);
    DBuf<int> sing(1);
    XRL_CUDA(cudaMemsetAsync(sing.p, 0, 4, st));
    if (pc->nblocks > 0) {
        const int smem = kBS * (kBS + 1) * (int)sizeof(double2);
        XRL_CUDA(cudaFuncSetAttribute(k_block_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        k_block_inverse<<<pc->nblocks, 256, smem, st>>>(pc->bptr.p, T->cl_ptr.p, T->cl_col.p, T->cl_val64.p, T->cp_ptr.p,
                                                     T->cp_col.p, T->cp_val64.p, dk.p, qd.p, pc->inv.p, sing.p);
        XRL_LAUNCH_CHECK();
    }
    int hs = 0;
    XRL_CUDA(cudaMemcpyAsync(&hs, sing.p, 4, cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaStreamSynchronize(st));
    if (hs) { set_error("xrl_precond_build: singular block %d (pivot below 1e-13 of the block max)", hs - 1); return XRL_ESINGULAR; }
    ++op->refs;
    *out = pc.release();
    return XRL_OK;
}

static xrl_status precond_build_exact_kind(xrl_op op, int32_t qkind, xrl_precond* out, int ilu = 0)
{
    if (op->part) {
        set_error("the exact Q^-1 is not sharded: partitioned operators use block-Jacobi preconditioners");
        return XRL_EUNSUPPORTED;
    }
    XRL_CUDA(cudaSetDevice(op->tree->ctx->device));
    auto pc = std::make_unique<xrl_precond_s>();
    pc->op = op;
    pc->kind = 1;
    pc->qkind = qkind;
    pc->ilu = ilu;
    pc->bs = 0;
    const xrl_status s = exact_build(pc.get());
    if (s != XRL_OK) return s;
    ++op->refs;
    *out = pc.release();
    return XRL_OK;
}

xrl_status xrl_precond_build(xrl_op op, int32_t block_size, xrl_precond* out)
{
    if (!op || !out) { set_error("xrl_precond_build: null argument"); return XRL_EINVAL; }
    *out = nullptr;
    if (block_size < 1 || block_size > kBS) { set_error("xrl_precond_build: block_size must be 1..%d", kBS); return XRL_EINVAL; }
    API_TRY
        return precond_build_blocks(op, 0, block_size, out);
    API_CATCH
}

xrl_status xrl_precond_build_kind(xrl_op op, int32_t kind, int32_t block_size, xrl_precond* out)
{
    if (!op || !out) { set_error("xrl_precond_build_kind: null argument"); return XRL_EINVAL; }
    *out = nullptr;
    if (kind != XRL_PRECOND_DIAG_P && kind != XRL_PRECOND_DIAG_L) { set_error("xrl_precond_build_kind: bad kind %d", kind); return XRL_EINVAL; }
    if (block_size != -1 && block_size != -2 && (block_size < 1 || block_size > kBS)) {
        set_error("xrl_precond_build_kind: block_size must be -1 (exact), -2 (ILU(0)) or 1..%d", kBS);
        return XRL_EINVAL;
    }
    API_TRY
        if (block_size < 0) return precond_build_exact_kind(op, kind, out, block_size == -2);
        return precond_build_blocks(op, kind, block_size, out);
    API_CATCH
}

xrl_status xrl_precond_build_exact(xrl_op op, xrl_precond* out)
{
    if (!op || !out) { set_error("xrl_precond_build_exact: null argument"); return XRL_EINVAL; }
    *out = nullptr;
    API_TRY
        return precond_build_exact_kind(op, 0, out);
    API_CATCH
}

void xrl_precond_destroy(xrl_precond pc)
{
    if (!pc) return;
    if (pc->kind == 1) exact_free(pc);
    xrl_op op = pc->op;
    delete pc;
    --op->refs;
    op_release(op);
}

xrl_status xrl_precond_apply(xrl_precond pc, const void* v, void* z, int32_t nrhs)
{
    if (!pc || !v || !z || nrhs < 1) { set_error("xrl_precond_apply: bad argument"); return XRL_EINVAL; }
    API_TRY
        XRL_CUDA(cudaSetDevice(pc->op->tree->ctx->device));
        pc_apply(pc, (const float2*)v, (float2*)z, nrhs);
        return XRL_OK;
    API_CATCH
}

xrl_status xrl_precond_export(xrl_precond pc, int32_t* n_blocks, int32_t* block_size, int32_t* block_ptr, void* inv)
{
    if (!pc) { set_error("xrl_precond_export: null handle"); return XRL_EINVAL; }
    if (pc->kind != 0) { set_error("xrl_precond_export: not a block preconditioner"); return XRL_EINVAL; }
    API_TRY
        if (n_blocks) *n_blocks = pc->nblocks;
        if (block_size) *block_size = kBS;
        if (block_ptr) std::copy(pc->bptr_h.begin(), pc->bptr_h.end(), block_ptr);
        if (inv) {
            // device stores column-major per block; export row-major
            std::vector<float2> h((size_t)pc->nblocks * kBS * kBS);
            XRL_CUDA(cudaMemcpy(h.data(), pc->inv.p, 8 * h.size(), cudaMemcpyDeviceToHost));
            float2* o = (float2*)inv;
            for (int b = 0; b < pc->nblocks; ++b)
                for (int i = 0; i < kBS; ++i)
                    for (int j = 0; j < kBS; ++j) o[((size_t)b * kBS + i) * kBS + j] = h[((size_t)b * kBS + j) * kBS + i];
        }
        return XRL_OK;
    API_CATCH
}

xrl_status xrl_port_rhs(xrl_topo T, int32_t port, double volts, void* b)
{
    if (!T || !b || port < 0 || port >= T->n_ports) { set_error("xrl_port_rhs: bad argument"); return XRL_EINVAL; }
    API_TRY
        xrl_ctx ctx = T->tree->ctx;
        XRL_CUDA(cudaSetDevice(ctx->device));
        std::vector<float2> h(T->n_loops, make_float2(0.f, 0.f));
        // V_l = sum_b M(l,b) V_b, V_b = volts on the port branch only
        int port_branch = -1, seen = -1;
        for (int64_t b2 = 0; b2 < T->n_branches; ++b2)
            if (T->br_kind[b2] == 2 && ++seen == port) { port_branch = (int)b2; break; }
        for (int64_t l = 0; l < T->n_loops; ++l)
            for (int64_t q = T->m_ptr[l]; q < T->m_ptr[l + 1]; ++q)
                if (T->m_idx[q] == port_branch) h[l].x += (float)(T->m_val[q] * volts);
        XRL_CUDA(cudaMemcpyAsync(b, h.data(), 8 * h.size(), cudaMemcpyHostToDevice, ctx->stream));
        XRL_CUDA(cudaStreamSynchronize(ctx->stream));
        return XRL_OK;
    API_CATCH
}

xrl_status xrl_port_currents(xrl_topo T, const void* x, int32_t nrhs, double* ip)
{
    if (!T || !x || !ip || nrhs < 1) { set_error("xrl_port_currents: bad argument"); return XRL_EINVAL; }
    API_TRY
        xrl_ctx ctx = T->tree->ctx;
        XRL_CUDA(cudaSetDevice(ctx->device));
        const int64_t nl = T->n_loops;
        for (int r = 0; r < nrhs; ++r)
            for (int p = 0; p < T->n_ports; ++p) {
                // I_branch = (M^T I_l)[port branch] = sign * I_l(port loop)
                const int l = T->port_loop[p];
                int sign = 0;
                for (int64_t q = T->m_ptr[l]; q < T->m_ptr[l + 1]; ++q)
                    if (T->br_kind[T->m_idx[q]] == 2) sign = T->m_val[q];
                float2 v;
                XRL_CUDA(cudaMemcpyAsync(&v, (const float2*)x + (size_t)r * nl + l, 8, cudaMemcpyDeviceToHost, ctx->stream));
                XRL_CUDA(cudaStreamSynchronize(ctx->stream));
                ip[2 * ((size_t)r * T->n_ports + p)] = sign * (double)v.x;
                ip[2 * ((size_t)r * T->n_ports + p) + 1] = sign * (double)v.y;
            }
        return XRL_OK;
    API_CATCH
}

// Restarted GMRES over the parts of a loop-space system: one part (single-rank operator, or this rank of a
// multi-rank operator: partial dots all-reduced over NCCL) or k parts of a virtual-rank run (partial dots
// summed on the host).  Every column r has its own Krylov space; all columns step together, so every
// operator and preconditioner call is batched (reading C-A12).  Hessenberg / Givens in FP64 on the host.
struct GPart {
    xrl_op op;
    xrl_precond pc;
    const float2* b;
    float2* x;
    int64_t nl;
    DBuf<float2> V, w, tmp;
    DBuf<double2> dh;
    DBuf<double2> dc;  // one Arnoldi step's coefficients on the device: CGS2 passes [2][nrhs][m+1], norms [nrhs]
    DBuf<double> ds, ones;
};

// virtual ranks: buf[q][off .. off + cnt) summed over the k parts, the sum written back to every part
__global__ void k_sum_parts(int k, double2* const* __restrict__ buf, size_t off, int cnt)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    double2 a = make_double2(0, 0);
    for (int q = 0; q < k; ++q) { const double2 v = buf[q][off + i]; a.x += v.x; a.y += v.y; }
    for (int q = 0; q < k; ++q) buf[q][off + i] = a;
}

// ds[r] = 1 / sqrt(max(dn[r].x, 0)) (0 below 1e-300): the new basis vector's scale from the device norm
__global__ void k_inv_norm(int nrhs, const double2* __restrict__ dn, double* __restrict__ ds)
{
    const int r = threadIdx.x;
    if (r >= nrhs) return;
    const double hn = sqrt(fmax(dn[r].x, 0.0));
    ds[r] = hn > 1e-300 ? 1.0 / hn : 0.0;
}

static xrl_status gmres_parts(std::vector<GPart>& P, bool nccl, int32_t nrhs, const xrl_gmres_opts* opts,
                              int32_t* iters_out, double* rre_out, double* true_rre_out, int32_t* conv_out)
{
    const int k = (int)P.size();
    const int m = opts && opts->restart > 0 ? opts->restart : 50;
    const int maxit = opts && opts->max_iters > 0 ? opts->max_iters : 2000;
    double tol = opts ? opts->tol : 0;
    const bool have_pc = P[0].pc != nullptr;
    // right preconditioning (A M^-1 u = b, x = M^-1 u; default when opts is NULL, reading R15)
    const bool right = have_pc && (!opts || opts->right_precond);
    if (!(tol > 0)) tol = P[0].op->freq > 1e6 ? 1e-4 : 1e-6;  // PAPER.md:152, reading C-A8
    if (tol >= 1) { set_error("xrl_gmres: tol must be < 1"); return XRL_EINVAL; }
    xrl_ctx ctx = P[0].op->tree->ctx;
    cudaStream_t st = ctx->stream;
    const bool sharded = P[0].op->part != nullptr;
    for (auto& p : P) {
        p.V.alloc(std::max<size_t>(1, (size_t)nrhs * (m + 1) * p.nl));
        p.w.alloc(std::max<size_t>(1, (size_t)nrhs * p.nl));
        p.tmp.alloc(std::max<size_t>(1, (size_t)nrhs * p.nl));
        p.dh.alloc((size_t)nrhs * (m + 1));
        p.dc.alloc((size_t)nrhs * (2 * (m + 1) + 1));
        p.ds.alloc(nrhs);
        p.ones.alloc(nrhs);
        std::vector<double> one(nrhs, 1.0);
        XRL_CUDA(cudaMemcpyAsync(p.ones.p, one.data(), 8 * nrhs, cudaMemcpyHostToDevice, st));
    }
    std::vector<double2> hh((size_t)nrhs * (m + 1)), hsum((size_t)nrhs * (m + 1));
    DBuf<double2*> dcptr(k);  // the parts' step-coefficient buffers (device sum over virtual ranks)
    {
        std::vector<double2*> h(k);
        for (int q = 0; q < k; ++q) h[q] = P[q].dc.p;
        XRL_CUDA(cudaMemcpyAsync(dcptr.p, h.data(), sizeof(double2*) * k, cudaMemcpyHostToDevice, st));
    }
    using BufSel = DBuf<float2> GPart::*;
    auto opA = [&](std::function<const float2*(GPart&)> in, std::function<float2*(GPart&)> out) -> xrl_status {
        if (!sharded) return op_apply(P[0].op, in(P[0]), out(P[0]), nrhs);
        std::vector<xrl_op> ops;
        std::vector<const float2*> vi;
        std::vector<float2*> wo;
        for (auto& p : P) { ops.push_back(p.op); vi.push_back(in(p)); wo.push_back(out(p)); }
        return op_apply_parts(ops, vi, wo, nrhs, nccl);
    };
    auto Mx = [&](GPart& p, const float2* in, float2* o) {  // o = M^-1 in (or copy)
        if (p.pc) pc_apply(p.pc, in, o, nrhs);
        else if (p.nl) XRL_CUDA(cudaMemcpyAsync(o, in, 8 * nrhs * p.nl, cudaMemcpyDeviceToDevice, st));
    };
    // h[r][i] = sum over the parts (and ranks) of conj(V_i) . w  -> host
    auto dots = [&](std::function<const float2*(GPart&)> a, int ldv, std::function<const float2*(GPart&)> b, int ni,
                    std::vector<double2>& out) -> xrl_status {
        std::fill(hsum.begin(), hsum.begin() + (size_t)nrhs * ni, make_double2(0, 0));
        for (auto& p : P) {
            XRL_CUDA(cudaMemsetAsync(p.dh.p, 0, 16 * nrhs * ni, st));
            if (p.nl > 0) {
                k_gdots<<<dim3(ni, nrhs, (unsigned)((p.nl + kDotChunk - 1) / kDotChunk)), 256, 0, st>>>(p.nl, ldv, a(p),
                                                                                                       b(p), p.dh.p, ni);
                XRL_LAUNCH_CHECK();
            }
            if (nccl) {
                xrl_status s = nccl_allreduce_sum_f64(ctx, (double*)p.dh.p, (size_t)2 * nrhs * ni, st);
                if (s) return s;
            }
            XRL_CUDA(cudaMemcpyAsync(hh.data(), p.dh.p, 16 * nrhs * ni, cudaMemcpyDeviceToHost, st));
            XRL_CUDA(cudaStreamSynchronize(st));
            for (size_t i = 0; i < (size_t)nrhs * ni; ++i) { hsum[i].x += hh[i].x; hsum[i].y += hh[i].y; }
        }
        out.assign(hsum.begin(), hsum.begin() + (size_t)nrhs * ni);
        return XRL_OK;
    };
    auto norms = [&](std::function<const float2*(GPart&)> a, std::vector<double>& out) -> xrl_status {
        std::vector<double2> h;
        xrl_status s = dots(a, 1, a, 1, h);
        out.resize(nrhs);
        for (int r = 0; r < nrhs; ++r) out[r] = std::sqrt(std::max(h[r].x, 0.0));
        return s;
    };
    auto setscale = [&](const std::vector<double>& sc) {
        for (auto& p : P) XRL_CUDA(cudaMemcpyAsync(p.ds.p, sc.data(), 8 * nrhs, cudaMemcpyHostToDevice, st));
    };
    auto fB = [](GPart& p) -> const float2* { return p.b; };
    auto fX = [](GPart& p) -> float2* { return p.x; };
    auto fW = [](GPart& p) -> float2* { return p.w.p; };
    auto fT = [](GPart& p) -> float2* { return p.tmp.p; };
    auto cW = [](GPart& p) -> const float2* { return p.w.p; };
    auto cT = [](GPart& p) -> const float2* { return p.tmp.p; };
    auto cX = [](GPart& p) -> const float2* { return p.x; };
    (void)fX;
    xrl_status s;
    // reference: ||M^-1 b|| (left: preconditioned RRE) or ||b|| (right / none)
    std::vector<double> bnorm, pbnorm;
    if ((s = norms(fB, bnorm))) return s;
    if (right) {
        pbnorm = bnorm;
    } else {
        for (auto& p : P) Mx(p, p.b, p.tmp.p);
        if ((s = norms(cT, pbnorm))) return s;
    }
    std::vector<int> iters(nrhs, 0), conv(nrhs, 0);
    std::vector<double> rre(nrhs, 1.0);
    for (int r = 0; r < nrhs; ++r)
        if (bnorm[r] == 0) { conv[r] = 1; rre[r] = 0; }
    int total = 0;
    while (total < maxit) {
        bool all = true;
        for (int r = 0; r < nrhs; ++r) all = all && conv[r];
        if (all) break;
        // r0 = M^-1 (b - A x) (left) or b - A x (right)
        if ((s = opA(cX, fW))) return s;
        for (auto& p : P) {
            if (!p.nl) continue;
            k_gsub<<<nblk(nrhs * p.nl, 256), 256, 0, st>>>(nrhs * p.nl, p.b, p.w.p, p.tmp.p);
            XRL_LAUNCH_CHECK();
            if (right) XRL_CUDA(cudaMemcpyAsync(p.w.p, p.tmp.p, 8 * nrhs * p.nl, cudaMemcpyDeviceToDevice, st));
            else Mx(p, p.tmp.p, p.w.p);
        }
        std::vector<double> beta;
        if ((s = norms(cW, beta))) return s;
        std::vector<double> sc(nrhs);
        for (int r = 0; r < nrhs; ++r) sc[r] = beta[r] > 0 ? 1.0 / beta[r] : 0.0;
        setscale(sc);
        for (auto& p : P)
            if (p.nl) {
                k_gscale<<<nblk(p.nl, 256), 256, 0, st>>>(p.nl, nrhs, p.w.p, p.nl, p.ds.p, p.V.p, (int64_t)(m + 1) * p.nl);
                XRL_LAUNCH_CHECK();
            }
        // per-column Hessenberg, Givens and residual vector (FP64 host)
        std::vector<std::vector<cd>> H(nrhs, std::vector<cd>((m + 1) * m, 0.0));
        std::vector<std::vector<cd>> g(nrhs, std::vector<cd>(m + 1, 0.0)), cs(nrhs, std::vector<cd>(m)), sn(nrhs, std::vector<cd>(m));
        for (int r = 0; r < nrhs; ++r) g[r][0] = beta[r];
        std::vector<int> jlen(nrhs, 0);
        std::vector<int> active(nrhs);
        for (int r = 0; r < nrhs; ++r) active[r] = !conv[r] && beta[r] > 0;
        int j = 0;
        for (; j < m && total < maxit; ++j, ++total) {
            bool any = false;
            for (int r = 0; r < nrhs; ++r) any = any || active[r];
            if (!any) break;
            // w = M^-1 A v_j (left) or A M^-1 v_j (right), batched over the columns
            for (auto& p : P)
                if (p.nl) {
                    k_gscale<<<nblk(p.nl, 256), 256, 0, st>>>(p.nl, nrhs, p.V.p + (int64_t)j * p.nl, (int64_t)(m + 1) * p.nl,
                                                              p.ones.p, p.tmp.p, p.nl);
                    XRL_LAUNCH_CHECK();
                }
            if (right) {
                for (auto& p : P) Mx(p, p.tmp.p, p.w.p);
                if ((s = opA(cW, fT))) return s;
                for (auto& p : P)
                    if (p.nl) XRL_CUDA(cudaMemcpyAsync(p.w.p, p.tmp.p, 8 * nrhs * p.nl, cudaMemcpyDeviceToDevice, st));
            } else {
                if ((s = opA(cT, fW))) return s;
                for (auto& p : P) {
                    Mx(p, p.w.p, p.tmp.p);
                    if (p.nl) XRL_CUDA(cudaMemcpyAsync(p.w.p, p.tmp.p, 8 * nrhs * p.nl, cudaMemcpyDeviceToDevice, st));
                }
            }
            // CGS2
            std::vector<std::vector<cd>> hcol(nrhs, std::vector<cd>(j + 2, 0.0));
            std::vector<double> hn;
            {
                // one host synchronisation per step: both projection passes and the norm stay on the device (the
                // update and the scale read the coefficients there; NCCL -- or, for virtual ranks, a device sum
                // over the parts -- adds them up across the ranks), then one copy of [h1 | h2 | |w|^2] feeds the
                // host's Hessenberg / Givens step
                const int ni = j + 1;
                const size_t o1 = 0, o2 = (size_t)nrhs * (m + 1), on = (size_t)2 * nrhs * (m + 1);
                auto reduce = [&](size_t off, int cnt) -> xrl_status {
                    if (nccl) return nccl_allreduce_sum_f64(ctx, (double*)(P[0].dc.p + off), (size_t)2 * cnt, st);
                    if (k > 1) {
                        k_sum_parts<<<nblk(cnt, 128), 128, 0, st>>>(k, dcptr.p, off, cnt);
                        XRL_LAUNCH_CHECK();
                    }
                    return XRL_OK;
                };
                for (int pass = 0; pass < 2; ++pass) {
                    const size_t off = pass ? o2 : o1;
                    for (auto& p : P) {
                        XRL_CUDA(cudaMemsetAsync(p.dc.p + off, 0, 16 * (size_t)nrhs * ni, st));
                        if (p.nl > 0) {
                            k_gdots<<<dim3(ni, nrhs, (unsigned)((p.nl + kDotChunk - 1) / kDotChunk)), 256, 0, st>>>(
                                p.nl, m + 1, p.V.p, p.w.p, p.dc.p + off, ni);
                            XRL_LAUNCH_CHECK();
                        }
                    }
                    if ((s = reduce(off, nrhs * ni))) return s;
                    for (auto& p : P)
                        if (p.nl > 0) {
                            k_gupdate<<<nblk(p.nl, 256), 256, 0, st>>>(p.nl, m + 1, nrhs, p.V.p, p.dc.p + off, ni, -1.f,
                                                                       p.w.p);
                            XRL_LAUNCH_CHECK();
                        }
                }
                for (auto& p : P) {
                    XRL_CUDA(cudaMemsetAsync(p.dc.p + on, 0, 16 * (size_t)nrhs, st));
                    if (p.nl > 0) {
                        k_gdots<<<dim3(1, nrhs, (unsigned)((p.nl + kDotChunk - 1) / kDotChunk)), 256, 0, st>>>(
                            p.nl, 1, p.w.p, p.w.p, p.dc.p + on, 1);
                        XRL_LAUNCH_CHECK();
                    }
                }
                if ((s = reduce(on, nrhs))) return s;
                for (auto& p : P) {
                    k_inv_norm<<<1, 32, 0, st>>>(nrhs, p.dc.p + on, p.ds.p);
                    XRL_LAUNCH_CHECK();
                    if (p.nl > 0) {
                        k_gscale<<<nblk(p.nl, 256), 256, 0, st>>>(p.nl, nrhs, p.w.p, p.nl, p.ds.p,
                                                                  p.V.p + (int64_t)(j + 1) * p.nl, (int64_t)(m + 1) * p.nl);
                        XRL_LAUNCH_CHECK();
                    }
                }
                std::vector<double2> hb((size_t)nrhs * (2 * (m + 1) + 1));
                XRL_CUDA(cudaMemcpyAsync(hb.data(), P[0].dc.p, 16 * hb.size(), cudaMemcpyDeviceToHost, st));
                XRL_CUDA(cudaStreamSynchronize(st));
                hn.resize(nrhs);
                for (int r = 0; r < nrhs; ++r) {
                    for (int i = 0; i <= j; ++i) {
                        const double2 a = hb[o1 + (size_t)r * ni + i], b2 = hb[o2 + (size_t)r * ni + i];
                        hcol[r][i] += cd(a.x + b2.x, a.y + b2.y);
                    }
                    hn[r] = std::sqrt(std::max(hb[on + r].x, 0.0));
                    hcol[r][j + 1] = hn[r];
                }
            }
            for (int r = 0; r < nrhs; ++r) {
                if (!active[r]) continue;
                auto& hc = hcol[r];
                for (int i = 0; i < j; ++i) {  // apply previous rotations
                    const cd a = hc[i], bb = hc[i + 1];
                    hc[i] = std::conj(cs[r][i]) * a + std::conj(sn[r][i]) * bb;
                    hc[i + 1] = -sn[r][i] * a + cs[r][i] * bb;
                }
                const double den = std::sqrt(std::norm(hc[j]) + std::norm(hc[j + 1]));
                cs[r][j] = den > 0 ? hc[j] / den : 1.0;
                sn[r][j] = den > 0 ? hc[j + 1] / den : 0.0;
                hc[j] = den;
                hc[j + 1] = 0;
                g[r][j + 1] = -sn[r][j] * g[r][j];
                g[r][j] = std::conj(cs[r][j]) * g[r][j];
                for (int i = 0; i <= j; ++i) H[r][(size_t)i * m + j] = hc[i];
                jlen[r] = j + 1;
                iters[r]++;
                rre[r] = std::abs(g[r][j + 1]) / (pbnorm[r] > 0 ? pbnorm[r] : 1.0);
                if (rre[r] < tol || hn[r] <= 1e-300) { conv[r] = 1; active[r] = 0; }
            }
        }
        // x += V y,  H y = g (upper triangular, per column)
        std::vector<double2> hy((size_t)nrhs * m, make_double2(0, 0));
        int jmax = 0;
        for (int r = 0; r < nrhs; ++r) {
            const int jl = jlen[r];
            jmax = std::max(jmax, jl);
            std::vector<cd> y(jl);
            for (int i = jl - 1; i >= 0; --i) {
                cd acc = g[r][i];
                for (int q = i + 1; q < jl; ++q) acc -= H[r][(size_t)i * m + q] * y[q];
                y[i] = acc / H[r][(size_t)i * m + i];
            }
            for (int i = 0; i < jl; ++i) hy[(size_t)r * m + i] = make_double2(y[i].real(), y[i].imag());
        }
        if (jmax > 0) {
            DBuf<double2> dy((size_t)nrhs * jmax);
            std::vector<double2> hy2((size_t)nrhs * jmax);
            for (int r = 0; r < nrhs; ++r)
                for (int i = 0; i < jmax; ++i) hy2[(size_t)r * jmax + i] = hy[(size_t)r * m + i];
            XRL_CUDA(cudaMemcpyAsync(dy.p, hy2.data(), 16 * hy2.size(), cudaMemcpyHostToDevice, st));
            for (auto& p : P) {
                if (!p.nl) continue;
                if (right) {  // x += M^-1 (V y)
                    XRL_CUDA(cudaMemsetAsync(p.tmp.p, 0, 8 * nrhs * p.nl, st));
                    k_gupdate<<<nblk(p.nl, 256), 256, 0, st>>>(p.nl, m + 1, nrhs, p.V.p, dy.p, jmax, 1.f, p.tmp.p);
                    XRL_LAUNCH_CHECK();
                    Mx(p, p.tmp.p, p.w.p);
                    k_gaxpy<<<nblk(nrhs * p.nl, 256), 256, 0, st>>>(nrhs * p.nl, p.w.p, p.x);
                    XRL_LAUNCH_CHECK();
                } else {
                    k_gupdate<<<nblk(p.nl, 256), 256, 0, st>>>(p.nl, m + 1, nrhs, p.V.p, dy.p, jmax, 1.f, p.x);
                    XRL_LAUNCH_CHECK();
                }
            }
            XRL_CUDA(cudaStreamSynchronize(st));
        }
        if (j == 0) break;
    }
    // true relative residual ||b - A x|| / ||b||
    if ((s = opA(cX, fW))) return s;
    for (auto& p : P)
        if (p.nl) {
            k_gsub<<<nblk(nrhs * p.nl, 256), 256, 0, st>>>(nrhs * p.nl, p.b, p.w.p, p.tmp.p);
            XRL_LAUNCH_CHECK();
        }
    std::vector<double> rn;
    if ((s = norms(cT, rn))) return s;
    bool all = true;
    for (int r = 0; r < nrhs; ++r) {
        if (iters_out) iters_out[r] = iters[r];
        if (rre_out) rre_out[r] = rre[r];
        if (true_rre_out) true_rre_out[r] = bnorm[r] > 0 ? rn[r] / bnorm[r] : 0.0;
        if (conv_out) conv_out[r] = conv[r];
        all = all && conv[r];
    }
    (void)sizeof(BufSel);
    return all ? XRL_OK : XRL_ENOCONV;
}

xrl_status xrl_gmres(xrl_op op, xrl_precond pc, const void* b_, void* x_, int32_t nrhs, const xrl_gmres_opts* opts,
                     int32_t* iters_out, double* rre_out, double* true_rre_out, int32_t* conv_out)
{
    if (!op || !b_ || !x_ || nrhs < 1) { set_error("xrl_gmres: bad argument"); return XRL_EINVAL; }
    if (pc && pc->op != op) { set_error("xrl_gmres: preconditioner built for another operator"); return XRL_EPROVENANCE; }
    if (op->part && op->tree->ctx->world == 1) {
        set_error("xrl_gmres: a virtual-rank operator runs through xrl_gmres_vranks");
        return XRL_EUNSUPPORTED;
    }
    API_TRY
        XRL_CUDA(cudaSetDevice(op->tree->ctx->device));
        std::vector<GPart> P(1);
        P[0].op = op;
        P[0].pc = pc;
        P[0].b = (const float2*)b_;
        P[0].x = (float2*)x_;
        P[0].nl = op->part ? op->part->nlo : op->topo->n_loops;
        return gmres_parts(P, op->part != nullptr, nrhs, opts, iters_out, rre_out, true_rre_out, conv_out);
    API_CATCH
}

xrl_status xrl_gmres_vranks(int32_t k, const xrl_op* ops, const xrl_precond* pcs, const void* const* b,
                            void* const* x, int32_t nrhs, const xrl_gmres_opts* opts, int32_t* iters_out,
                            double* rre_out, double* true_rre_out, int32_t* conv_out)
{
    xrl_status s = check_vrank_ops(k, ops, "xrl_gmres_vranks");
    if (s) return s;
    if (!b || !x || nrhs < 1) { set_error("xrl_gmres_vranks: bad argument"); return XRL_EINVAL; }
    for (int r = 0; r < k; ++r) {
        if (!b[r] || !x[r]) { set_error("xrl_gmres_vranks: null vector %d", r); return XRL_EINVAL; }
        if (pcs && (!pcs[r] != !pcs[0] || (pcs[r] && pcs[r]->op != ops[r]))) {
            set_error("xrl_gmres_vranks: preconditioner %d missing or built for another operator", r);
            return XRL_EPROVENANCE;
        }
    }
    API_TRY
        XRL_CUDA(cudaSetDevice(ops[0]->tree->ctx->device));
        std::vector<GPart> P(k);
        for (int r = 0; r < k; ++r) {
            P[r].op = ops[r];
            P[r].pc = pcs ? pcs[r] : nullptr;
            P[r].b = (const float2*)b[r];
            P[r].x = (float2*)x[r];
            P[r].nl = ops[r]->part ? ops[r]->part->nlo : ops[r]->topo->n_loops;
        }
        return gmres_parts(P, false, nrhs, opts, iters_out, rre_out, true_rre_out, conv_out);
    API_CATCH
}

}  // extern "C"
