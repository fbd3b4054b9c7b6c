// xrl_near_assemble: near-pair search over the octree and FP64 analytic
// single-triangle integrals -> near-field CSR.  Rectangle panels
// (hybrid meshes, NEXT f4) integrate as their two diagonal triangles; the optional
// Galerkin rule averages the self and vertex-adjacent entries over an
// outer quadrature of the observation panel (reading R17).
//
// the near-field matrix is filled directly on panel
// centroids (O(N_p)), with the Eq. 6 kernel.  Near pairs follow
// the geometric criterion of DESIGN.md reading R3; entries are the
// symmetrised collocation integrals of reading R2.  The far part 1/r is applied
// by the FMM, so the CSR stores the correction N_kl = P_kl - 1/|c_k - c_l| and
// the self term N_kk = P_kk.
#include <cub/cub.cuh>

#include <cmath>
#include <vector>

#include "xrl_internal.h"

using namespace xrl;

namespace {

struct V3 {
    double x, y, z;
};
__device__ __forceinline__ V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ V3 cross(V3 a, V3 b)
{
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ V3 scale(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ double norm(V3 a) { return sqrt(dot(a, a)); }

// Potential of a unit-density flat triangle at r: int_T dS'/|r - r'|.
// Edge decomposition: for each edge (a -> b) with tangent t, outward in-plane
// normal u = t x n, signed foot distance p = (a - rho).u, tangential
// coordinates s- = (a - rho).t, s+ = (b - rho).t, height h:
//   I = sum p ln[(R+ + s+)/(R- + s-)] - |h| sum [atan(p s+/(p^2+h^2+|h|R+)) - atan(p s-/(p^2+h^2+|h|R-))]
__device__ double tri_potential(V3 r, V3 v0, V3 v1, V3 v2)
{
    V3 n = cross(sub(v1, v0), sub(v2, v0));
    n = scale(n, 1.0 / norm(n));
    const double h = dot(sub(r, v0), n);
    const double ah = fabs(h);
    const V3 rho = sub(r, scale(n, h));
    const V3 vs[3] = {v0, v1, v2};
    double acc_log = 0.0, acc_ang = 0.0;
#pragma unroll
    for (int e = 0; e < 3; ++e) {
        const V3 a = vs[e], b = vs[(e + 1) % 3];
        V3 t = sub(b, a);
        t = scale(t, 1.0 / norm(t));
        const V3 u = cross(t, n);
        const V3 ar = sub(a, rho), br = sub(b, rho);
        const double p = dot(ar, u);
        if (p == 0.0) continue;
        const double sm = dot(ar, t), sp = dot(br, t);
        const double q2 = p * p + h * h;
        const double Rm = norm(sub(r, a)), Rp = norm(sub(r, b));
        double lg;
        if (sm >= 0.0) lg = log((Rp + sp) / (Rm + sm));
        else if (sp <= 0.0) lg = log((Rm - sm) / (Rp - sp));
        else lg = log((Rp + sp) * (Rm - sm) / q2);
        acc_log += p * lg;
        if (ah > 0.0) acc_ang += atan(p * sp / (q2 + ah * Rp)) - atan(p * sm / (q2 + ah * Rm));
    }
    return acc_log - ah * acc_ang;
}

// Near criterion, correctly rounded FP64 with no contraction (reading R3).
__device__ __forceinline__ bool is_near(const double* ck, const double* cl, double Dk, double Dl, double eta)
{
    double dx = __dsub_rn(ck[0], cl[0]), dy = __dsub_rn(ck[1], cl[1]), dz = __dsub_rn(ck[2], cl[2]);
    double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    double t = __dmul_rn(eta, Dk > Dl ? Dk : Dl);
    return d2 < __dmul_rn(t, t);
}

struct TreeView {
    const int32_t *level, *ix, *iy, *iz, *child, *nchild, *pb, *pe;
    const double* bdmax;
    const double* cent;
    const double* dmax;
    double lo0, lo1, lo2, W;
};

// Depth-first search from the root in Morton order; emits columns ascending.
template <bool FILL>
__global__ void k_near_search(int64_t n, TreeView tv, double eta, int64_t* cnt, const int64_t* __restrict__ ptr,
                              int32_t* cols, int* overflow)
{
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double* ck = tv.cent + 3 * k;
    const double Dk = tv.dmax[k];
    const double invW = 1.0 / tv.W;
    const double p[3] = {(ck[0] - tv.lo0) * invW, (ck[1] - tv.lo1) * invW, (ck[2] - tv.lo2) * invW};
    int stack[8 * 22 + 8];
    int sp = 0;
    stack[sp++] = 0;
    int64_t c = 0;
    int64_t out = FILL ? ptr[k] : 0;
    while (sp > 0) {
        int b = stack[--sp];
        double s = ldexp(1.0, -tv.level[b]);
        double bl[3] = {tv.ix[b] * s, tv.iy[b] * s, tv.iz[b] * s};
        double d2 = 0;
        for (int d = 0; d < 3; ++d) {
            double lo = bl[d] - 1e-9, hi = bl[d] + s + 1e-9;
            double q = p[d] < lo ? lo - p[d] : (p[d] > hi ? p[d] - hi : 0.0);
            d2 += q * q;
        }
        double R = eta * fmax(Dk, tv.bdmax[b]) * invW * (1.0 + 1e-6);
        if (d2 > R * R) continue;
        int c0 = tv.child[b];
        if (c0 >= 0) {
            int nc = tv.nchild[b];
            if (sp + nc > 8 * 22 + 8) { atomicOr(overflow, 1); return; }
            for (int j = nc - 1; j >= 0; --j) stack[sp++] = c0 + j;
        } else {
            for (int l = tv.pb[b]; l < tv.pe[b]; ++l) {
                if (l == k || is_near(ck, tv.cent + 3 * (int64_t)l, Dk, tv.dmax[l], eta)) {
                    if (FILL) cols[out + c] = l;
                    ++c;
                }
            }
        }
    }
    if (!FILL) cnt[k] = c;
}

// Panel l (library order): a triangle, or a rectangle as its triangles (v0, v1, v2) + (v0, v2, v3) split
// on the diagonal v0-v2 (the integral is additive; tverts' 4th vertex is NaN for triangles).
struct Panel {
    V3 v[4];
    bool quad;
};
__device__ __forceinline__ Panel load_panel(const double* __restrict__ tverts, int64_t l)
{
    const double* t = tverts + 12 * l;
    Panel P;
#pragma unroll
    for (int i = 0; i < 4; ++i) P.v[i] = {t[3 * i], t[3 * i + 1], t[3 * i + 2]};
    P.quad = !isnan(t[9]);
    return P;
}
__device__ __forceinline__ double panel_potential(V3 r, const Panel& P)
{
    double I = tri_potential(r, P.v[0], P.v[1], P.v[2]);
    if (P.quad) I += tri_potential(r, P.v[0], P.v[2], P.v[3]);
    return I;
}

// Galerkin near rule (NEXT f4): the mean of I(x; S_l) over the observation panel k by an outer
// quadrature -- Radon's 7-point degree-5 rule on a triangle (centroid weight 9/40; (a, a, 1 - 2a) with
// a = (6 -+ sqrt 15)/21, weights (155 -+ sqrt 15)/1200), the 2 x 2 Gauss product rule on a rectangle.
__device__ double galerkin_term(const Panel& K, const Panel& L)
{
    double s = 0.0;
    if (K.quad) {
        const double g[2] = {(1.0 - 1.0 / sqrt(3.0)) / 2.0, (1.0 + 1.0 / sqrt(3.0)) / 2.0};
        const V3 e1 = sub(K.v[1], K.v[0]), e2 = sub(K.v[3], K.v[0]);
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) {
                const V3 x = {K.v[0].x + g[i] * e1.x + g[j] * e2.x, K.v[0].y + g[i] * e1.y + g[j] * e2.y,
                              K.v[0].z + g[i] * e1.z + g[j] * e2.z};
                s += 0.25 * panel_potential(x, L);
            }
        return s;
    }
    const double s15 = sqrt(15.0);
    const double al[2] = {(6.0 - s15) / 21.0, (6.0 + s15) / 21.0};
    const double wt[2] = {(155.0 - s15) / 1200.0, (155.0 + s15) / 1200.0};
    const V3 c = {(K.v[0].x + K.v[1].x + K.v[2].x) / 3.0, (K.v[0].y + K.v[1].y + K.v[2].y) / 3.0,
                  (K.v[0].z + K.v[1].z + K.v[2].z) / 3.0};
    s = 9.0 / 40.0 * panel_potential(c, L);
    for (int q = 0; q < 2; ++q)
        for (int v = 0; v < 3; ++v) {
            const V3 A = K.v[v], B = K.v[(v + 1) % 3], C = K.v[(v + 2) % 3];
            const double b0 = 1.0 - 2.0 * al[q];
            const V3 x = {b0 * A.x + al[q] * B.x + al[q] * C.x, b0 * A.y + al[q] * B.y + al[q] * C.y,
                          b0 * A.z + al[q] * B.z + al[q] * C.z};
            s += wt[q] * panel_potential(x, L);
        }
    return s;
}

__device__ __forceinline__ bool share_vertex(int4 a, int4 b)
{
    const int va[4] = {a.x, a.y, a.z, a.w}, vb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (va[i] >= 0 && va[i] == vb[j]) return true;
    return false;
}

__global__ void k_near_values(int64_t n, const int64_t* __restrict__ ptr, const int32_t* __restrict__ cols,
                              const double* __restrict__ cent, const double* __restrict__ area,
                              const double* __restrict__ tverts, const int4* __restrict__ pvid, int galerkin,
                              float* val, double* val64)
{
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const Panel K = load_panel(tverts, k);
    const V3 ck = {cent[3 * k], cent[3 * k + 1], cent[3 * k + 2]};
    const double Ak = area[k];
    for (int64_t j = ptr[k]; j < ptr[k + 1]; ++j) {
        const int64_t l = cols[j];
        double v64, v32;
        if (l == k) {
            v64 = (galerkin ? galerkin_term(K, K) : panel_potential(ck, K)) / Ak;
            v32 = v64;
        } else {
            const Panel L = load_panel(tverts, l);
            const V3 cl = {cent[3 * l], cent[3 * l + 1], cent[3 * l + 2]};
            if (galerkin && share_vertex(pvid[k], pvid[l])) {
                v64 = 0.5 * (galerkin_term(K, L) / area[l] + galerkin_term(L, K) / Ak);
            } else {
                const double Ikl = panel_potential(ck, L) / area[l];
                const double Ilk = panel_potential(cl, K) / Ak;
                v64 = 0.5 * (Ikl + Ilk);
            }
            v32 = v64 - 1.0 / norm(sub(ck, cl));
        }
        val[j] = (float)v32;
        if (val64) val64[j] = v64;
    }
}

inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

// ---------------------------------------------------------------- row-group format of the near SpMV
// (SURVEY §8(a) a12).  The owned rows are taken in groups of kNearG = 4 consecutive rows (Morton order, so the
// rows of a group are neighbouring panels with overlapping near sets).  A group's columns are the sorted union
// of its rows' columns; per union column the format stores one float4 of the four rows' N values (0 where a row
// has no entry) and the u16 lower column bits.  The union is cut into segments: runs that share the upper 16
// column bits, at most kNearSegLen union columns long.  A segment stores its group, the column base and its
// slot offset.  One 32-byte charge gather then serves up to four rows (config 3: 2.6 entries per gather, 6.9 B
// per entry): the per-row format was bound by its L1 gather wavefronts (ncu, r03g: L1 87 % busy, 2.2 TB/s).
// Each segment is padded to a multiple of 4 slots (value 0, offset repeated).  Values are stored in the
// union's column order; the u16 offsets are lane-interleaved within blocks of 32 slots: with nc = (slots of
// the block) / 4, stored offset 4l + u is union column u nc + l, so lane l of a segment's 8 lanes reads its
// four offsets as one u64 and its u-th value at u nc + l (the 8 lanes' u-th loads and gathers are consecutive).

// visits the union columns of group g in ascending order: f(column, src[kNearG]) with src[i] the CSR entry of
// row 4g + i at that column, or -1
template <typename F>
__device__ __forceinline__ void rg_merge(int64_t r0, int64_t nr, int64_t g, const int64_t* __restrict__ ptr,
                                         const int32_t* __restrict__ col, F&& f)
{
    int64_t j[kNearG], e[kNearG];
#pragma unroll
    for (int i = 0; i < kNearG; ++i) {
        const int64_t r = kNearG * g + i;
        j[i] = r < nr ? ptr[r0 + r] : 0;
        e[i] = r < nr ? ptr[r0 + r + 1] : 0;
    }
    for (;;) {
        int32_t c = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < kNearG; ++i)
            if (j[i] < e[i]) c = min(c, col[j[i]]);
        if (c == 0x7fffffff) break;
        int64_t src[kNearG];
#pragma unroll
        for (int i = 0; i < kNearG; ++i) {
            src[i] = -1;
            if (j[i] < e[i] && col[j[i]] == c) src[i] = j[i]++;
        }
        f(c, src);
    }
}

__global__ void k_rg_count(int64_t r0, int64_t nr, int64_t ng, const int64_t* __restrict__ ptr,
                           const int32_t* __restrict__ col, int64_t* __restrict__ cnt)
{
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= ng) return;
    int64_t c = 0;
    int len = 0, hi = -1;
    rg_merge(r0, nr, g, ptr, col, [&](int32_t cl, const int64_t*) {
        const int h = cl >> 16;
        if (h != hi || len == kNearSegLen) { ++c; hi = h; len = 0; }
        ++len;
    });
    cnt[g] = c;
}

__global__ void k_rg_emit(int64_t r0, int64_t nr, int64_t ng, const int64_t* __restrict__ ptr,
                          const int32_t* __restrict__ col, const int64_t* __restrict__ start,
                          int32_t* __restrict__ seg_grp, int32_t* __restrict__ seg_base, int32_t* __restrict__ seg_cnt,
                          int64_t* __restrict__ seg_pad)
{
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= ng) return;
    int64_t s = start[g] - 1;
    int len = 0, hi = -1;
    auto close = [&]() {
        if (s >= start[g]) { seg_cnt[s] = len; seg_pad[s] = (len + 3) & ~3; }
    };
    rg_merge(r0, nr, g, ptr, col, [&](int32_t cl, const int64_t*) {
        const int h = cl >> 16;
        if (h != hi || len == kNearSegLen) {
            close();
            ++s;
            seg_grp[s] = (int32_t)g;
            seg_base[s] = h << 16;
            hi = h;
            len = 0;
        }
        ++len;
    });
    close();
}

// stored index of union column e of a segment with `padded` slots (offset interleave above)
__device__ __forceinline__ int64_t rg_off_slot(int64_t e, int64_t padded)
{
    const int64_t blk = e & ~int64_t(31);
    const int nc = (int)((padded - blk < 32 ? padded - blk : 32) >> 2);
    const int q = (int)(e - blk);
    return blk + 4 * (q % nc) + q / nc;
}

__global__ void k_rg_fill(int64_t r0, int64_t nr, int64_t ng, const int64_t* __restrict__ ptr,
                          const int32_t* __restrict__ col, const float* __restrict__ val,
                          const int64_t* __restrict__ start, const int32_t* __restrict__ seg_base,
                          const int32_t* __restrict__ seg_cnt, const int64_t* __restrict__ seg_off,
                          float4* __restrict__ gval, uint16_t* __restrict__ eoff)
{
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= ng) return;
    int64_t s = start[g];
    int64_t e = 0;
    uint16_t last = 0;
    auto pad = [&]() {  // padding slots of segment s (after its seg_cnt union columns)
        const int64_t dst = seg_off[s], padded = seg_off[s + 1] - dst;
        for (int64_t k = seg_cnt[s]; k < padded; ++k) {
            gval[dst + k] = make_float4(0.f, 0.f, 0.f, 0.f);
            eoff[dst + rg_off_slot(k, padded)] = last;
        }
    };
    rg_merge(r0, nr, g, ptr, col, [&](int32_t cl, const int64_t* src) {
        if (e == seg_cnt[s]) { pad(); ++s; e = 0; }
        const int64_t dst = seg_off[s], padded = seg_off[s + 1] - dst;
        float w[kNearG];
#pragma unroll
        for (int i = 0; i < kNearG; ++i) w[i] = src[i] >= 0 ? val[src[i]] : 0.f;
        gval[dst + e] = make_float4(w[0], w[1], w[2], w[3]);
        last = (uint16_t)(cl - seg_base[s]);
        eoff[dst + rg_off_slot(e, padded)] = last;
        ++e;
    });
    if (e > 0) pad();
}
}  // namespace

// Row-group format (above) for the owned rows [t->p0, t->p1) of the CSR in N.
template <typename T>
static void exclusive_sum(const T* in, T* out, int64_t n, cudaStream_t st)
{
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int)n, st);
    DBuf<char> tmp(std::max<size_t>(tb, 1));
    XRL_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, (int)n, st));
}

static void build_near_groups(xrl_tree t, xrl_near N, cudaStream_t st)
{
    static_assert(kNearG == 4, "the SpMV kernel reads one float4 of values per union column");
    const int64_t r0 = t->p0, nr = t->p1 - t->p0, ng = (nr + kNearG - 1) / kNearG;
    N->n_segs = 0;
    N->n_entries = 0;
    if (nr <= 0) {
        N->seg_off.alloc(1);
        XRL_CUDA(cudaMemsetAsync(N->seg_off.p, 0, 8, st));
        XRL_CUDA(cudaStreamSynchronize(st));
        return;
    }
    DBuf<int64_t> cnt(ng + 1), start(ng + 1);
    XRL_CUDA(cudaMemsetAsync(cnt.p + ng, 0, 8, st));
    k_rg_count<<<nblk(ng, 128), 128, 0, st>>>(r0, nr, ng, N->row_ptr.p, N->col.p, cnt.p);
    XRL_LAUNCH_CHECK();
    exclusive_sum(cnt.p, start.p, ng + 1, st);
    int64_t nseg = 0;
    XRL_CUDA(cudaMemcpyAsync(&nseg, start.p + ng, 8, cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaStreamSynchronize(st));
    N->n_segs = nseg;
    N->seg_grp.alloc(nseg);
    N->seg_base.alloc(nseg);
    N->seg_off.alloc(nseg + 1);
    DBuf<int64_t> pad(nseg + 1);
    DBuf<int32_t> scnt(nseg);
    XRL_CUDA(cudaMemsetAsync(pad.p + nseg, 0, 8, st));
    k_rg_emit<<<nblk(ng, 128), 128, 0, st>>>(r0, nr, ng, N->row_ptr.p, N->col.p, start.p, N->seg_grp.p,
                                             N->seg_base.p, scnt.p, pad.p);
    XRL_LAUNCH_CHECK();
    exclusive_sum(pad.p, N->seg_off.p, nseg + 1, st);
    XRL_CUDA(cudaMemcpyAsync(&N->n_entries, N->seg_off.p + nseg, 8, cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaStreamSynchronize(st));
    N->gval.alloc(std::max<int64_t>(4, N->n_entries));
    N->eoff.alloc(std::max<int64_t>(4, N->n_entries));
    k_rg_fill<<<nblk(ng, 128), 128, 0, st>>>(r0, nr, ng, N->row_ptr.p, N->col.p, N->val.p, start.p, N->seg_base.p,
                                             scnt.p, N->seg_off.p, N->gval.p, N->eoff.p);
    XRL_LAUNCH_CHECK();
    XRL_CUDA(cudaStreamSynchronize(st));
}

static xrl_status near_impl(xrl_tree t, double eta, int galerkin, xrl_near* out)
{
    xrl_ctx ctx = t->ctx;
    cudaStream_t st = ctx->stream;
    XRL_CUDA(cudaSetDevice(ctx->device));
    auto N = std::make_unique<xrl_near_s>();
    N->tree = t;
    N->eta = eta;
    const int64_t n = t->n;
    TreeView tv{t->blevel.p, t->bix.p, t->biy.p, t->biz.p, t->bchild.p, t->bnchild.p, t->bpb.p, t->bpe.p,
                t->bdmax.p, t->cent.p, t->dmax.p, t->lo[0], t->lo[1], t->lo[2], t->W};
    DBuf<int64_t> cnt(n);
    DBuf<int> ovf(1);
    XRL_CUDA(cudaMemsetAsync(ovf.p, 0, 4, st));
    k_near_search<false><<<nblk(n, 128), 128, 0, st>>>(n, tv, eta, cnt.p, nullptr, nullptr, ovf.p);
    XRL_LAUNCH_CHECK();
    std::vector<int64_t> hc(n), hp(n + 1, 0);
    XRL_CUDA(cudaMemcpyAsync(hc.data(), cnt.p, 8 * n, cudaMemcpyDeviceToHost, st));
    int hovf = 0;
    XRL_CUDA(cudaMemcpyAsync(&hovf, ovf.p, 4, cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaStreamSynchronize(st));
    if (hovf) { set_error("xrl_near_assemble: traversal stack overflow"); return XRL_EGEOM; }
    for (int64_t i = 0; i < n; ++i) hp[i + 1] = hp[i] + hc[i];
    N->nnz = hp[n];
    N->row_ptr.alloc(n + 1);
    N->col.alloc(std::max<int64_t>(1, N->nnz));
    N->val.alloc(std::max<int64_t>(1, N->nnz));
    N->val64.alloc(std::max<int64_t>(1, N->nnz));
    XRL_CUDA(cudaMemcpyAsync(N->row_ptr.p, hp.data(), 8 * (n + 1), cudaMemcpyHostToDevice, st));
    k_near_search<true><<<nblk(n, 128), 128, 0, st>>>(n, tv, eta, nullptr, N->row_ptr.p, N->col.p, ovf.p);
    XRL_LAUNCH_CHECK();
    k_near_values<<<nblk(n, 64), 64, 0, st>>>(n, N->row_ptr.p, N->col.p, t->cent.p, t->area.p, t->tverts.p,
                                              t->pvid.p, galerkin, N->val.p, N->val64.p);
    XRL_LAUNCH_CHECK();
    // the segment format the SpMV streams (owned rows)
    build_near_groups(t, N.get(), st);
    // the halo of x a partitioned tree's MVM exchanges (near columns + remote P2P / P2L leaves)
    if (t->part_world > 1) build_halo_plan(t, N.get(), st);
    ++t->refs;
    *out = N.release();
    return XRL_OK;
}

// Near-field row lengths (the first pass of the assembly) for the partition's cost model (tree.cu).
std::vector<int64_t> xrl::near_row_counts(xrl_tree t, double eta, cudaStream_t st)
{
    const int64_t n = t->n;
    TreeView tv{t->blevel.p, t->bix.p, t->biy.p, t->biz.p, t->bchild.p, t->bnchild.p, t->bpb.p, t->bpe.p,
                t->bdmax.p, t->cent.p, t->dmax.p, t->lo[0], t->lo[1], t->lo[2], t->W};
    DBuf<int64_t> cnt(n);
    DBuf<int> ovf(1);
    XRL_CUDA(cudaMemsetAsync(ovf.p, 0, 4, st));
    k_near_search<false><<<nblk(n, 128), 128, 0, st>>>(n, tv, eta, cnt.p, nullptr, nullptr, ovf.p);
    XRL_LAUNCH_CHECK();
    std::vector<int64_t> h(n);
    XRL_CUDA(cudaMemcpyAsync(h.data(), cnt.p, 8 * n, cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaStreamSynchronize(st));
    return h;
}

void xrl::near_release(xrl_near nr)
{
    if (!nr->dead || nr->refs > 0) return;
    xrl_tree t = nr->tree;
    cudaSetDevice(t->ctx->device);
    cudaStreamSynchronize(t->ctx->stream);
    delete nr;
    --t->refs;
    tree_release(t);
}

extern "C" {

xrl_status xrl_near_assemble(xrl_tree t, const xrl_near_opts* opts, xrl_near* out)
{
    if (!t || !out) { set_error("xrl_near_assemble: null argument"); return XRL_EINVAL; }
    *out = nullptr;
    double eta = opts ? opts->eta : 1.5;
    const int galerkin = opts ? opts->galerkin : 0;
    if (!(eta > 0)) { set_error("xrl_near_assemble: eta must be > 0"); return XRL_EINVAL; }
    if (galerkin != 0 && galerkin != 1) { set_error("xrl_near_assemble: galerkin must be 0 or 1"); return XRL_EINVAL; }
    try {
        return near_impl(t, eta, galerkin, out);
    } catch (const CudaError& e) {
        return e.code;
    } catch (const std::bad_alloc&) {
        set_error("host out of memory");
        return XRL_ENOMEM;
    }
}

void xrl_near_destroy(xrl_near nr)
{
    if (!nr) return;
    nr->dead = true;
    near_release(nr);  // deferred while operators built on it are alive
}

xrl_status xrl_near_export(xrl_near nr, int64_t* row_ptr, int32_t* col, float* val32, double* val64, int64_t* nnz)
{
    if (!nr) { set_error("xrl_near_export: null handle"); return XRL_EINVAL; }
    try {
        cudaStream_t st = nr->tree->ctx->stream;
        XRL_CUDA(cudaSetDevice(nr->tree->ctx->device));
        if (nnz) *nnz = nr->nnz;
        const int64_t n = nr->tree->n;
        if (row_ptr) XRL_CUDA(cudaMemcpyAsync(row_ptr, nr->row_ptr.p, 8 * (n + 1), cudaMemcpyDeviceToHost, st));
        if (col && nr->nnz) XRL_CUDA(cudaMemcpyAsync(col, nr->col.p, 4 * nr->nnz, cudaMemcpyDeviceToHost, st));
        if (val32 && nr->nnz) XRL_CUDA(cudaMemcpyAsync(val32, nr->val.p, 4 * nr->nnz, cudaMemcpyDeviceToHost, st));
        if (val64 && nr->nnz) XRL_CUDA(cudaMemcpyAsync(val64, nr->val64.p, 8 * nr->nnz, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaStreamSynchronize(st));
        return XRL_OK;
    } catch (const CudaError& e) {
        return e.code;
    }
}

xrl_status xrl_near_info(xrl_near nr, int64_t* nnz, int64_t* n_segments, int64_t* n_entries)
{
    if (!nr) { set_error("xrl_near_info: null handle"); return XRL_EINVAL; }
    if (nnz) *nnz = nr->nnz;
    if (n_segments) *n_segments = nr->n_segs;
    if (n_entries) *n_entries = nr->n_entries;
    return XRL_OK;
}

xrl_status xrl_near_export_rows(xrl_near nr, int64_t nrows, const int64_t* rows, int64_t* cnt, int32_t* col,
                                float* val32, double* val64)
{
    if (!nr || nrows < 0 || (nrows > 0 && (!rows || !cnt))) { set_error("xrl_near_export_rows: bad argument"); return XRL_EINVAL; }
    const int64_t n = nr->tree->n;
    for (int64_t i = 0; i < nrows; ++i)
        if (rows[i] < 0 || rows[i] >= n) { set_error("xrl_near_export_rows: row %lld out of range", (long long)rows[i]); return XRL_EINVAL; }
    try {
        cudaStream_t st = nr->tree->ctx->stream;
        XRL_CUDA(cudaSetDevice(nr->tree->ctx->device));
        std::vector<int64_t> ptr(n + 1);
        XRL_CUDA(cudaMemcpyAsync(ptr.data(), nr->row_ptr.p, 8 * (n + 1), cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaStreamSynchronize(st));
        int64_t off = 0;
        for (int64_t i = 0; i < nrows; ++i) {
            const int64_t b = ptr[rows[i]], c = ptr[rows[i] + 1] - b;
            cnt[i] = c;
            if (c > 0) {
                if (col) XRL_CUDA(cudaMemcpyAsync(col + off, nr->col.p + b, 4 * c, cudaMemcpyDeviceToHost, st));
                if (val32) XRL_CUDA(cudaMemcpyAsync(val32 + off, nr->val.p + b, 4 * c, cudaMemcpyDeviceToHost, st));
                if (val64) XRL_CUDA(cudaMemcpyAsync(val64 + off, nr->val64.p + b, 8 * c, cudaMemcpyDeviceToHost, st));
            }
            off += c;
        }
        XRL_CUDA(cudaStreamSynchronize(st));
        return XRL_OK;
    } catch (const CudaError& e) {
        return e.code;
    }
}

}  // extern "C"
