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

// ---------------------------------------------------------------- segment format of the near SpMV
// (SURVEY §8(a) a12).  The owned rows' entries are cut into segments: a run of one row's (ascending) columns
// that share their upper 16 bits, at most kNearSegLen entries long.  A segment stores its row, the column
// base (upper bits) and per entry the FP32 value and the u16 lower column bits: 6 B per entry instead of
// 8 B for (int32 column, FP32 value).  Near columns of a Morton-ordered row are clustered, so a row has
// ~1.4 segments on config 4; the length cap bounds the work of the 8 lanes a segment gets.  Each segment's
// entries are padded to a multiple of 4 (value 0, offset repeated) for float4 / ushort4 loads and stored
// lane-interleaved within blocks of 32 (k_seg_fill), so a warp's gathers touch consecutive columns.

__global__ void k_seg_count(int64_t r0, int64_t nr, const int64_t* __restrict__ ptr, const int32_t* __restrict__ col,
                            int64_t* __restrict__ cnt)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nr) return;
    const int64_t r = r0 + i;
    int64_t c = 0;
    int len = 0, hi = -1;
    for (int64_t j = ptr[r]; j < ptr[r + 1]; ++j) {
        const int h = col[j] >> 16;
        if (h != hi || len == kNearSegLen) { ++c; hi = h; len = 0; }
        ++len;
    }
    cnt[i] = c;
}

__global__ void k_seg_emit(int64_t r0, int64_t nr, const int64_t* __restrict__ ptr, const int32_t* __restrict__ col,
                           const int64_t* __restrict__ start, int32_t* __restrict__ seg_row, int32_t* __restrict__ seg_base,
                           int64_t* __restrict__ seg_src, int32_t* __restrict__ seg_cnt, int64_t* __restrict__ seg_pad)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nr) return;
    const int64_t r = r0 + i;
    int64_t s = start[i] - 1;
    int len = 0, hi = -1;
    auto close = [&]() {
        if (s >= start[i]) { seg_cnt[s] = len; seg_pad[s] = (len + 3) & ~3; }
    };
    for (int64_t j = ptr[r]; j < ptr[r + 1]; ++j) {
        const int h = col[j] >> 16;
        if (h != hi || len == kNearSegLen) {
            close();
            ++s;
            seg_row[s] = (int32_t)i;
            seg_base[s] = h << 16;
            seg_src[s] = j;
            hi = h;
            len = 0;
        }
        ++len;
    }
    close();
}

// one warp per segment: FP32 values and u16 lower column bits; the padding repeats the last offset with
// value 0 (keeps every gather inside the segment's column block)
__global__ void k_seg_fill(int64_t nseg, const int32_t* __restrict__ seg_base, const int64_t* __restrict__ seg_src,
                           const int32_t* __restrict__ seg_cnt, const int64_t* __restrict__ seg_off,
                           const int32_t* __restrict__ col, const float* __restrict__ val, float* __restrict__ eval,
                           uint16_t* __restrict__ eoff)
{
    const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= nseg) return;
    const int64_t src = seg_src[s], dst = seg_off[s], padded = seg_off[s + 1] - dst;
    const int32_t base = seg_base[s];
    const int cnt = seg_cnt[s];
    for (int64_t i = lane; i < padded; i += 32) {
        // within each block of 32 stored entries (8 chunks of 4: one per lane of the segment), chunk l holds the
        // logical entries l, l + nc, l + 2 nc, l + 3 nc (nc = chunks in the block), so the 8 lanes' u-th
        // gathers hit 8 consecutive columns (one or two cache lines) instead of a strided set
        const int64_t blk = i & ~int64_t(31);
        const int nc = (int)((padded - blk < 32 ? padded - blk : 32) >> 2);
        const int q = (int)(i - blk), l = q >> 2, u = q & 3;
        const int64_t e = blk + u * nc + l;
        const int64_t j = src + (e < cnt ? e : cnt - 1);
        eval[dst + i] = e < cnt ? val[j] : 0.f;
        eoff[dst + i] = (uint16_t)(col[j] - base);
    }
}
}  // namespace

// Segment format (above) for the owned rows [t->p0, t->p1) of the CSR in N.
template <typename T>
static void exclusive_sum(const T* in, T* out, int64_t n, cudaStream_t st)
{
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int)n, st);
    DBuf<char> tmp(std::max<size_t>(tb, 1));
    XRL_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, (int)n, st));
}

static void build_near_segments(xrl_tree t, xrl_near N, cudaStream_t st)
{
    const int64_t r0 = t->p0, nr = t->p1 - t->p0;
    N->n_segs = 0;
    N->n_entries = 0;
    if (nr <= 0) {
        N->seg_off.alloc(1);
        XRL_CUDA(cudaMemsetAsync(N->seg_off.p, 0, 8, st));
        XRL_CUDA(cudaStreamSynchronize(st));
        return;
    }
    DBuf<int64_t> cnt(nr + 1), start(nr + 1);
    XRL_CUDA(cudaMemsetAsync(cnt.p + nr, 0, 8, st));
    k_seg_count<<<nblk(nr, 256), 256, 0, st>>>(r0, nr, N->row_ptr.p, N->col.p, cnt.p);
    XRL_LAUNCH_CHECK();
    exclusive_sum(cnt.p, start.p, nr + 1, st);
    int64_t nseg = 0;
    XRL_CUDA(cudaMemcpyAsync(&nseg, start.p + nr, 8, cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaStreamSynchronize(st));
    N->n_segs = nseg;
    N->seg_row.alloc(nseg);
    N->seg_base.alloc(nseg);
    N->seg_off.alloc(nseg + 1);
    DBuf<int64_t> src(nseg), pad(nseg + 1);
    DBuf<int32_t> scnt(nseg);
    XRL_CUDA(cudaMemsetAsync(pad.p + nseg, 0, 8, st));
    k_seg_emit<<<nblk(nr, 256), 256, 0, st>>>(r0, nr, N->row_ptr.p, N->col.p, start.p, N->seg_row.p, N->seg_base.p,
                                              src.p, scnt.p, pad.p);
    XRL_LAUNCH_CHECK();
    exclusive_sum(pad.p, N->seg_off.p, nseg + 1, st);
    XRL_CUDA(cudaMemcpyAsync(&N->n_entries, N->seg_off.p + nseg, 8, cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaStreamSynchronize(st));
    N->eval.alloc(std::max<int64_t>(4, N->n_entries));
    N->eoff.alloc(std::max<int64_t>(4, N->n_entries));
    k_seg_fill<<<nblk(nseg * 32, 256), 256, 0, st>>>(nseg, N->seg_base.p, src.p, scnt.p, N->seg_off.p, N->col.p,
                                                    N->val.p, N->eval.p, N->eoff.p);
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
    build_near_segments(t, N.get(), st);
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
