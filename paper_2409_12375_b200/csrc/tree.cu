// xrl_tree_build: geometry, Morton keys, radix sort, adaptive octree and the
// U/V/W/X interaction lists, all on the GPU (setup).
//
// PAPER.md:116 treats the panels as particles at their centroids (PAPER.md:56:
// centroids are the PEEC nodes), so the tree is built over centroids.  The
// paper gives no tree parameters (refs [22],[23] only); this build uses an
// adaptive octree (split while count > leaf_max), classical one-box
// separation and the adaptive U/V/W/X lists of Carrier-Greengard-Rokhlin.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <array>
#include <cmath>

#include "xrl_internal.h"

using namespace xrl;

namespace {

constexpr int kMortonBits = 21;

// ----------------------------------------------------------------- K1 geometry
// Correctly rounded FP64, no contraction: the near criterion downstream must
// reproduce the oracle's decisions bit for bit (reading R3).
// Panels: tri[stride*k + 0..2]; stride 4 with tri[4k+3] >= 0 is a rectangle (planar parallelogram
// a b c d in cyclic order): centroid = (a + c) * 0.5 (the diagonals' intersection),
// area = |(b-a) x (d-a)|, D = the longer diagonal (reading R16).
__device__ __forceinline__ double len_rn(const double* e)
{
    return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(e[0], e[0]), __dmul_rn(e[1], e[1])), __dmul_rn(e[2], e[2])));
}

__global__ void k_geometry(int64_t n, int64_t nv, const double* __restrict__ vert, const int32_t* __restrict__ tri,
                           int stride, double* cent, double* area, double* dmax, int* bad)
{
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    int i0 = tri[stride * k], i1 = tri[stride * k + 1], i2 = tri[stride * k + 2];
    const int i3 = stride == 4 ? tri[4 * k + 3] : -1;
    if (i0 < 0 || i1 < 0 || i2 < 0 || i0 >= nv || i1 >= nv || i2 >= nv || i3 >= nv) {
        atomicOr(bad, 1);
        return;
    }
    const double* a = vert + 3 * (int64_t)i0;
    const double* b = vert + 3 * (int64_t)i1;
    const double* c = vert + 3 * (int64_t)i2;
    if (i3 >= 0) {
        const double* q = vert + 3 * (int64_t)i3;
        double e1[3], e2[3], d1[3], d2[3], sk[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            cent[3 * k + d] = __dmul_rn(__dadd_rn(a[d], c[d]), 0.5);
            e1[d] = __dsub_rn(b[d], a[d]);
            e2[d] = __dsub_rn(q[d], a[d]);
            d1[d] = __dsub_rn(c[d], a[d]);
            d2[d] = __dsub_rn(q[d], b[d]);
            sk[d] = (c[d] - b[d]) - (q[d] - a[d]);  // parallelogram test: c - b == d - a
        }
        double cx = __dsub_rn(__dmul_rn(e1[1], e2[2]), __dmul_rn(e1[2], e2[1]));
        double cy = __dsub_rn(__dmul_rn(e1[2], e2[0]), __dmul_rn(e1[0], e2[2]));
        double cz = __dsub_rn(__dmul_rn(e1[0], e2[1]), __dmul_rn(e1[1], e2[0]));
        const double ar = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(cx, cx), __dmul_rn(cy, cy)), __dmul_rn(cz, cz)));
        const double l1 = len_rn(d1), l2 = len_rn(d2);
        dmax[k] = l1 > l2 ? l1 : l2;
        area[k] = ar;
        if (!(ar > 0.0)) atomicOr(bad, 2);
        // planar parallelogram: c - b == d - a within 1e-9 D
        const double tol = 1e-9 * (l1 > l2 ? l1 : l2);
        if (sqrt(sk[0] * sk[0] + sk[1] * sk[1] + sk[2] * sk[2]) > tol) atomicOr(bad, 8);  // (then planar too)
        return;
    }
    double e1[3], e2[3], e3[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        cent[3 * k + d] = __ddiv_rn(__dadd_rn(__dadd_rn(a[d], b[d]), c[d]), 3.0);
        e1[d] = __dsub_rn(b[d], a[d]);
        e2[d] = __dsub_rn(c[d], a[d]);
        e3[d] = __dsub_rn(c[d], b[d]);
    }
    double cx = __dsub_rn(__dmul_rn(e1[1], e2[2]), __dmul_rn(e1[2], e2[1]));
    double cy = __dsub_rn(__dmul_rn(e1[2], e2[0]), __dmul_rn(e1[0], e2[2]));
    double cz = __dsub_rn(__dmul_rn(e1[0], e2[1]), __dmul_rn(e1[1], e2[0]));
    double ar = __dmul_rn(0.5, __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(cx, cx), __dmul_rn(cy, cy)), __dmul_rn(cz, cz))));
    double l1 = len_rn(e1), l2 = len_rn(e2), l3 = len_rn(e3);
    double m = l1 > l2 ? l1 : l2;
    dmax[k] = m > l3 ? m : l3;
    area[k] = ar;
    if (!(ar > 0.0)) atomicOr(bad, 2);
}

__global__ void k_bbox(int64_t n, const double* __restrict__ cent, double* part /* [grid][6] */)
{
    double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            double v = cent[3 * k + d];
            mn[d] = fmin(mn[d], v);
            mx[d] = fmax(mx[d], v);
        }
    typedef cub::BlockReduce<double, 256> BR;
    __shared__ typename BR::TempStorage ts;
    for (int d = 0; d < 3; ++d) {
        double a = BR(ts).Reduce(mn[d], [](double x, double y) { return fmin(x, y); });
        __syncthreads();
        double b = BR(ts).Reduce(mx[d], [](double x, double y) { return fmax(x, y); });
        __syncthreads();
        if (threadIdx.x == 0) { part[6 * blockIdx.x + d] = a; part[6 * blockIdx.x + 3 + d] = b; }
    }
}

__device__ __forceinline__ uint64_t spread3(uint32_t v)
{
    uint64_t x = v & 0x1fffff;
    x = (x | x << 32) & 0x1f00000000ffffULL;
    x = (x | x << 16) & 0x1f0000ff0000ffULL;
    x = (x | x << 8) & 0x100f00f00f00f00fULL;
    x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
    x = (x | x << 2) & 0x1249249249249249ULL;
    return x;
}

// K2: 63-bit Morton key, bit group per level = bx | by<<1 | bz<<2.
__global__ void k_morton(int64_t n, const double* __restrict__ cent, double lo0, double lo1, double lo2, double invW,
                         uint64_t* key, int32_t* id)
{
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double lo[3] = {lo0, lo1, lo2};
    uint32_t q[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        double u = (cent[3 * k + d] - lo[d]) * invW * double(1 << kMortonBits);
        long long t = (long long)floor(u);
        t = t < 0 ? 0 : (t > (1 << kMortonBits) - 1 ? (1 << kMortonBits) - 1 : t);
        q[d] = (uint32_t)t;
    }
    key[k] = spread3(q[0]) | (spread3(q[1]) << 1) | (spread3(q[2]) << 2);
    id[k] = (int32_t)k;
}

__global__ void k_dup_check(int64_t n, const uint64_t* __restrict__ key, const int32_t* __restrict__ perm,
                            const double* __restrict__ cent_orig, int* bad)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* a = cent_orig + 3 * (int64_t)perm[i];
    for (int64_t j = i + 1; j < n && j < i + 32 && key[j] == key[i]; ++j) {
        const double* b = cent_orig + 3 * (int64_t)perm[j];
        if (a[0] == b[0] && a[1] == b[1] && a[2] == b[2]) atomicOr(bad, 4);
    }
}

__global__ void k_gather_panels(int64_t n, const int32_t* __restrict__ perm, const double* __restrict__ cent_o,
                                const double* __restrict__ area_o, const double* __restrict__ dmax_o,
                                const double* __restrict__ vert, const int32_t* __restrict__ tri, int stride,
                                double* cent, double* area, double* dmax, double* tv, int4* pvid, int32_t* iperm)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t k = perm[i];
    iperm[k] = (int32_t)i;
#pragma unroll
    for (int d = 0; d < 3; ++d) cent[3 * i + d] = cent_o[3 * k + d];
    area[i] = area_o[k];
    dmax[i] = dmax_o[k];
    const int v3 = stride == 4 ? tri[4 * k + 3] : -1;
    pvid[i] = make_int4(tri[stride * k], tri[stride * k + 1], tri[stride * k + 2], v3);
#pragma unroll
    for (int v = 0; v < 3; ++v)
#pragma unroll
        for (int d = 0; d < 3; ++d) tv[12 * i + 3 * v + d] = vert[3 * (int64_t)tri[stride * k + v] + d];
#pragma unroll
    for (int d = 0; d < 3; ++d) tv[12 * i + 9 + d] = v3 >= 0 ? vert[3 * (int64_t)v3 + d] : __longlong_as_double(0x7ff8000000000000LL);
}

// ----------------------------------------------------------------- K4 octree
struct LevelBoxes {
    DBuf<int32_t> ix, iy, iz, pb, pe, parent;
};

__global__ void k_split_count(int nb, int level, int leaf_max, int max_depth, const int32_t* __restrict__ pb,
                              const int32_t* __restrict__ pe, const uint64_t* __restrict__ key, int32_t* nch,
                              int32_t* bounds /* [nb][9] */)
{
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    int s = pb[b], e = pe[b];
    if (e - s <= leaf_max || level >= max_depth) { nch[b] = 0; return; }
    const int shift = 3 * (kMortonBits - level - 1);
    int cnt = 0;
    bounds[9 * b] = s;
    int lo = s;
    for (int o = 1; o < 8; ++o) {
        int l = lo, h = e;  // first index with octant >= o
        while (l < h) {
            int mid = (l + h) >> 1;
            if ((int)((key[mid] >> shift) & 7) < o) l = mid + 1; else h = mid;
        }
        bounds[9 * b + o] = l;
        if (l > lo) ++cnt;  // octant o-1 non-empty
        lo = l;
    }
    bounds[9 * b + 8] = e;
    if (e > lo) ++cnt;
    nch[b] = cnt;
}

__global__ void k_split_emit(int nb, int base, int next_base, const int32_t* __restrict__ ix, const int32_t* __restrict__ iy,
                             const int32_t* __restrict__ iz, const int32_t* __restrict__ nch,
                             const int32_t* __restrict__ coff, const int32_t* __restrict__ bounds, int32_t* cix,
                             int32_t* ciy, int32_t* ciz, int32_t* cpb, int32_t* cpe, int32_t* cpar, int32_t* first_child)
{
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    if (nch[b] == 0) { first_child[b] = -1; return; }
    int c = coff[b];
    first_child[b] = next_base + c;
    for (int o = 0; o < 8; ++o) {
        int s = bounds[9 * b + o], e = bounds[9 * b + o + 1];
        if (e <= s) continue;
        cix[c] = 2 * ix[b] + (o & 1);
        ciy[c] = 2 * iy[b] + ((o >> 1) & 1);
        ciz[c] = 2 * iz[b] + ((o >> 2) & 1);
        cpb[c] = s;
        cpe[c] = e;
        cpar[c] = base + b;
        ++c;
    }
}

// ----------------------------------------------------------------- K5 lists
constexpr int kMaxColl = 26;
constexpr int kMaxAdj = 26;
constexpr int kM2LChunk = 4096;   // target boxes per M2L tile chunk (L2 locality)

struct BoxView {
    const int32_t *level, *ix, *iy, *iz, *child, *nchild;
};

__device__ __forceinline__ bool adjacent_fine(int ax, int ay, int az, int la, int bx, int by, int bz, int lb)
{
    // box a at level la (finer or equal), b at level lb <= la; touching or overlapping
    int s = la - lb;
    int lo[3] = {bx << s, by << s, bz << s};
    int hi[3] = {(bx + 1) << s, (by + 1) << s, (bz + 1) << s};
    int a[3] = {ax, ay, az};
#pragma unroll
    for (int d = 0; d < 3; ++d)
        if (a[d] > hi[d] || a[d] + 1 < lo[d]) return false;
    return true;
}

// Level pass: colleagues, coarse adjacent leaves, and counts of V / X pairs.
__global__ void k_lists_level(int b0, int b1, BoxView bv, const int32_t* __restrict__ parent, int32_t* coll,
                              int32_t* ncoll, int32_t* adjc, int32_t* nadjc, int32_t* nV, int32_t* nX, int* overflow)
{
    int b = b0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= b1) return;
    const int P = parent[b];
    const int lb = bv.level[b], x = bv.ix[b], y = bv.iy[b], z = bv.iz[b];
    int nc = 0, na = 0, cv = 0, cx = 0;
    // same-level candidates: children of P's colleagues and of P itself
    for (int qi = -1; qi < ncoll[P]; ++qi) {
        int Q = qi < 0 ? P : coll[kMaxColl * P + qi];
        int c0 = bv.child[Q], nq = bv.nchild[Q];
        if (c0 < 0) continue;
        for (int c = c0; c < c0 + nq; ++c) {
            if (c == b) continue;
            int dx = x - bv.ix[c], dy = y - bv.iy[c], dz = z - bv.iz[c];
            if (abs(dx) <= 1 && abs(dy) <= 1 && abs(dz) <= 1) {
                if (nc < kMaxColl) coll[kMaxColl * b + nc] = c; else atomicOr(overflow, 1);
                ++nc;
            } else {
                ++cv;
            }
        }
    }
    // coarse leaves: adjc(P) and P's leaf colleagues
    for (int qi = 0; qi < nadjc[P] + ncoll[P]; ++qi) {
        int L = qi < nadjc[P] ? adjc[kMaxAdj * P + qi] : coll[kMaxColl * P + (qi - nadjc[P])];
        if (bv.child[L] >= 0) continue;  // only leaves
        if (adjacent_fine(x, y, z, lb, bv.ix[L], bv.iy[L], bv.iz[L], bv.level[L])) {
            if (na < kMaxAdj) adjc[kMaxAdj * b + na] = L; else atomicOr(overflow, 2);
            ++na;
        } else {
            ++cx;
        }
    }
    ncoll[b] = nc < kMaxColl ? nc : kMaxColl;
    nadjc[b] = na < kMaxAdj ? na : kMaxAdj;
    nV[b] = cv;
    nX[b] = cx;
}

// Emits V pairs (keyed for the M2L tile order) and classifies every X pair
// (b <- L, L a coarser leaf not adjacent to b, parent(b) adjacent to L) and
// its W dual (L <- b):
//   X kept as P2L only if b is not a leaf, else direct P2P (b <- L);
//   W kept as M2P only if b holds more than kWDirect panels, else P2P (L <- b).
// Direct evaluation is exact and cheaper than the expansion for small boxes.
// Unused slots hold kSent and sort to the end.
constexpr uint64_t kSent = ~0ull;
constexpr int kWDirect = 96;

__global__ void k_lists_emit(int nbox, BoxView bv, const int32_t* __restrict__ parent, const int32_t* __restrict__ coll,
                             const int32_t* __restrict__ ncoll, const int32_t* __restrict__ adjc,
                             const int32_t* __restrict__ nadjc, const int64_t* __restrict__ vptr,
                             const int64_t* __restrict__ xptr, const int32_t* __restrict__ pb,
                             const int32_t* __restrict__ pe, int32_t* vsrc, uint64_t* vkey, uint64_t* xkey,
                             uint64_t* wkey, uint64_t* ukx, uint64_t* ukw, const int* __restrict__ m2l_index)
{
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nbox || b == 0) return;
    const int P = parent[b];
    const int lb = bv.level[b], x = bv.ix[b], y = bv.iy[b], z = bv.iz[b];
    int64_t pv = vptr[b], px = xptr[b];
    for (int qi = 0; qi < ncoll[P]; ++qi) {
        int Q = coll[kMaxColl * P + qi];
        int c0 = bv.child[Q], nq = bv.nchild[Q];
        if (c0 < 0) continue;
        for (int c = c0; c < c0 + nq; ++c) {
            int dx = x - bv.ix[c], dy = y - bv.iy[c], dz = z - bv.iz[c];
            if (abs(dx) <= 1 && abs(dy) <= 1 && abs(dz) <= 1) continue;
            int off = m2l_index[(dx + 3) * 49 + (dy + 3) * 7 + (dz + 3)];
            vsrc[pv] = c;
            vkey[pv] = ((uint64_t)(b / kM2LChunk) << 41) | ((uint64_t)(uint32_t)off << 32) | (uint32_t)b;
            ++pv;
        }
    }
    const bool b_leaf = bv.child[b] < 0;
    const bool b_big = pe[b] - pb[b] > kWDirect;
    for (int qi = 0; qi < nadjc[P] + ncoll[P]; ++qi) {
        int L = qi < nadjc[P] ? adjc[kMaxAdj * P + qi] : coll[kMaxColl * P + (qi - nadjc[P])];
        if (bv.child[L] >= 0) continue;
        if (adjacent_fine(x, y, z, lb, bv.ix[L], bv.iy[L], bv.iz[L], bv.level[L])) continue;
        const uint64_t bl = ((uint64_t)(uint32_t)b << 32) | (uint32_t)L;
        const uint64_t lbk = ((uint64_t)(uint32_t)L << 32) | (uint32_t)b;
        xkey[px] = b_leaf ? kSent : bl;
        ukx[px] = b_leaf ? bl : kSent;
        wkey[px] = b_big ? lbk : kSent;
        ukw[px] = b_big ? kSent : lbk;
        ++px;
    }
}

__global__ void k_count_valid(int64_t n, const uint64_t* __restrict__ key, int64_t* out)
{
    // keys sorted ascending, sentinels last: out = first index holding kSent
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (key[mid] == kSent) hi = mid; else lo = mid + 1;
    }
    *out = lo;
}

// U pairs: per leaf b: self, leaf colleagues, coarse adjacent leaves (b <- L) and the reverse (L <- b).
__global__ void k_u_count(int nbox, const int32_t* __restrict__ child, const int32_t* __restrict__ coll,
                          const int32_t* __restrict__ ncoll, const int32_t* __restrict__ nadjc, int64_t* cnt)
{
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nbox) return;
    if (child[b] >= 0) { cnt[b] = 0; return; }
    int c = 1 + 2 * nadjc[b];
    for (int i = 0; i < ncoll[b]; ++i)
        if (child[coll[kMaxColl * b + i]] < 0) ++c;
    cnt[b] = c;
}

__global__ void k_u_emit(int nbox, const int32_t* __restrict__ child, const int32_t* __restrict__ coll,
                         const int32_t* __restrict__ ncoll, const int32_t* __restrict__ adjc,
                         const int32_t* __restrict__ nadjc, const int64_t* __restrict__ off, uint64_t* ukey)
{
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nbox || child[b] >= 0) return;
    int64_t p = off[b];
    auto put = [&](int t, int s) { ukey[p++] = ((uint64_t)(uint32_t)t << 32) | (uint32_t)s; };
    put(b, b);
    for (int i = 0; i < ncoll[b]; ++i) {
        int c = coll[kMaxColl * b + i];
        if (child[c] < 0) put(b, c);
    }
    for (int i = 0; i < nadjc[b]; ++i) {
        int L = adjc[kMaxAdj * b + i];
        put(b, L);
        put(L, b);
    }
}

__global__ void k_split_keys(int64_t n, const uint64_t* __restrict__ key, int32_t* hi, int32_t* lo)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (hi) hi[i] = (int32_t)(key[i] >> 32);
    lo[i] = (int32_t)(key[i] & 0xffffffffu);
}

// CSR row pointers from sorted target ids.
__global__ void k_csr_ptr(int64_t n, const int32_t* __restrict__ tgt, int nrows, int64_t* ptr)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    int a = (i == 0) ? -1 : tgt[i - 1];
    int b = (i == n) ? nrows : tgt[i];
    for (int r = a + 1; r <= b; ++r) ptr[r] = i;
}

__global__ void k_panel_leaf(int nleaf, const int32_t* __restrict__ leaves, const int32_t* __restrict__ pb,
                             const int32_t* __restrict__ pe, const int32_t* __restrict__ level,
                             const int32_t* __restrict__ ix, const int32_t* __restrict__ iy,
                             const int32_t* __restrict__ iz, const double* __restrict__ cent, double lo0, double lo1,
                             double lo2, double invW, int32_t* panel_leaf, float4* loc)
{
    int li = blockIdx.x;
    if (li >= nleaf) return;
    int b = leaves[li];
    double s = ldexp(1.0, -level[b]);
    double c[3] = {(ix[b] + 0.5) * s, (iy[b] + 0.5) * s, (iz[b] + 0.5) * s};
    const double lo[3] = {lo0, lo1, lo2};
    for (int i = pb[b] + threadIdx.x; i < pe[b]; i += blockDim.x) {
        panel_leaf[i] = b;
        float v[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) v[d] = (float)((cent[3 * (int64_t)i + d] - lo[d]) * invW - c[d]);
        loc[i] = make_float4(v[0], v[1], v[2], 0.f);
    }
}


__global__ void k_box_dmax(int nbox, const int32_t* __restrict__ pb, const int32_t* __restrict__ pe,
                           const double* __restrict__ dmax, double* bd)
{
    int b = blockIdx.x;
    if (b >= nbox) return;
    double m = 0;
    for (int i = pb[b] + threadIdx.x; i < pe[b]; i += blockDim.x) m = fmax(m, dmax[i]);
    typedef cub::BlockReduce<double, 128> BR;
    __shared__ typename BR::TempStorage ts;
    m = BR(ts).Reduce(m, [](double a, double c) { return fmax(a, c); });
    if (threadIdx.x == 0) bd[b] = m;
}

__global__ void k_p2p_count(int nleaf, const int32_t* __restrict__ leaves, const int32_t* __restrict__ pb,
                            const int32_t* __restrict__ pe, const int64_t* __restrict__ uptr,
                            const int32_t* __restrict__ usrc, unsigned long long* total)
{
    int li = blockIdx.x * blockDim.x + threadIdx.x;
    if (li >= nleaf) return;
    int b = leaves[li];
    long long nt = pe[b] - pb[b], s = 0;
    for (int64_t j = uptr[b]; j < uptr[b + 1]; ++j) s += pe[usrc[j]] - pb[usrc[j]];
    atomicAdd(total, (unsigned long long)(nt * s - nt));
}

template <typename KeyT, typename ValT>
void sort_pairs(KeyT* keys, ValT* vals, int64_t n, int end_bit, cudaStream_t st)
{
    if (n == 0) return;
    DBuf<KeyT> k2(n);
    DBuf<ValT> v2;
    if (vals) v2.alloc(n);
    size_t tb = 0;
    if (vals) {
        cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, k2.p, vals, v2.p, (int)n, 0, end_bit, st);
        DBuf<char> tmp(tb);
        XRL_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys, k2.p, vals, v2.p, (int)n, 0, end_bit, st));
        XRL_CUDA(cudaMemcpyAsync(vals, v2.p, n * sizeof(ValT), cudaMemcpyDeviceToDevice, st));
    } else {
        cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, k2.p, (int)n, 0, end_bit, st);
        DBuf<char> tmp(tb);
        XRL_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, keys, k2.p, (int)n, 0, end_bit, st));
    }
    XRL_CUDA(cudaMemcpyAsync(keys, k2.p, n * sizeof(KeyT), cudaMemcpyDeviceToDevice, st));
    XRL_CUDA(cudaStreamSynchronize(st));
}

template <typename T>
void exclusive_scan(const T* in, T* out, int64_t n, cudaStream_t st)
{
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int)n, st);
    DBuf<char> tmp(tb);
    XRL_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, (int)n, st));
    XRL_CUDA(cudaStreamSynchronize(st));
}

inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

// Static load balance of the persistent translation kernel (k_m2l_tc): CTA c of a grid of G takes blocks
// c, c + G, c + 2G, ...  Blocks (first tile, #tiles, operator, chunk) are assigned to the G CTAs by
// longest-processing-time (weight: its tiles + 1 for the 128 KB operator load), chunk after chunk so that
// all CTAs stay inside one L2-resident target chunk, and laid out in that strided order, padded with empty
// blocks (0 tiles; the kernel skips them).  Round-robin over runs of 1-16 tiles left the last CTA with up
// to twice the mean on small (per-rank) workloads.
std::vector<int4> balance_blocks(const std::vector<int4>& blocks, int G)
{
    if (blocks.empty() || G <= 1) return blocks;
    std::vector<std::vector<int4>> per(G);
    std::vector<int64_t> load(G, 0);
    size_t i = 0;
    while (i < blocks.size()) {
        size_t j = i;
        while (j < blocks.size() && blocks[j].w == blocks[i].w) ++j;  // one chunk
        std::vector<int4> ch(blocks.begin() + i, blocks.begin() + j);
        std::stable_sort(ch.begin(), ch.end(), [](const int4& a, const int4& b) { return a.y > b.y; });
        for (const int4& bk : ch) {
            const int c = (int)(std::min_element(load.begin(), load.end()) - load.begin());
            per[c].push_back(bk);
            load[c] += bk.y + 1;
        }
        i = j;
    }
    size_t len = 0;
    for (auto& v : per) len = std::max(len, v.size());
    std::vector<int4> out(len * G, make_int4(0, 0, 0, 0));
    for (int c = 0; c < G; ++c)
        for (size_t q = 0; q < per[c].size(); ++q) out[q * G + c] = per[c][q];
    return out;
}

}  // namespace

// ----------------------------------------------------------------- build
// Root placement of one candidate tree: centred on the bounding box, or at its low corner with the thinnest
// axis shifted down by `shift` x W (tree_build_checked searches these by the cost model).
struct RootPlace {
    bool centred = false;
    double shift = 0.0;
};

static xrl_status tree_build_impl(xrl_ctx ctx, int64_t n_vert, const double* vert_h, int64_t n, const int32_t* tri_h,
                                  int stride, const xrl_fmm_opts* opts, xrl_tree* out, RootPlace place,
                                  double* cost_only = nullptr)
{
    cudaStream_t st = ctx->stream;
    XRL_CUDA(cudaSetDevice(ctx->device));
    auto T = std::make_unique<xrl_tree_s>();
    T->ctx = ctx;
    struct CtxRef {
        xrl_ctx c;
        bool keep = false;
        ~CtxRef() { if (!keep) --c->refs; }
    } cref{ctx};
    ++ctx->refs;
    T->n = n;
    T->leaf_max = opts ? opts->leaf_max : 64;
    T->h_vert.assign(vert_h, vert_h + 3 * n_vert);
    T->stride = stride;
    T->h_tri.assign(tri_h, tri_h + (int64_t)stride * n);
    T->max_depth = opts ? opts->max_depth : kMortonBits;
    T->part_rank = ctx->world > 1 ? ctx->rank : (opts ? opts->part_rank : 0);
    T->part_world = ctx->world > 1 ? ctx->world : (opts && opts->part_world > 0 ? opts->part_world : 1);

    DBuf<double> vert(3 * n_vert);
    DBuf<int32_t> tri(stride * n);
    XRL_CUDA(cudaMemcpyAsync(vert.p, vert_h, vert.bytes(), cudaMemcpyHostToDevice, st));
    XRL_CUDA(cudaMemcpyAsync(tri.p, tri_h, tri.bytes(), cudaMemcpyHostToDevice, st));
    DBuf<double> cent_o(3 * n), area_o(n), dmax_o(n);
    DBuf<int> bad(1);
    XRL_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    k_geometry<<<nblk(n, 256), 256, 0, st>>>(n, n_vert, vert.p, tri.p, stride, cent_o.p, area_o.p, dmax_o.p, bad.p);
    XRL_LAUNCH_CHECK();
    int hbad = 0;
    XRL_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaStreamSynchronize(st));
    if (hbad & 1) { set_error("xrl_tree_build: vertex index out of range"); return XRL_EGEOM; }
    if (hbad & 2) { set_error("xrl_tree_build: zero-area panel"); return XRL_EGEOM; }
    if (hbad & 8) { set_error("xrl_tree_build: rectangle panel is not a planar parallelogram"); return XRL_EGEOM; }

    // XRL_SETUP_TIMES=1: per-section wall times of the build on stderr (the stream synchronised at each mark)
    static const bool setup_times = getenv("XRL_SETUP_TIMES") != nullptr;
    auto setup_t0 = std::chrono::steady_clock::now();
    auto setup_mark = [&](const char* what) {
        if (!setup_times) return;
        XRL_CUDA(cudaStreamSynchronize(st));
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "xrl setup: %-45s %8.1f ms\n", what,
                std::chrono::duration<double, std::milli>(now - setup_t0).count());
        setup_t0 = now;
    };
    setup_mark("start");
    // root cube
    const int nbb = 256;
    DBuf<double> part(6 * nbb);
    k_bbox<<<nbb, 256, 0, st>>>(n, cent_o.p, part.p);
    XRL_LAUNCH_CHECK();
    std::vector<double> hp(6 * nbb);
    XRL_CUDA(cudaMemcpyAsync(hp.data(), part.p, part.bytes(), cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaStreamSynchronize(st));
    double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
    for (int b = 0; b < nbb; ++b)
        for (int d = 0; d < 3; ++d) { mn[d] = std::min(mn[d], hp[6 * b + d]); mx[d] = std::max(mx[d], hp[6 * b + 3 + d]); }
    double ext = std::max({mx[0] - mn[0], mx[1] - mn[1], mx[2] - mn[2]});
    if (!(ext > 0)) ext = 1e-6;
    T->W = ext * (1.0 + 1e-6);
    // centred on the bounding box, or starting at its low corner (the thinnest axis optionally shifted down).
    // They differ only on axes thinner than the cube (the layers of a package): with the corner the top
    // levels never split the geometry in that axis, so the first Morton cuts -- the rank partition's cuts --
    // run across the layers, not between them (config 4 at 2 ranks: 35 k halo panels vs 0.78 M centred), and
    // the boxes cut the layer stack at different heights (tree_build_checked picks the cheapest placement)
    for (int d = 0; d < 3; ++d)
        T->lo[d] = place.centred ? 0.5 * (mn[d] + mx[d]) - 0.5 * T->W : mn[d] - 0.25e-6 * ext;
    if (!place.centred && place.shift > 0) {
        int dt = 0;
        for (int d = 1; d < 3; ++d) if (mx[d] - mn[d] < mx[dt] - mn[dt]) dt = d;
        if (mx[dt] - mn[dt] + place.shift * T->W < (1.0 - 1e-6) * T->W) T->lo[dt] = mn[dt] - place.shift * T->W;
        else if (cost_only) { *cost_only = 1e300; return XRL_OK; }  // the geometry would leave the cube
    }
    const double invW = 1.0 / T->W;

    setup_mark("root");
    // Morton keys + stable radix sort
    DBuf<uint64_t> key(n);
    DBuf<int32_t> id(n);
    k_morton<<<nblk(n, 256), 256, 0, st>>>(n, cent_o.p, T->lo[0], T->lo[1], T->lo[2], invW, key.p, id.p);
    XRL_LAUNCH_CHECK();
    sort_pairs(key.p, id.p, n, 63, st);
    T->perm = std::move(id);
    k_dup_check<<<nblk(n, 256), 256, 0, st>>>(n, key.p, T->perm.p, cent_o.p, bad.p);
    XRL_LAUNCH_CHECK();
    XRL_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaStreamSynchronize(st));
    if (hbad & 4) { set_error("xrl_tree_build: coincident centroids"); return XRL_EGEOM; }

    T->iperm.alloc(n);
    T->cent.alloc(3 * n);
    T->area.alloc(n);
    T->dmax.alloc(n);
    T->tverts.alloc(12 * n);
    T->pvid.alloc(n);
    k_gather_panels<<<nblk(n, 256), 256, 0, st>>>(n, T->perm.p, cent_o.p, area_o.p, dmax_o.p, vert.p, tri.p, stride,
                                                  T->cent.p, T->area.p, T->dmax.p, T->tverts.p, T->pvid.p,
                                                  T->iperm.p);
    XRL_LAUNCH_CHECK();

    setup_mark("morton sort");
    // octree, level by level
    std::vector<LevelBoxes> lv;
    std::vector<DBuf<int32_t>> lv_first_child;
    std::vector<int> cnt = {1};
    lv.emplace_back();
    {
        auto& L0 = lv[0];
        for (auto* b : {&L0.ix, &L0.iy, &L0.iz, &L0.pb, &L0.pe, &L0.parent}) b->alloc(1);
        int32_t z0 = 0, nn = (int32_t)n, m1 = -1;
        for (auto* b : {&L0.ix, &L0.iy, &L0.iz, &L0.pb})
            XRL_CUDA(cudaMemcpyAsync(b->p, &z0, 4, cudaMemcpyHostToDevice, st));
        XRL_CUDA(cudaMemcpyAsync(L0.pe.p, &nn, 4, cudaMemcpyHostToDevice, st));
        XRL_CUDA(cudaMemcpyAsync(L0.parent.p, &m1, 4, cudaMemcpyHostToDevice, st));
    }
    int base = 0;
    for (int l = 0;; ++l) {
        int nb = cnt[l];
        DBuf<int32_t> nch(nb), coff(nb), bounds(9 * (size_t)nb), fc(nb);
        k_split_count<<<nblk(nb, 128), 128, 0, st>>>(nb, l, T->leaf_max, T->max_depth, lv[l].pb.p, lv[l].pe.p,
                                                      key.p, nch.p, bounds.p);
        XRL_LAUNCH_CHECK();
        exclusive_scan(nch.p, coff.p, nb, st);
        int32_t last_c = 0, last_n = 0;
        XRL_CUDA(cudaMemcpyAsync(&last_c, coff.p + nb - 1, 4, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaMemcpyAsync(&last_n, nch.p + nb - 1, 4, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaStreamSynchronize(st));
        int nnext = last_c + last_n;
        LevelBoxes next;
        if (nnext > 0)
            for (auto* b : {&next.ix, &next.iy, &next.iz, &next.pb, &next.pe, &next.parent}) b->alloc(nnext);
        k_split_emit<<<nblk(nb, 128), 128, 0, st>>>(nb, base, base + nb, lv[l].ix.p, lv[l].iy.p, lv[l].iz.p, nch.p,
                                                     coff.p, bounds.p, next.ix.p, next.iy.p, next.iz.p, next.pb.p,
                                                     next.pe.p, next.parent.p, fc.p);
        XRL_LAUNCH_CHECK();
        lv_first_child.push_back(std::move(fc));
        base += nb;
        if (nnext == 0) break;
        cnt.push_back(nnext);
        lv.push_back(std::move(next));
    }
    const int nlev = (int)cnt.size();
    T->nlevel = nlev;
    T->lvl_start.assign(nlev + 1, 0);
    for (int l = 0; l < nlev; ++l) T->lvl_start[l + 1] = T->lvl_start[l] + cnt[l];
    const int nbox = T->lvl_start[nlev];
    T->nbox = nbox;
    for (auto* b : {&T->blevel, &T->bix, &T->biy, &T->biz, &T->bparent, &T->bchild, &T->bnchild, &T->bpb, &T->bpe})
        b->alloc(nbox);
    {
        std::vector<int32_t> hl(nbox);
        for (int l = 0; l < nlev; ++l)
            for (int i = T->lvl_start[l]; i < T->lvl_start[l + 1]; ++i) hl[i] = l;
        XRL_CUDA(cudaMemcpyAsync(T->blevel.p, hl.data(), 4 * nbox, cudaMemcpyHostToDevice, st));
        XRL_CUDA(cudaStreamSynchronize(st));
    }
    for (int l = 0; l < nlev; ++l) {
        size_t o = T->lvl_start[l], c = cnt[l];
        XRL_CUDA(cudaMemcpyAsync(T->bix.p + o, lv[l].ix.p, 4 * c, cudaMemcpyDeviceToDevice, st));
        XRL_CUDA(cudaMemcpyAsync(T->biy.p + o, lv[l].iy.p, 4 * c, cudaMemcpyDeviceToDevice, st));
        XRL_CUDA(cudaMemcpyAsync(T->biz.p + o, lv[l].iz.p, 4 * c, cudaMemcpyDeviceToDevice, st));
        XRL_CUDA(cudaMemcpyAsync(T->bpb.p + o, lv[l].pb.p, 4 * c, cudaMemcpyDeviceToDevice, st));
        XRL_CUDA(cudaMemcpyAsync(T->bpe.p + o, lv[l].pe.p, 4 * c, cudaMemcpyDeviceToDevice, st));
        XRL_CUDA(cudaMemcpyAsync(T->bparent.p + o, lv[l].parent.p, 4 * c, cudaMemcpyDeviceToDevice, st));
        XRL_CUDA(cudaMemcpyAsync(T->bchild.p + o, lv_first_child[l].p, 4 * c, cudaMemcpyDeviceToDevice, st));
    }
    // nchild from parents (host; setup only)
    std::vector<int32_t> hpar(nbox), hchild(nbox), hnch(nbox, 0), hpb(nbox), hpe(nbox);
    XRL_CUDA(cudaMemcpyAsync(hpar.data(), T->bparent.p, 4 * nbox, cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaMemcpyAsync(hchild.data(), T->bchild.p, 4 * nbox, cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaMemcpyAsync(hpb.data(), T->bpb.p, 4 * nbox, cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaMemcpyAsync(hpe.data(), T->bpe.p, 4 * nbox, cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaStreamSynchronize(st));
    for (int b = 1; b < nbox; ++b) hnch[hpar[b]]++;
    XRL_CUDA(cudaMemcpyAsync(T->bnchild.p, hnch.data(), 4 * nbox, cudaMemcpyHostToDevice, st));
    std::vector<int32_t> hleaves, hparents;
    T->par_start.assign(nlev + 1, 0);
    for (int l = 0; l < nlev; ++l) {
        T->par_start[l] = (int)hparents.size();
        for (int b = T->lvl_start[l]; b < T->lvl_start[l + 1]; ++b) {
            if (hchild[b] < 0) hleaves.push_back(b);
            else hparents.push_back(b);
        }
    }
    T->par_start[nlev] = (int)hparents.size();
    T->nleaf = (int)hleaves.size();
    T->leaves.alloc(T->nleaf);
    XRL_CUDA(cudaMemcpyAsync(T->leaves.p, hleaves.data(), 4 * hleaves.size(), cudaMemcpyHostToDevice, st));
    T->parents.alloc(std::max<size_t>(1, hparents.size()));
    if (!hparents.empty())
        XRL_CUDA(cudaMemcpyAsync(T->parents.p, hparents.data(), 4 * hparents.size(), cudaMemcpyHostToDevice, st));

    setup_mark("octree");
    // panel -> leaf, local coordinates, per-box max edge
    T->panel_leaf.alloc(n);
    T->loc.alloc(n);
    k_panel_leaf<<<T->nleaf, 128, 0, st>>>(T->nleaf, T->leaves.p, T->bpb.p, T->bpe.p, T->blevel.p, T->bix.p, T->biy.p,
                                           T->biz.p, T->cent.p, T->lo[0], T->lo[1], T->lo[2], invW,
                                           T->panel_leaf.p, T->loc.p);
    XRL_LAUNCH_CHECK();
    T->bdmax.alloc(nbox);
    k_box_dmax<<<nbox, 128, 0, st>>>(nbox, T->bpb.p, T->bpe.p, T->dmax.p, T->bdmax.p);
    XRL_LAUNCH_CHECK();

    setup_mark("local coords");
    // lists
    DBuf<int32_t> coll((size_t)kMaxColl * nbox), ncoll(nbox), adjc((size_t)kMaxAdj * nbox), nadjc(nbox);
    DBuf<int32_t> nV(nbox), nX(nbox);
    DBuf<int> ovf(1), m2l_index(343);
    XRL_CUDA(cudaMemsetAsync(ovf.p, 0, 4, st));
    XRL_CUDA(cudaMemsetAsync(ncoll.p, 0, 4 * nbox, st));
    XRL_CUDA(cudaMemsetAsync(nadjc.p, 0, 4 * nbox, st));
    XRL_CUDA(cudaMemsetAsync(nV.p, 0, 4 * nbox, st));
    XRL_CUDA(cudaMemsetAsync(nX.p, 0, 4 * nbox, st));
    XRL_CUDA(cudaMemcpyAsync(m2l_index.p, ctx->ops.m2l_index, 343 * 4, cudaMemcpyHostToDevice, st));
    BoxView bv{T->blevel.p, T->bix.p, T->biy.p, T->biz.p, T->bchild.p, T->bnchild.p};
    for (int l = 1; l < nlev; ++l) {
        int b0 = T->lvl_start[l], b1 = T->lvl_start[l + 1];
        k_lists_level<<<nblk(b1 - b0, 128), 128, 0, st>>>(b0, b1, bv, T->bparent.p, coll.p, ncoll.p, adjc.p, nadjc.p,
                                                          nV.p, nX.p, ovf.p);
        XRL_LAUNCH_CHECK();
    }
    int hovf = 0;
    XRL_CUDA(cudaMemcpyAsync(&hovf, ovf.p, 4, cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaStreamSynchronize(st));
    if (hovf) { set_error("xrl_tree_build: interaction list overflow (%d)", hovf); return XRL_EGEOM; }

    auto counts_to_ptr = [&](const int32_t* c32, DBuf<int64_t>& ptr, int rows) -> int64_t {
        DBuf<int64_t> c64(rows + 1);
        XRL_CUDA(cudaMemsetAsync(c64.p, 0, 8 * (rows + 1), st));
        // widen
        std::vector<int32_t> h(rows);
        XRL_CUDA(cudaMemcpyAsync(h.data(), c32, 4 * rows, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaStreamSynchronize(st));
        std::vector<int64_t> hp2(rows + 1, 0);
        for (int i = 0; i < rows; ++i) hp2[i + 1] = hp2[i] + h[i];
        ptr.alloc(rows + 1);
        XRL_CUDA(cudaMemcpyAsync(ptr.p, hp2.data(), 8 * (rows + 1), cudaMemcpyHostToDevice, st));
        XRL_CUDA(cudaStreamSynchronize(st));
        return hp2[rows];
    };
    T->nv = counts_to_ptr(nV.p, T->v_ptr, nbox);
    DBuf<int64_t> xcand_ptr;
    const int64_t nxc = counts_to_ptr(nX.p, xcand_ptr, nbox);  // X candidates (before classification)
    T->v_src.alloc(std::max<int64_t>(1, T->nv));
    DBuf<uint64_t> vkey(std::max<int64_t>(1, T->nv)), xkey(std::max<int64_t>(1, nxc)), wkey(std::max<int64_t>(1, nxc));
    DBuf<uint64_t> ukx(std::max<int64_t>(1, nxc)), ukw(std::max<int64_t>(1, nxc));
    k_lists_emit<<<nblk(nbox, 128), 128, 0, st>>>(nbox, bv, T->bparent.p, coll.p, ncoll.p, adjc.p, nadjc.p,
                                                  T->v_ptr.p, xcand_ptr.p, T->bpb.p, T->bpe.p, T->v_src.p, vkey.p,
                                                  xkey.p, wkey.p, ukx.p, ukw.p, m2l_index.p);
    XRL_LAUNCH_CHECK();
    DBuf<int64_t> dcount(1);
    auto sort_valid = [&](DBuf<uint64_t>& k, int64_t cnt) -> int64_t {
        if (cnt == 0) return 0;
        sort_pairs<uint64_t, int32_t>(k.p, nullptr, cnt, 64, st);
        k_count_valid<<<1, 1, 0, st>>>(cnt, k.p, dcount.p);
        XRL_LAUNCH_CHECK();
        int64_t h = 0;
        XRL_CUDA(cudaMemcpyAsync(&h, dcount.p, 8, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaStreamSynchronize(st));
        return h;
    };
    auto keys_to_csr = [&](const uint64_t* k, int64_t cnt, DBuf<int64_t>& ptr, DBuf<int32_t>& src) {
        ptr.alloc(nbox + 1);
        src.alloc(std::max<int64_t>(1, cnt));
        if (cnt == 0) { XRL_CUDA(cudaMemsetAsync(ptr.p, 0, 8 * (nbox + 1), st)); return; }
        DBuf<int32_t> tg(cnt);
        k_split_keys<<<nblk(cnt, 256), 256, 0, st>>>(cnt, k, tg.p, src.p);
        k_csr_ptr<<<nblk(cnt + 1, 256), 256, 0, st>>>(cnt, tg.p, nbox, ptr.p);
        XRL_LAUNCH_CHECK();
        XRL_CUDA(cudaStreamSynchronize(st));
    };
    T->nx = sort_valid(xkey, nxc);
    keys_to_csr(xkey.p, T->nx, T->x_ptr, T->x_src);
    T->nw = sort_valid(wkey, nxc);
    keys_to_csr(wkey.p, T->nw, T->w_ptr, T->w_src);
    const int64_t nukx = sort_valid(ukx, nxc);
    int64_t nukw = sort_valid(ukw, nxc);
    // Direct W pairs (L <- w) whose source box w is not a leaf: P2P re-bases
    // source panels relative to their own leaf, so expand w into its
    // descendant leaves (contiguous panel ranges in Morton order).
    DBuf<uint64_t> ukw_exp;
    if (nukw) {
        std::vector<uint64_t> hk(nukw);
        XRL_CUDA(cudaMemcpyAsync(hk.data(), ukw.p, 8 * nukw, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaStreamSynchronize(st));
        std::vector<std::pair<int32_t, int32_t>> lf;  // (pb, leaf id) sorted by pb
        for (int32_t b : hleaves) lf.push_back({hpb[b], b});
        std::sort(lf.begin(), lf.end());
        std::vector<uint64_t> ex;
        ex.reserve(nukw);
        for (uint64_t k : hk) {
            const int32_t t = (int32_t)(k >> 32), w = (int32_t)(k & 0xffffffffu);
            if (hchild[w] < 0) { ex.push_back(k); continue; }
            auto it = std::lower_bound(lf.begin(), lf.end(), std::make_pair(hpb[w], INT32_MIN));
            for (; it != lf.end() && it->first < hpe[w]; ++it)
                ex.push_back(((uint64_t)(uint32_t)t << 32) | (uint32_t)it->second);
        }
        nukw = (int64_t)ex.size();
        ukw_exp.alloc(nukw);
        XRL_CUDA(cudaMemcpyAsync(ukw_exp.p, ex.data(), 8 * nukw, cudaMemcpyHostToDevice, st));
        XRL_CUDA(cudaStreamSynchronize(st));
    }

    // U lists
    {
        DBuf<int64_t> ucnt(nbox), uoff(nbox);
        k_u_count<<<nblk(nbox, 128), 128, 0, st>>>(nbox, T->bchild.p, coll.p, ncoll.p, nadjc.p, ucnt.p);
        XRL_LAUNCH_CHECK();
        exclusive_scan(ucnt.p, uoff.p, nbox, st);
        int64_t lc = 0, lo_ = 0;
        XRL_CUDA(cudaMemcpyAsync(&lc, ucnt.p + nbox - 1, 8, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaMemcpyAsync(&lo_, uoff.p + nbox - 1, 8, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaStreamSynchronize(st));
        const int64_t nadj = lc + lo_;
        T->nu = nadj + nukx + nukw;
        DBuf<uint64_t> ukey(T->nu);
        k_u_emit<<<nblk(nbox, 128), 128, 0, st>>>(nbox, T->bchild.p, coll.p, ncoll.p, adjc.p, nadjc.p, uoff.p, ukey.p);
        XRL_LAUNCH_CHECK();
        if (nukx) XRL_CUDA(cudaMemcpyAsync(ukey.p + nadj, ukx.p, 8 * nukx, cudaMemcpyDeviceToDevice, st));
        if (nukw) XRL_CUDA(cudaMemcpyAsync(ukey.p + nadj + nukx, ukw_exp.p, 8 * nukw, cudaMemcpyDeviceToDevice, st));
        sort_pairs<uint64_t, int32_t>(ukey.p, nullptr, T->nu, 64, st);
        DBuf<int32_t> ut(T->nu);
        T->u_src.alloc(T->nu);
        T->u_ptr.alloc(nbox + 1);
        k_split_keys<<<nblk(T->nu, 256), 256, 0, st>>>(T->nu, ukey.p, ut.p, T->u_src.p);
        k_csr_ptr<<<nblk(T->nu + 1, 256), 256, 0, st>>>(T->nu, ut.p, nbox, T->u_ptr.p);
        XRL_LAUNCH_CHECK();
        DBuf<unsigned long long> tot(1);
        XRL_CUDA(cudaMemsetAsync(tot.p, 0, 8, st));
        k_p2p_count<<<nblk(T->nleaf, 128), 128, 0, st>>>(T->nleaf, T->leaves.p, T->bpb.p, T->bpe.p, T->u_ptr.p,
                                                         T->u_src.p, tot.p);
        XRL_LAUNCH_CHECK();
        unsigned long long ht = 0;
        XRL_CUDA(cudaMemcpyAsync(&ht, tot.p, 8, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaStreamSynchronize(st));
        T->np2p = (int64_t)ht;
    }
    setup_mark("lists");
    if (cost_only) {  // candidate evaluation: the MVM's cost model (P2P pairs, V-list pairs) only
        static const double wv = [] {  // XRL_COST_V (tuning): P2P pairs per V-list translation
            const char* e = getenv("XRL_COST_V");
            return e ? atof(e) : 1500.0;
        }();
        *cost_only = (double)T->np2p + wv * (double)T->nv;
        return XRL_OK;
    }
    // ---- partition over ranks: contiguous Morton ranges of
    // leaves balanced by estimated work; this rank owns panels [p0, p1).
    {
        std::vector<int64_t> hup(nbox + 1), hvp(nbox + 1);
        std::vector<int32_t> hus(std::max<int64_t>(1, T->nu));
        XRL_CUDA(cudaMemcpyAsync(hup.data(), T->u_ptr.p, 8 * (nbox + 1), cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaMemcpyAsync(hvp.data(), T->v_ptr.p, 8 * (nbox + 1), cudaMemcpyDeviceToHost, st));
        if (T->nu) XRL_CUDA(cudaMemcpyAsync(hus.data(), T->u_src.p, 4 * T->nu, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaStreamSynchronize(st));
        std::vector<std::pair<int32_t, int32_t>> lf;
        for (int32_t b : hleaves) lf.push_back({hpb[b], b});
        std::sort(lf.begin(), lf.end());
        std::vector<double> w(lf.size());
        // cost weights per M2L translation, per panel (P2M + L2P), per near nonzero, in P2P pairs (measured,
        // below); XRL_PART_W="a,b,c" overrides them (tuning)
        double cw[3] = {2.0, 0.7, 0.006};
        if (const char* e = getenv("XRL_PART_W")) sscanf(e, "%lf,%lf,%lf", &cw[0], &cw[1], &cw[2]);
        // near-field rows differ by an order of magnitude in length (coarse ground-plane panels see many fine
        // trace panels): a partitioned tree counts them (default eta) for the SpMV's share of the cost
        std::vector<int64_t> nnz_row;
        if (T->part_world > 1) nnz_row = near_row_counts(T.get(), 1.5, st);
        for (size_t i = 0; i < lf.size(); ++i) {
            const int L = lf[i].second;
            const double nL = hpe[L] - hpb[L];
            double src = 0;
            for (int64_t q = hup[L]; q < hup[L + 1]; ++q) src += hpe[hus[q]] - hpb[hus[q]];
            double m2l = 0;
            for (int a = L; a >= 0; a = hpar[a]) m2l += double(hvp[a + 1] - hvp[a]) * nL / double(hpe[a] - hpb[a]);
            // measured device costs on config 4 (B200), in units of one P2P pair (0.52 ns): an M2L translation on
            // tcgen05 ~1.05 ns = 2 pairs (175,692 flops at 168 TFLOP/s); P2M + L2P of a panel ~0.35 ns = 0.7; a near
            // nonzero 3.1 ps = 0.006
            double nnz = 0;
            if (!nnz_row.empty())
                for (int32_t p = hpb[L]; p < hpe[L]; ++p) nnz += (double)nnz_row[p];
            w[i] = nL * src + cw[0] * m2l + cw[1] * nL + cw[2] * nnz;
        }
        std::vector<int64_t> cuts(T->part_world + 1);
        xrl_partition_cuts((int64_t)w.size(), w.data(), T->part_world, cuts.data());
        const int64_t l0 = cuts[T->part_rank], l1 = cuts[T->part_rank + 1];
        T->p0 = l0 < (int64_t)lf.size() ? hpb[lf[l0].second] : (int32_t)n;
        T->p1 = l1 > l0 ? hpe[lf[l1 - 1].second] : T->p0;
        if (l1 <= l0) T->p1 = T->p0;
        T->part_cuts.resize(T->part_world + 1);
        for (int r = 0; r <= T->part_world; ++r)
            T->part_cuts[r] = cuts[r] < (int64_t)lf.size() ? hpb[lf[cuts[r]].second] : (int32_t)n;
        std::vector<int32_t> own;
        for (int64_t i = l0; i < l1; ++i) own.push_back(lf[i].second);
        T->n_own_leaves = (int)own.size();
        T->own_leaves.alloc(std::max<size_t>(1, own.size()));
        T->p2p_counter.alloc(1);
        if (!own.empty()) XRL_CUDA(cudaMemcpyAsync(T->own_leaves.p, own.data(), 4 * own.size(), cudaMemcpyHostToDevice, st));
        // P2P tasks: (leaf, target range), longest first (targets x U-list sources) so the dynamically
        // scheduled tasks end together (all P2P sources, 48 B per panel, stay resident in L2, so the order
        // costs no locality).  Leaves above 256 targets are cut into 256 + rest: with 8 targets per thread
        // a task of T <= 256 keeps >= 93 % of its 128 threads busy (T = 352 in one task: 69 %).
        {
            // (any leaf size: the first target is an absolute panel index, so a leaf of any size -- leaf_max
            // is unbounded -- is cut into as many 256-target tasks as it needs)
            std::vector<std::pair<int64_t, int4>> cost;
            for (int32_t L : own) {
                int64_t src = 0;
                for (int64_t q = hup[L]; q < hup[L + 1]; ++q) src += hpe[hus[q]] - hpb[hus[q]];
                const int nt = hpe[L] - hpb[L];
                for (int o = 0; o < nt;) {
#ifndef XRL_P2P_CUT
#define XRL_P2P_CUT 256
#endif
                    const int c = (nt - o > XRL_P2P_CUT) ? XRL_P2P_CUT : nt - o;
                    cost.push_back({-(int64_t)c * src, make_int4(L, hpb[L] + o, c, 0)});
                    o += c;
                }
            }
            std::stable_sort(cost.begin(), cost.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
            std::vector<int4> ord;
            for (auto& c : cost) ord.push_back(c.second);
            T->n_p2p_tasks = (int)ord.size();
            T->p2p_tasks.alloc(std::max<size_t>(1, ord.size()));
            if (!ord.empty())
                XRL_CUDA(cudaMemcpyAsync(T->p2p_tasks.p, ord.data(), sizeof(int4) * ord.size(), cudaMemcpyHostToDevice, st));
            XRL_CUDA(cudaStreamSynchronize(st));
        }
        // relevant boxes: panel range meets [p0, p1) (owned subtrees and their ancestors)
        T->rel.assign(nbox, 0);
        for (int b = 0; b < nbox; ++b) T->rel[b] = hpb[b] < T->p1 && hpe[b] > T->p0;
        // expansions to zero per MVM: multipoles of the relevant non-leaf boxes (the P2M overwrites the leaves'
        // whole records; LET boxes are overwritten by the exchange), local expansions of the relevant boxes
        {
            std::vector<int32_t> mz, ez;
            for (int b = 0; b < nbox; ++b)
                if (T->rel[b]) {
                    ez.push_back(b);
                    if (hchild[b] >= 0) mz.push_back(b);
                }
            T->n_mu_zero = (int32_t)mz.size();
            T->n_ell_zero = (int32_t)ez.size();
            T->mu_zero.alloc(std::max<size_t>(1, mz.size()));
            T->ell_zero.alloc(std::max<size_t>(1, ez.size()));
            if (!mz.empty()) XRL_CUDA(cudaMemcpyAsync(T->mu_zero.p, mz.data(), 4 * mz.size(), cudaMemcpyHostToDevice, st));
            if (!ez.empty()) XRL_CUDA(cudaMemcpyAsync(T->ell_zero.p, ez.data(), 4 * ez.size(), cudaMemcpyHostToDevice, st));
            XRL_CUDA(cudaStreamSynchronize(st));
        }
        // L2L lists per level (levels >= 3)
        std::vector<int32_t> l2l;
        T->l2l_start.assign(nlev + 1, 0);
        for (int l = 0; l < nlev; ++l) {
            T->l2l_start[l] = (int)l2l.size();
            if (l >= 3)
                for (int b = T->lvl_start[l]; b < T->lvl_start[l + 1]; ++b)
                    if (T->rel[b]) l2l.push_back(b);
        }
        T->l2l_start[nlev] = (int)l2l.size();
        T->l2l_boxes.alloc(std::max<size_t>(1, l2l.size()));
        if (!l2l.empty()) XRL_CUDA(cudaMemcpyAsync(T->l2l_boxes.p, l2l.data(), 4 * l2l.size(), cudaMemcpyHostToDevice, st));
        XRL_CUDA(cudaStreamSynchronize(st));
        // M2M and L2L as tensor-core translation tiles (the M2L kernel, operators 316.. in the image table):
        // per level, (target, source, octant operator) pairs sorted by (operator, target), tiles of <= 21
        // pairs of one operator, blocks of <= 16 tiles.  M2M: parent <- child for the relevant children
        // (a rank's P2M covers its own leaves only, so a box straddling a cut gets a partial multipole,
        // summed over the ranks per MVM, exchange.cu); L2L: child <- parent (relevant boxes of levels >= 3).
        std::vector<int32_t> hx(nbox), hy(nbox), hz(nbox), hpar(nbox), hch(nbox), hnc(nbox);
        XRL_CUDA(cudaMemcpyAsync(hx.data(), T->bix.p, 4 * nbox, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaMemcpyAsync(hy.data(), T->biy.p, 4 * nbox, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaMemcpyAsync(hz.data(), T->biz.p, 4 * nbox, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaMemcpyAsync(hpar.data(), T->bparent.p, 4 * nbox, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaMemcpyAsync(hch.data(), T->bchild.p, 4 * nbox, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaMemcpyAsync(hnc.data(), T->bnchild.p, 4 * nbox, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaStreamSynchronize(st));
        auto oct = [&](int b) { return (hx[b] & 1) | ((hy[b] & 1) << 1) | ((hz[b] & 1) << 2); };
        std::vector<int4> tiles, blocks;
        std::vector<int32_t> ptgt, psrc;
        auto emit_level = [&](std::vector<std::array<int, 3>>& pr) {  // (op, target, source)
            std::sort(pr.begin(), pr.end());
            const int first_block = (int)blocks.size();
            // tiles per block: up to 16 (one 128 KB operator load per block), fewer when the level has few tiles,
            // so that its blocks spread over all SMs (a rank's share of a level can be a few dozen tiles)
            int64_t ntile = 0;
            for (size_t i = 0, j; i < pr.size(); i = j) {
                for (j = i; j < pr.size() && pr[j][0] == pr[i][0]; ++j) {
                }
                ntile += (int64_t)(j - i + 20) / 21;
            }
            const int bt = (int)std::max<int64_t>(1, std::min<int64_t>(16, (ntile + ctx->num_sms - 1) / ctx->num_sms));
            size_t i = 0;
            while (i < pr.size()) {
                size_t j = i;
                while (j < pr.size() && pr[j][0] == pr[i][0]) ++j;
                for (size_t s0 = i; s0 < j; s0 += 21) {
                    if (s0 == i || blocks.back().y == bt) blocks.push_back(make_int4((int)tiles.size(), 0, pr[i][0], 0));
                    const int cnt = (int)std::min<size_t>(21, j - s0);
                    tiles.push_back(make_int4(pr[i][0], (int)ptgt.size(), cnt, 0));
                    for (int q = 0; q < cnt; ++q) { ptgt.push_back(pr[s0 + q][1]); psrc.push_back(pr[s0 + q][2]); }
                    blocks.back().y += 1;
                }
                i = j;
            }
            return std::make_pair(first_block, (int)blocks.size() - first_block);
        };
        // One launch per pass (all M2M levels bottom-up, all L2L levels top-down): each level's blocks are
        // LPT-balanced over the pass's persistent grid G and padded to whole rows of G, so the kernel knows a
        // block's level from its row; CTAs meet at a grid barrier between levels (k_m2l_tc).
        auto pack_pass = [&](std::vector<std::pair<int, int>>& lv, TransPass& P) {
            int G = 1;
            for (auto& r : lv) G = std::max(G, std::min(ctx->num_sms, r.second));
            std::vector<int4> out;
            std::vector<int32_t> rows(1, 0);
            for (auto& r : lv) {
                std::vector<int4> b(blocks.begin() + r.first, blocks.begin() + r.first + r.second);
                b = balance_blocks(b, G);
                if (!b.empty() && (int)b.size() < G) b.resize(G, make_int4(0, 0, 0, 0));
                out.insert(out.end(), b.begin(), b.end());
                rows.push_back(rows.back() + (int)(b.size() / G));
            }
            P.grid = G;
            P.nlev = (int)lv.size();
            P.nblocks = (int)out.size();
            P.rows_h = rows;
            return out;
        };
        T->m2m_lvl.assign(nlev, {0, 0});
        T->l2l_lvl.assign(nlev, {0, 0});
        for (int l = nlev - 2; l >= 2; --l) {  // parents at level l
            std::vector<std::array<int, 3>> pr;
            for (int b = T->lvl_start[l]; b < T->lvl_start[l + 1]; ++b)
                for (int c = hch[b]; hch[b] >= 0 && c < hch[b] + hnc[b]; ++c)
                    if (T->rel[c]) pr.push_back({kOpM2M + oct(c), b, c});  // (partial) multipoles of own subtrees
            T->m2m_lvl[l] = emit_level(pr);
        }
        for (int l = 3; l < nlev; ++l) {  // children at level l
            std::vector<std::array<int, 3>> pr;
            for (int q = T->l2l_start[l]; q < T->l2l_start[l + 1]; ++q) {
                const int c = l2l[q];
                pr.push_back({kOpL2L + oct(c), c, hpar[c]});
            }
            T->l2l_lvl[l] = emit_level(pr);
        }
        {
            std::vector<std::pair<int, int>> mlv, llv;
            for (int l = nlev - 2; l >= 2; --l) mlv.push_back(T->m2m_lvl[l]);
            for (int l = 3; l < nlev; ++l) llv.push_back(T->l2l_lvl[l]);
            std::vector<int4> mb = pack_pass(mlv, T->m2m_pass), lb = pack_pass(llv, T->l2l_pass);
            T->m2m_pass.first = 0;
            T->l2l_pass.first = (int)mb.size();
            blocks = mb;
            blocks.insert(blocks.end(), lb.begin(), lb.end());
            for (TransPass* P : {&T->m2m_pass, &T->l2l_pass}) {
                P->rows.alloc(P->rows_h.size());
                XRL_CUDA(cudaMemcpyAsync(P->rows.p, P->rows_h.data(), 4 * P->rows_h.size(), cudaMemcpyHostToDevice, st));
                P->done.alloc(std::max(1, P->nlev));
            }
            XRL_CUDA(cudaStreamSynchronize(st));
        }
        T->tr_tiles.alloc(std::max<size_t>(1, tiles.size()));
        T->tr_blocks.alloc(std::max<size_t>(1, blocks.size()));
        T->tr_tgt.alloc(std::max<size_t>(1, ptgt.size()));
        T->tr_src.alloc(std::max<size_t>(1, psrc.size()));
        if (!tiles.empty()) {
            XRL_CUDA(cudaMemcpyAsync(T->tr_tiles.p, tiles.data(), sizeof(int4) * tiles.size(), cudaMemcpyHostToDevice, st));
            XRL_CUDA(cudaMemcpyAsync(T->tr_blocks.p, blocks.data(), sizeof(int4) * blocks.size(), cudaMemcpyHostToDevice, st));
            XRL_CUDA(cudaMemcpyAsync(T->tr_tgt.p, ptgt.data(), 4 * ptgt.size(), cudaMemcpyHostToDevice, st));
            XRL_CUDA(cudaMemcpyAsync(T->tr_src.p, psrc.data(), 4 * psrc.size(), cudaMemcpyHostToDevice, st));
        }
        XRL_CUDA(cudaStreamSynchronize(st));
    }
    setup_mark("partition + P2P tasks + translation passes");
    // M2L pairs sorted by (offset, target)
    T->m2l_tgt.alloc(std::max<int64_t>(1, T->nv));
    T->m2l_srcb.alloc(std::max<int64_t>(1, T->nv));
    XRL_CUDA(cudaMemcpyAsync(T->m2l_srcb.p, T->v_src.p, 4 * T->nv, cudaMemcpyDeviceToDevice, st));
    sort_pairs(vkey.p, T->m2l_srcb.p, T->nv, 64, st);
    {
        DBuf<int32_t> offs(std::max<int64_t>(1, T->nv));
        if (T->nv) {
            k_split_keys<<<nblk(T->nv, 256), 256, 0, st>>>(T->nv, vkey.p, offs.p, T->m2l_tgt.p);
            XRL_LAUNCH_CHECK();
        }
        std::vector<int32_t> ho(T->nv), htg(T->nv), hsr(T->nv);
        if (T->nv) {
            XRL_CUDA(cudaMemcpyAsync(ho.data(), offs.p, 4 * T->nv, cudaMemcpyDeviceToHost, st));
            XRL_CUDA(cudaMemcpyAsync(htg.data(), T->m2l_tgt.p, 4 * T->nv, cudaMemcpyDeviceToHost, st));
            XRL_CUDA(cudaMemcpyAsync(hsr.data(), T->m2l_srcb.p, 4 * T->nv, cudaMemcpyDeviceToHost, st));
        }
        XRL_CUDA(cudaStreamSynchronize(st));
        if (T->part_world > 1) {  // keep only the translations into relevant target boxes
            int64_t k = 0;
            for (int64_t q = 0; q < T->nv; ++q)
                if (T->rel[htg[q]]) { ho[k] = ho[q]; htg[k] = htg[q]; hsr[k] = hsr[q]; ++k; }
            ho.resize(k); htg.resize(k); hsr.resize(k);
            if (k) {
                XRL_CUDA(cudaMemcpyAsync(T->m2l_tgt.p, htg.data(), 4 * k, cudaMemcpyHostToDevice, st));
                XRL_CUDA(cudaMemcpyAsync(T->m2l_srcb.p, hsr.data(), 4 * k, cudaMemcpyHostToDevice, st));
                XRL_CUDA(cudaStreamSynchronize(st));
            }
        }
        const int64_t nvk = (int64_t)ho.size();
        // tiles: <= 21 pairs of one (chunk, offset) group (one 128-row tcgen05 MMA group each);
        // blocks: runs of <= 16 tiles of one group (one operator load per block)
        std::vector<int4> tiles, blocks;
        const int TP = 21, BT = 16;
        int64_t i = 0;
        while (i < nvk) {
            int64_t j = i;
            while (j < nvk && ho[j] == ho[i]) ++j;  // same (chunk, offset)
            for (int64_t s = i; s < j; s += TP) {
                if ((int)tiles.size() == 0 || blocks.back().y == BT || blocks.back().z != (ho[i] & 511) ||
                    blocks.back().w != (ho[i] >> 9) || s == i)
                    blocks.push_back(make_int4((int)tiles.size(), 0, ho[i] & 511, ho[i] >> 9));
                tiles.push_back(make_int4(ho[i] & 511, (int)s, (int)std::min<int64_t>(TP, j - s), ho[i] >> 9));
                blocks.back().y += 1;
            }
            i = j;
        }
        T->n_m2l_tiles = (int)tiles.size();
        T->n_m2l_subtiles = (int64_t)tiles.size();  // one tcgen05 MMA group (M = N = K = 128) per tile
        T->m2l_tiles.alloc(std::max<size_t>(1, tiles.size()));
        if (!tiles.empty())
            XRL_CUDA(cudaMemcpyAsync(T->m2l_tiles.p, tiles.data(), sizeof(int4) * tiles.size(), cudaMemcpyHostToDevice, st));
        T->m2l_grid = std::min<int>(ctx->num_sms, (int)blocks.size());
        blocks = balance_blocks(blocks, T->m2l_grid);
        T->n_m2l_blocks = (int)blocks.size();
        T->m2l_blocks.alloc(std::max<size_t>(1, blocks.size()));
        if (!blocks.empty())
            XRL_CUDA(cudaMemcpyAsync(T->m2l_blocks.p, blocks.data(), sizeof(int4) * blocks.size(), cudaMemcpyHostToDevice, st));
        XRL_CUDA(cudaStreamSynchronize(st));  // host vectors go out of scope
    }
    setup_mark("M2L tiles");
    // X targets (boxes with kept P2L pairs)
    {
        std::vector<int64_t> hx(nbox + 1);
        XRL_CUDA(cudaMemcpyAsync(hx.data(), T->x_ptr.p, 8 * (nbox + 1), cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaStreamSynchronize(st));
        std::vector<int32_t> xt;
        for (int b = 0; b < nbox; ++b)
            if (hx[b + 1] > hx[b] && T->rel[b]) xt.push_back(b);
        T->n_x_targets = (int)xt.size();
        T->x_targets.alloc(std::max<size_t>(1, xt.size()));
        if (!xt.empty()) XRL_CUDA(cudaMemcpyAsync(T->x_targets.p, xt.data(), 4 * xt.size(), cudaMemcpyHostToDevice, st));
    }
    setup_mark("X");
    // W pairs of the owned leaves (M2P: one CTA per pair)
    {
        std::vector<int64_t> hw(nbox + 1);
        std::vector<int32_t> own(std::max(1, T->n_own_leaves));
        XRL_CUDA(cudaMemcpyAsync(hw.data(), T->w_ptr.p, 8 * (nbox + 1), cudaMemcpyDeviceToHost, st));
        if (T->n_own_leaves)
            XRL_CUDA(cudaMemcpyAsync(own.data(), T->own_leaves.p, 4 * T->n_own_leaves, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaStreamSynchronize(st));
        std::vector<int32_t> hws(std::max<int64_t>(1, T->nw));
        if (T->nw) XRL_CUDA(cudaMemcpyAsync(hws.data(), T->w_src.p, 4 * T->nw, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaStreamSynchronize(st));
        std::vector<int2> wp;  // (target leaf, source box) pairs of the owned leaves
        for (int i = 0; i < T->n_own_leaves; ++i)
            for (int64_t q = hw[own[i]]; q < hw[own[i] + 1]; ++q) wp.push_back(make_int2(own[i], hws[q]));
        T->n_w_targets = (int)wp.size();
        T->w_targets.alloc(std::max<size_t>(1, wp.size()));
        if (!wp.empty()) XRL_CUDA(cudaMemcpyAsync(T->w_targets.p, wp.data(), sizeof(int2) * wp.size(), cudaMemcpyHostToDevice, st));
        XRL_CUDA(cudaStreamSynchronize(st));
    }
    setup_mark("W");
    // multi-rank exchange plan: shared boxes, LET lists, remote leaves for the halo (exchange.cu)
    if (T->part_world > 1) {
        build_let_plan(T.get(), hpb, hpe, hchild, st);
        // the shared boxes this rank is not relevant to enter the all-reduce with a zero partial multipole
        std::vector<int32_t> mz(T->n_mu_zero);
        if (T->n_mu_zero) XRL_CUDA(cudaMemcpyAsync(mz.data(), T->mu_zero.p, 4 * mz.size(), cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaStreamSynchronize(st));
        for (int32_t b : T->shared_boxes)
            if (!T->rel[b]) mz.push_back(b);
        T->n_mu_zero = (int32_t)mz.size();
        T->mu_zero.alloc(std::max<size_t>(1, mz.size()));
        if (!mz.empty()) XRL_CUDA(cudaMemcpyAsync(T->mu_zero.p, mz.data(), 4 * mz.size(), cudaMemcpyHostToDevice, st));
        XRL_CUDA(cudaStreamSynchronize(st));
    }
    setup_mark("exchange plans");
    // MVM scratch
    T->mu.alloc((size_t)nbox * kMuStride);
    T->ell.alloc((size_t)nbox * kEllStride);
    T->xq.alloc((size_t)n * 8);
    XRL_CUDA(cudaMemsetAsync(T->mu.p, 0, T->mu.bytes(), st));
    XRL_CUDA(cudaMemsetAsync(T->xq.p, 0, T->xq.bytes(), st));
    XRL_CUDA(cudaStreamSynchronize(st));
    setup_mark("scratch");
    cref.keep = true;
    *out = T.release();
    return XRL_OK;
}

void xrl::tree_release(xrl_tree t)
{
    if (!t->dead || t->refs > 0) return;
    xrl_ctx ctx = t->ctx;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    delete t;
    --ctx->refs;
    ctx_release(ctx);
}

extern "C" {

xrl_status xrl_partition_cuts(int64_t n, const double* w, int32_t world, int64_t* cuts)
{
    if (n < 0 || world < 1 || !cuts || (n > 0 && !w)) { set_error("xrl_partition_cuts: bad argument"); return XRL_EINVAL; }
    double tot = 0;
    for (int64_t i = 0; i < n; ++i) tot += w[i] > 0 ? w[i] : 0;
    cuts[0] = 0;
    double acc = 0;
    int64_t i = 0;
    for (int r = 1; r < world; ++r) {
        const double target = tot * r / world;
        while (i < n && acc + 0.5 * (w[i] > 0 ? w[i] : 0) < target) { acc += w[i] > 0 ? w[i] : 0; ++i; }
        cuts[r] = i;
    }
    cuts[world] = n;
    return XRL_OK;
}

static xrl_status tree_build_checked(xrl_ctx ctx, int64_t n_vert, const double* vert, int64_t n_tri,
                                     const int32_t* tri, int stride, const xrl_fmm_opts* opts, xrl_tree* out);

xrl_status xrl_tree_build(xrl_ctx ctx, int64_t n_vert, const double* vert, int64_t n_tri, const int32_t* tri,
                          const xrl_fmm_opts* opts, xrl_tree* out)
{
    return tree_build_checked(ctx, n_vert, vert, n_tri, tri, 3, opts, out);
}

xrl_status xrl_tree_build_poly(xrl_ctx ctx, int64_t n_vert, const double* vert, int64_t n_panel, const int32_t* pv,
                               const xrl_fmm_opts* opts, xrl_tree* out)
{
    return tree_build_checked(ctx, n_vert, vert, n_panel, pv, 4, opts, out);
}

static xrl_status tree_build_checked(xrl_ctx ctx, int64_t n_vert, const double* vert, int64_t n_tri,
                                     const int32_t* tri, int stride, const xrl_fmm_opts* opts, xrl_tree* out)
{
    if (!ctx || !vert || !tri || !out) { set_error("xrl_tree_build: null argument"); return XRL_EINVAL; }
    *out = nullptr;
    if (n_tri < 1 || n_vert < 3 || n_tri > (int64_t)1 << 30) { set_error("xrl_tree_build: bad sizes"); return XRL_EINVAL; }
    if (opts) {
        if (opts->p != kP) { set_error("xrl_tree_build: p=%d not compiled (p=%d only)", opts->p, kP); return XRL_EUNSUPPORTED; }
        if (opts->leaf_max < 1) { set_error("xrl_tree_build: leaf_max < 1"); return XRL_EINVAL; }
        if (opts->max_depth < 1 || opts->max_depth > kMortonBits) { set_error("xrl_tree_build: max_depth"); return XRL_EINVAL; }
        if (ctx->world > 1 && (opts->part_world != ctx->world || opts->part_rank != ctx->rank)) {
            set_error("xrl_tree_build: part_rank/part_world must equal the context's rank/world");
            return XRL_EINVAL;
        }
        if (opts->part_world < 0 || (opts->part_world > 0 && (opts->part_rank < 0 || opts->part_rank >= opts->part_world))) {
            set_error("xrl_tree_build: bad part_rank/part_world");
            return XRL_EINVAL;
        }
    }
    try {
        // the root cube's placement is chosen by the MVM's cost model -- P2P pairs + 1500 x V-list pairs
        // (isolated on config 4: 0.49 ns per pair, 1.0 us per 3xFP16 translation, i.e. 2050 pairs; in the step
        // the M2L hosts 7 fused P2P warps, so a translation costs less than that: tools/cost_sweep.sh, weights
        // 1000 / 1500 give the same trees as 2180 at leaf 384 / 416, and avoid 2180's P2P-heavy pick at leaf 352:
        // 5.82 vs 6.79 ms).  Every rank of a
        // partition evaluates the same global candidates, so all ranks pick the same one.
        // XRL_ROOT_ALIGN=corner or centre skips the search.
        static const int forced = [] {
            const char* e = getenv("XRL_ROOT_ALIGN");
            return !e ? -1 : (e[0] == 'c' && e[1] == 'o') ? 0 : (e[0] == 'c') ? 1 : -1;
        }();
        RootPlace best;
        best.centred = forced == 1;
        if (forced < 0) {
            // candidates: centred, and the corner with the thinnest axis shifted by 0 .. 0.024 W; each is built
            // up to its interaction lists (about a third of a build) and costed, the cheapest is built in full
            // (config 4: leaf 384 5.49 -> 5.40 ms of modelled P2P + M2L, leaf 64 9.12 -> 8.39 ms)
            static const double shifts[] = {0.0, 0.002, 0.004, 0.006, 0.008, 0.012, 0.016, 0.024};
            double cbest = 1e301;
            for (int c = -1; c < (int)(sizeof(shifts) / sizeof(shifts[0])); ++c) {
                RootPlace pl;
                pl.centred = c < 0;
                pl.shift = c < 0 ? 0.0 : shifts[c];
                double cost = 1e300;
                xrl_tree dummy = nullptr;
                const xrl_status s = tree_build_impl(ctx, n_vert, vert, n_tri, tri, stride, opts, &dummy, pl, &cost);
                if (s != XRL_OK) return s;
                if (cost < cbest) { cbest = cost; best = pl; }
            }
        }
        return tree_build_impl(ctx, n_vert, vert, n_tri, tri, stride, opts, out, best);
    } catch (const CudaError& e) {
        return e.code;
    } catch (const std::bad_alloc&) {
        set_error("host out of memory");
        return XRL_ENOMEM;
    }
}

void xrl_tree_destroy(xrl_tree t)
{
    if (!t) return;
    t->dead = true;
    tree_release(t);
}

xrl_status xrl_tree_info(xrl_tree t, xrl_tree_info_t* info)
{
    if (!t || !info) { set_error("xrl_tree_info: null argument"); return XRL_EINVAL; }
    info->n = t->n;
    info->n_local = t->p1 - t->p0;
    info->offset = t->p0;
    info->n_boxes = t->nbox;
    info->n_leaves = t->nleaf;
    info->n_levels = t->nlevel;
    info->p = kP;
    info->n_v_pairs = t->nv;
    info->n_x_pairs = t->nx;
    info->n_w_pairs = t->nw;
    info->n_u_pairs = t->nu;
    info->n_p2p = t->np2p;
    for (int d = 0; d < 3; ++d) info->root_lo[d] = t->lo[d];
    info->root_width = t->W;
    info->n_m2l_tiles = t->n_m2l_tiles;
    info->n_m2l_subtiles = t->n_m2l_subtiles;
    return XRL_OK;
}

xrl_status xrl_tree_perm(xrl_tree t, int32_t* perm)
{
    if (!t || !perm) { set_error("xrl_tree_perm: null argument"); return XRL_EINVAL; }
    try {
        XRL_CUDA(cudaSetDevice(t->ctx->device));
        XRL_CUDA(cudaMemcpyAsync(perm, t->perm.p, 4 * t->n, cudaMemcpyDeviceToHost, t->ctx->stream));
        XRL_CUDA(cudaStreamSynchronize(t->ctx->stream));
        return XRL_OK;
    } catch (const CudaError& e) {
        return e.code;
    }
}

xrl_status xrl_tree_export(xrl_tree t, int32_t* box_level, int32_t* box_ijk, int32_t* box_parent, int32_t* box_pb,
                           int32_t* box_pe, int32_t* is_leaf, int64_t* u_ptr, int32_t* u_src, int64_t* v_ptr,
                           int32_t* v_src, int64_t* x_ptr, int32_t* x_src, int64_t* w_ptr, int32_t* w_src)
{
    if (!t) { set_error("xrl_tree_export: null tree"); return XRL_EINVAL; }
    try {
        cudaStream_t st = t->ctx->stream;
        XRL_CUDA(cudaSetDevice(t->ctx->device));
        const size_t nb = t->nbox;
        auto cp = [&](void* dst, const void* src, size_t bytes) {
            if (dst && bytes) XRL_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
        };
        cp(box_level, t->blevel.p, 4 * nb);
        cp(box_parent, t->bparent.p, 4 * nb);
        cp(box_pb, t->bpb.p, 4 * nb);
        cp(box_pe, t->bpe.p, 4 * nb);
        if (box_ijk) {
            std::vector<int32_t> a(nb), b(nb), c(nb);
            cp(a.data(), t->bix.p, 4 * nb);
            cp(b.data(), t->biy.p, 4 * nb);
            cp(c.data(), t->biz.p, 4 * nb);
            XRL_CUDA(cudaStreamSynchronize(st));
            for (size_t i = 0; i < nb; ++i) { box_ijk[3 * i] = a[i]; box_ijk[3 * i + 1] = b[i]; box_ijk[3 * i + 2] = c[i]; }
        }
        if (is_leaf) {
            std::vector<int32_t> ch(nb);
            cp(ch.data(), t->bchild.p, 4 * nb);
            XRL_CUDA(cudaStreamSynchronize(st));
            for (size_t i = 0; i < nb; ++i) is_leaf[i] = ch[i] < 0;
        }
        cp(u_ptr, t->u_ptr.p, 8 * (nb + 1));
        cp(u_src, t->u_src.p, 4 * t->nu);
        cp(v_ptr, t->v_ptr.p, 8 * (nb + 1));
        cp(v_src, t->v_src.p, 4 * t->nv);
        cp(x_ptr, t->x_ptr.p, 8 * (nb + 1));
        cp(x_src, t->x_src.p, 4 * t->nx);
        cp(w_ptr, t->w_ptr.p, 8 * (nb + 1));
        cp(w_src, t->w_src.p, 4 * t->nw);
        XRL_CUDA(cudaStreamSynchronize(st));
        return XRL_OK;
    } catch (const CudaError& e) {
        return e.code;
    }
}

}  // extern "C"
