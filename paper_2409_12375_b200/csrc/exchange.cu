// Multi-GPU exchange plans of the sharded MVM and their pack / unpack kernels.
//
// Every rank builds the same tree; rank r owns the contiguous Morton range of leaves (panels
// [cut[r], cut[r+1])) the work-balanced partition gives it (tree.cu).  Per MVM a rank computes
//   * P2M for its own leaves and M2M for the boxes whose range meets its own (partial multipoles of the
//     boxes that straddle a cut: "shared" boxes, at most (world-1) per level);
//   * the shared boxes' multipoles are summed over the ranks (one small all-reduce: M2M is linear, so
//     the sum of the partial multipoles is the full one);
//   * the local-essential tree (LET): the multipoles of boxes wholly owned by another rank that appear
//     as M2L sources of its relevant boxes or as M2P (W-list) sources of its leaves, received from their
//     owner (grouped point-to-point);
//   * the halo of x: the charges of remote panels its P2P (U list), P2L (X list) and near-field rows
//     read, received from their owners before the P2P starts.
// Every rank derives every rank's lists from the shared tree and near pattern, so the send list of
// q -> r and the receive list of r <- q are the same ascending index list on both sides; no plan is
// exchanged at setup.  The exchanges themselves run over NCCL (comm.cu) on a multi-rank context, or as
// device copies between the trees of one process (xrl_mvm_vranks, "virtual ranks": the same plans and
// the same kernels on one GPU).
#include <cub/cub.cuh>

#include <algorithm>

#include "xrl_internal.h"

using namespace xrl;

namespace {

inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

// dst[i][0..w) = src[idx[i]][0..w)
__global__ void k_gather_rec(int64_t cnt, int w, const int32_t* __restrict__ idx, const float* __restrict__ src,
                             float* __restrict__ dst)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= cnt * w) return;
    const int64_t i = t / w;
    const int j = (int)(t - i * w);
    dst[t] = src[(int64_t)idx[i] * w + j];
}

// dst[idx[i]][0..w) = src[i][0..w)
__global__ void k_scatter_rec(int64_t cnt, int w, const int32_t* __restrict__ idx, const float* __restrict__ src,
                              float* __restrict__ dst)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= cnt * w) return;
    const int64_t i = t / w;
    const int j = (int)(t - i * w);
    dst[(int64_t)idx[i] * w + j] = src[t];
}

__global__ void k_add(int64_t cnt, const float* __restrict__ a, float* __restrict__ acc)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < cnt) acc[t] += a[t];
}

// mark[c] = 1 for the near columns c of rows [r0, r1) outside [r0, r1)
__global__ void k_mark_near_cols(int64_t r0, int64_t r1, const int64_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                 uint8_t* __restrict__ mark)
{
    const int64_t r = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= r1) return;
    for (int64_t j = ptr[r]; j < ptr[r + 1]; ++j) {
        const int32_t c = col[j];
        if (c < r0 || c >= r1) mark[c] = 1;
    }
}

// mark the panels of the given panel ranges [b, e)
__global__ void k_mark_ranges(int nr, const int2* __restrict__ rng, uint8_t* __restrict__ mark)
{
    const int2 q = rng[blockIdx.x];
    for (int i = q.x + threadIdx.x; i < q.y; i += blockDim.x) mark[i] = 1;
}

int owner_of(const std::vector<int32_t>& cut, int64_t p)
{
    // the largest r with cut[r] <= p (empty ranks have cut[r] == cut[r+1] and are skipped)
    return (int)(std::upper_bound(cut.begin(), cut.end() - 1, (int32_t)p) - cut.begin()) - 1;
}

template <typename T>
void upload(DBuf<T>& d, const std::vector<T>& h, cudaStream_t st)
{
    d.alloc(std::max<size_t>(1, h.size()));
    if (!h.empty()) XRL_CUDA(cudaMemcpyAsync(d.p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, st));
}

}  // namespace

namespace xrl {

// ---------------------------------------------------------------- plans
// Host core of the tree part of the plan (also exported as xrl_plan_exchange for the CPU tests): for every
// rank r the boxes straddling a cut (shared), the LET boxes r needs (M2L sources of its relevant boxes and
// M2P sources of its own leaves that are neither relevant to r nor shared, ascending) and the remote
// leaves its P2P (U list of its own leaves) and P2L (X list of its relevant boxes) read (ascending).
struct PlanCore {
    std::vector<int32_t> shared;
    std::vector<std::vector<int32_t>> let_need, halo_leaves;
};

static PlanCore plan_core(int nbox, const int32_t* pb, const int32_t* pe, const int32_t* child, const int64_t* vp,
                          const int32_t* vs, const int64_t* xp, const int32_t* xs, const int64_t* wp, const int32_t* ws,
                          const int64_t* up, const int32_t* us, const std::vector<int32_t>& cut)
{
    const int W = (int)cut.size() - 1;
    PlanCore P;
    std::vector<uint8_t> is_sh(nbox, 0);
    for (int b = 0; b < nbox; ++b)
        if (pe[b] > pb[b] && owner_of(cut, pb[b]) != owner_of(cut, pe[b] - 1)) { is_sh[b] = 1; P.shared.push_back(b); }
    P.let_need.assign(W, {});
    P.halo_leaves.assign(W, {});
    std::vector<uint8_t> seen(nbox);
    for (int r = 0; r < W; ++r) {
        const int32_t c0 = cut[r], c1 = cut[r + 1];
        auto rel = [&](int b) { return pb[b] < c1 && pe[b] > c0; };
        auto own = [&](int b) { return pb[b] >= c0 && pe[b] <= c1; };
        std::fill(seen.begin(), seen.end(), 0);
        std::vector<int32_t>& need = P.let_need[r];
        std::vector<int32_t>& hl = P.halo_leaves[r];
        auto need_mu = [&](int s) {
            if (!rel(s) && !is_sh[s] && !(seen[s] & 1)) { seen[s] |= 1; need.push_back(s); }
        };
        auto need_x = [&](int L) {
            if (!own(L) && !(seen[L] & 2)) { seen[L] |= 2; hl.push_back(L); }
        };
        for (int b = 0; b < nbox; ++b) {
            if (!rel(b)) continue;
            for (int64_t q = vp[b]; q < vp[b + 1]; ++q) need_mu(vs[q]);           // M2L sources
            for (int64_t q = xp[b]; q < xp[b + 1]; ++q) need_x(xs[q]);            // P2L source leaves
            if (child[b] < 0 && own(b)) {
                for (int64_t q = wp[b]; q < wp[b + 1]; ++q) need_mu(ws[q]);       // M2P sources
                for (int64_t q = up[b]; q < up[b + 1]; ++q) need_x(us[q]);        // P2P source leaves
            }
        }
        std::sort(need.begin(), need.end());
        std::sort(hl.begin(), hl.end());
    }
    return P;
}

// rank me's receive (from each owner q) and send (to each rank q) lists of the items need[r] (ascending),
// owned by the rank whose panel range holds key(item)
template <typename Key>
static void split_lists(const std::vector<std::vector<int32_t>>& need, int me, Key key, const std::vector<int32_t>& cut,
                        std::vector<int64_t>& roff, std::vector<int32_t>& ridx, std::vector<int64_t>& soff,
                        std::vector<int32_t>& sidx)
{
    const int W = (int)cut.size() - 1;
    roff.assign(W + 1, 0);
    soff.assign(W + 1, 0);
    ridx.clear();
    sidx.clear();
    for (int q = 0; q < W; ++q) {
        roff[q] = (int64_t)ridx.size();
        if (q != me)
            for (int32_t s : need[me])
                if (owner_of(cut, key(s)) == q) ridx.push_back(s);
        soff[q] = (int64_t)sidx.size();
        if (q != me)
            for (int32_t s : need[q])
                if (owner_of(cut, key(s)) == me) sidx.push_back(s);
    }
    roff[W] = (int64_t)ridx.size();
    soff[W] = (int64_t)sidx.size();
}

void build_let_plan(xrl_tree T, const std::vector<int32_t>& hpb, const std::vector<int32_t>& hpe,
                    const std::vector<int32_t>& hchild, cudaStream_t st)
{
    const int nbox = T->nbox;
    auto hcopy = [&](const auto* src, size_t cnt) {
        std::vector<std::remove_const_t<std::remove_pointer_t<decltype(src)>>> h(std::max<size_t>(1, cnt));
        if (cnt) XRL_CUDA(cudaMemcpyAsync(h.data(), src, sizeof(h[0]) * cnt, cudaMemcpyDeviceToHost, st));
        return h;
    };
    auto vp = hcopy(T->v_ptr.p, nbox + 1), xp = hcopy(T->x_ptr.p, nbox + 1), wp = hcopy(T->w_ptr.p, nbox + 1),
         up = hcopy(T->u_ptr.p, nbox + 1);
    auto vs = hcopy(T->v_src.p, T->nv), xs = hcopy(T->x_src.p, T->nx), ws = hcopy(T->w_src.p, T->nw),
         us = hcopy(T->u_src.p, T->nu);
    XRL_CUDA(cudaStreamSynchronize(st));
    PlanCore P = plan_core(nbox, hpb.data(), hpe.data(), hchild.data(), vp.data(), vs.data(), xp.data(), xs.data(),
                           wp.data(), ws.data(), up.data(), us.data(), T->part_cuts);
    T->shared_boxes = P.shared;
    upload(T->sh_idx, P.shared, st);
    T->sh_buf.alloc(std::max<size_t>(1, P.shared.size()) * kMuStride);
    T->halo_leaves = std::move(P.halo_leaves);
    std::vector<int32_t> ridx, sidx;
    split_lists(P.let_need, T->part_rank, [&](int32_t s) { return hpb[s]; }, T->part_cuts, T->let_roff, ridx,
                T->let_soff, sidx);
    upload(T->let_ridx, ridx, st);
    upload(T->let_sidx, sidx, st);
    T->let_rbuf.alloc(std::max<size_t>(1, ridx.size()) * kMuStride);
    T->let_sbuf.alloc(std::max<size_t>(1, sidx.size()) * kMuStride);
    XRL_CUDA(cudaStreamSynchronize(st));
}

void build_halo_plan(xrl_tree t, xrl_near N, cudaStream_t st)
{
    const int W = t->part_world, me = t->part_rank;
    const int64_t n = t->n;
    const std::vector<int32_t>& cut = t->part_cuts;
    std::vector<int32_t> hpb(t->nbox), hpe(t->nbox);
    XRL_CUDA(cudaMemcpyAsync(hpb.data(), t->bpb.p, 4 * t->nbox, cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaMemcpyAsync(hpe.data(), t->bpe.p, 4 * t->nbox, cudaMemcpyDeviceToHost, st));
    XRL_CUDA(cudaStreamSynchronize(st));
    DBuf<uint8_t> mark(n);
    DBuf<int32_t> sel(n), nsel(1);
    size_t tb = 0;
    cub::DeviceSelect::Flagged(nullptr, tb, cub::CountingInputIterator<int32_t>(0), mark.p, sel.p, nsel.p, (int)n, st);
    DBuf<char> tmp(tb);
    std::vector<int32_t> ridx, sidx;
    std::vector<std::vector<int32_t>> need(W);
    for (int r = 0; r < W; ++r) {
        // remote panels rank r reads: near columns of its rows, panels of its remote P2P / P2L leaves
        XRL_CUDA(cudaMemsetAsync(mark.p, 0, n, st));
        if (cut[r + 1] > cut[r])
            k_mark_near_cols<<<nblk(cut[r + 1] - cut[r], 128), 128, 0, st>>>(cut[r], cut[r + 1], N->row_ptr.p, N->col.p,
                                                                             mark.p);
        XRL_LAUNCH_CHECK();
        std::vector<int2> rg;
        for (int32_t L : t->halo_leaves[r]) rg.push_back(make_int2(hpb[L], hpe[L]));
        DBuf<int2> drg;
        if (!rg.empty()) {
            upload(drg, rg, st);
            k_mark_ranges<<<(int)rg.size(), 128, 0, st>>>((int)rg.size(), drg.p, mark.p);
            XRL_LAUNCH_CHECK();
        }
        XRL_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, cub::CountingInputIterator<int32_t>(0), mark.p, sel.p, nsel.p,
                                            (int)n, st));
        int32_t cnt = 0;
        XRL_CUDA(cudaMemcpyAsync(&cnt, nsel.p, 4, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaStreamSynchronize(st));
        need[r].resize(cnt);
        if (cnt) XRL_CUDA(cudaMemcpyAsync(need[r].data(), sel.p, 4 * (size_t)cnt, cudaMemcpyDeviceToHost, st));
        XRL_CUDA(cudaStreamSynchronize(st));
    }
    split_lists(need, me, [](int32_t p) { return p; }, cut, N->halo_roff, ridx, N->halo_soff, sidx);
    upload(N->halo_ridx, ridx, st);
    upload(N->halo_sidx, sidx, st);
    N->halo_rbuf.alloc(std::max<size_t>(1, ridx.size()) * 8);
    N->halo_sbuf.alloc(std::max<size_t>(1, sidx.size()) * 8);
    XRL_CUDA(cudaStreamSynchronize(st));
}

// ---------------------------------------------------------------- per-MVM pack / unpack
void gather_records(int64_t cnt, int w, const int32_t* idx, const float* src, float* dst, cudaStream_t st)
{
    if (cnt <= 0) return;
    k_gather_rec<<<nblk(cnt * w, 256), 256, 0, st>>>(cnt, w, idx, src, dst);
    XRL_LAUNCH_CHECK();
}

void scatter_records(int64_t cnt, int w, const int32_t* idx, const float* src, float* dst, cudaStream_t st)
{
    if (cnt <= 0) return;
    k_scatter_rec<<<nblk(cnt * w, 256), 256, 0, st>>>(cnt, w, idx, src, dst);
    XRL_LAUNCH_CHECK();
}

void add_into(int64_t cnt, const float* a, float* acc, cudaStream_t st)
{
    if (cnt <= 0) return;
    k_add<<<nblk(cnt, 256), 256, 0, st>>>(cnt, a, acc);
    XRL_LAUNCH_CHECK();
}

}  // namespace xrl

// ---------------------------------------------------------------- host ABI (CPU tests of the plans)
extern "C" xrl_status xrl_plan_exchange(int32_t nbox, const int32_t* pb, const int32_t* pe, const int32_t* child,
                                        const int64_t* v_ptr, const int32_t* v_src, const int64_t* x_ptr,
                                        const int32_t* x_src, const int64_t* w_ptr, const int32_t* w_src,
                                        const int64_t* u_ptr, const int32_t* u_src, int64_t n, const int64_t* near_ptr,
                                        const int32_t* near_col, int32_t world, const int32_t* cuts, int32_t rank,
                                        int64_t* n_shared, int32_t* shared, int64_t* let_roff, int32_t* let_ridx,
                                        int64_t* let_soff, int32_t* let_sidx, int64_t* halo_roff, int32_t* halo_ridx,
                                        int64_t* halo_soff, int32_t* halo_sidx)
{
    if (nbox < 1 || !pb || !pe || !child || !v_ptr || !x_ptr || !w_ptr || !u_ptr || world < 1 || !cuts || rank < 0 ||
        rank >= world || n < 1 || !near_ptr || !near_col || !n_shared || !let_roff || !let_soff || !halo_roff ||
        !halo_soff) {
        set_error("xrl_plan_exchange: bad argument");
        return XRL_EINVAL;
    }
    try {
        std::vector<int32_t> cut(cuts, cuts + world + 1);
        PlanCore P = plan_core(nbox, pb, pe, child, v_ptr, v_src, x_ptr, x_src, w_ptr, w_src, u_ptr, u_src, cut);
        std::vector<int64_t> lro, lso, hro, hso;
        std::vector<int32_t> lri, lsi, hri, hsi;
        split_lists(P.let_need, rank, [&](int32_t s) { return pb[s]; }, cut, lro, lri, lso, lsi);
        // halo: near columns of each rank's rows outside its range + the panels of its remote leaves
        std::vector<std::vector<int32_t>> need(world);
        std::vector<uint8_t> mark(n);
        for (int r = 0; r < world; ++r) {
            std::fill(mark.begin(), mark.end(), 0);
            for (int64_t k = cut[r]; k < cut[r + 1]; ++k)
                for (int64_t j = near_ptr[k]; j < near_ptr[k + 1]; ++j)
                    if (near_col[j] < cut[r] || near_col[j] >= cut[r + 1]) mark[near_col[j]] = 1;
            for (int32_t L : P.halo_leaves[r])
                for (int32_t p = pb[L]; p < pe[L]; ++p) mark[p] = 1;
            for (int64_t p = 0; p < n; ++p)
                if (mark[p]) need[r].push_back((int32_t)p);
        }
        split_lists(need, rank, [](int32_t p) { return p; }, cut, hro, hri, hso, hsi);
        *n_shared = (int64_t)P.shared.size();
        if (shared) std::copy(P.shared.begin(), P.shared.end(), shared);
        std::copy(lro.begin(), lro.end(), let_roff);
        std::copy(lso.begin(), lso.end(), let_soff);
        std::copy(hro.begin(), hro.end(), halo_roff);
        std::copy(hso.begin(), hso.end(), halo_soff);
        if (let_ridx) std::copy(lri.begin(), lri.end(), let_ridx);
        if (let_sidx) std::copy(lsi.begin(), lsi.end(), let_sidx);
        if (halo_ridx) std::copy(hri.begin(), hri.end(), halo_ridx);
        if (halo_sidx) std::copy(hsi.begin(), hsi.end(), halo_sidx);
        return XRL_OK;
    } catch (const std::bad_alloc&) {
        set_error("host out of memory");
        return XRL_ENOMEM;
    }
}
