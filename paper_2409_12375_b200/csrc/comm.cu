// Multi-GPU plumbing: NCCL communicator of a multi-rank context
// and the per-MVM gather of the rank-owned slices of x.
//
// Each rank owns a contiguous Morton range of leaves (panels [p0, p1),
// tree.cu).  An MVM needs the charges of every panel (P2M of all leaves, P2P
// and near-field sources outside the range), so the owned slices of the three
// complex components are gathered into the full vectors with one NCCL group of
// per-rank broadcasts (slices have different lengths, so ncclAllGather's equal
// counts do not fit).  The rest of the MVM is rank-local: the upward pass is
// computed redundantly, M2L/P2L/L2L only for boxes meeting the owned range,
// P2P/L2P/near only for owned targets.
#include <nccl.h>

#include "xrl_internal.h"

using namespace xrl;

#define XRL_NCCL(expr)                                                                               \
    do {                                                                                             \
        ncclResult_t _r = (expr);                                                                    \
        if (_r != ncclSuccess) {                                                                     \
            ::xrl::set_error("NCCL error %s at %s:%d", ncclGetErrorString(_r), __FILE__, __LINE__);   \
            return XRL_ENCCL;                                                                        \
        }                                                                                            \
    } while (0)

namespace xrl {

xrl_status comm_init(xrl_ctx ctx, const void* unique_id)
{
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    ncclComm_t comm;
    XRL_NCCL(ncclCommInitRank(&comm, ctx->world, id, ctx->rank));
    ctx->nccl_comm = comm;
    return XRL_OK;
}

void comm_destroy(xrl_ctx ctx)
{
    if (ctx->nccl_comm) ncclCommDestroy((ncclComm_t)ctx->nccl_comm);
    ctx->nccl_comm = nullptr;
}

xrl_status gather_slices(xrl_tree t, const float2* x_local, float2* x_full)
{
    xrl_ctx ctx = t->ctx;
    if (!ctx->nccl_comm) { set_error("gather_slices: context has no communicator"); return XRL_ENCCL; }
    const int64_t n = t->n, nl = t->p1 - t->p0;
    XRL_NCCL(ncclGroupStart());
    for (int v = 0; v < 3; ++v)
        for (int r = 0; r < t->part_world; ++r) {
            const int64_t c0 = t->part_cuts[r], c1 = t->part_cuts[r + 1];
            if (c1 <= c0) continue;
            float2* recv = x_full + (size_t)v * n + c0;
            // sendbuff is read on the root only; the other ranks pass their receive buffer (never NULL)
            const void* send = (r == ctx->rank) ? (const void*)(x_local + (size_t)v * nl) : (const void*)recv;
            const ncclResult_t e = ncclBroadcast(send, recv, (size_t)(c1 - c0) * 2, ncclFloat, r,
                                                 (ncclComm_t)ctx->nccl_comm, ctx->stream);
            if (e != ncclSuccess) {
                ncclGroupEnd();  // close the group before reporting, so later NCCL calls are not captured by it
                set_error("NCCL error %s in ncclBroadcast (gather_slices)", ncclGetErrorString(e));
                return XRL_ENCCL;
            }
        }
    XRL_NCCL(ncclGroupEnd());
    return XRL_OK;
}

}  // namespace xrl

extern "C" xrl_status xrl_nccl_unique_id(void* out)
{
    if (!out) { set_error("xrl_nccl_unique_id: null argument"); return XRL_EINVAL; }
    ncclUniqueId id;
    XRL_NCCL(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
    return XRL_OK;
}
