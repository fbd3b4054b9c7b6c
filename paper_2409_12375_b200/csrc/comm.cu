// Multi-GPU plumbing: NCCL communicator of a multi-rank context and the transport of
// the sharded MVM's exchanges (plans in exchange.cu): the halo of x and the local-essential-tree
// multipoles as grouped ncclSend/ncclRecv, the multipoles of the boxes that straddle a cut as one
// ncclAllReduce.  NVLink/NVSwitch carries them; the volumes are small.
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

// Grouped point-to-point exchange of packed records: to each peer q the records
// sbuf[soff[q] .. soff[q+1]) and from each peer q into rbuf[roff[q] .. roff[q+1]) (rec_floats floats per
// record); the plans are symmetric by construction (exchange.cu), so every send has its matching receive.
xrl_status nccl_exchange(xrl_ctx ctx, const float* sbuf, const std::vector<int64_t>& soff, float* rbuf,
                         const std::vector<int64_t>& roff, int rec_floats, cudaStream_t st)
{
    if (!ctx->nccl_comm) { set_error("nccl_exchange: context has no communicator"); return XRL_ENCCL; }
    ncclComm_t comm = (ncclComm_t)ctx->nccl_comm;
    XRL_NCCL(ncclGroupStart());
    for (int q = 0; q < ctx->world; ++q) {
        if (q == ctx->rank) continue;
        ncclResult_t e = ncclSuccess;
        const int64_t ns = soff[q + 1] - soff[q], nr = roff[q + 1] - roff[q];
        if (ns > 0) e = ncclSend(sbuf + soff[q] * rec_floats, (size_t)ns * rec_floats, ncclFloat, q, comm, st);
        if (e == ncclSuccess && nr > 0)
            e = ncclRecv(rbuf + roff[q] * rec_floats, (size_t)nr * rec_floats, ncclFloat, q, comm, st);
        if (e != ncclSuccess) {
            ncclGroupEnd();  // close the group before reporting, so later NCCL calls are not captured by it
            set_error("NCCL error %s in the MVM exchange", ncclGetErrorString(e));
            return XRL_ENCCL;
        }
    }
    XRL_NCCL(ncclGroupEnd());
    return XRL_OK;
}

xrl_status nccl_allreduce_sum(xrl_ctx ctx, float* buf, size_t count, cudaStream_t st)
{
    if (!ctx->nccl_comm) { set_error("nccl_allreduce_sum: context has no communicator"); return XRL_ENCCL; }
    if (count == 0) return XRL_OK;
    XRL_NCCL(ncclAllReduce(buf, buf, count, ncclFloat, ncclSum, (ncclComm_t)ctx->nccl_comm, st));
    return XRL_OK;
}

xrl_status nccl_allreduce_sum_f64(xrl_ctx ctx, double* buf, size_t count, cudaStream_t st)
{
    if (!ctx->nccl_comm) { set_error("nccl_allreduce_sum_f64: context has no communicator"); return XRL_ENCCL; }
    if (count == 0) return XRL_OK;
    XRL_NCCL(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, (ncclComm_t)ctx->nccl_comm, st));
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
