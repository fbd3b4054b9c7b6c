// C-ABI plumbing: errors, context, timing (include/xrl.h).
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "xrl_internal.h"

namespace xrl {

static thread_local char g_err[1024] = "";

bool sync_check_enabled()
{
    static const bool on = [] { const char* e = getenv("XRL_SYNC_CHECK"); return e && e[0] == '1'; }();
    return on;
}

void set_error(const char* fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

static const char* kPhaseNames[PH_COUNT] = {"pack", "p2m", "m2m", "m2l", "p2l", "l2l", "l2p_m2p", "p2p", "near"};

static cudaEvent_t get_event(xrl_ctx ctx)
{
    if (!ctx->event_pool.empty()) {
        cudaEvent_t e = ctx->event_pool.back();
        ctx->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    XRL_CUDA(cudaEventCreate(&e));
    return e;
}

void phase_begin(xrl_ctx ctx, int ph, cudaEvent_t* evb, cudaStream_t st)
{
    (void)ph;
    *evb = nullptr;
    if (!ctx->timing) return;
    *evb = get_event(ctx);
    XRL_CUDA(cudaEventRecord(*evb, st));
}

void phase_end(xrl_ctx ctx, int ph, cudaEvent_t evb, cudaStream_t st)
{
    if (!ctx->timing || !evb) return;
    cudaEvent_t e = get_event(ctx);
    XRL_CUDA(cudaEventRecord(e, st));
    ctx->pending.push_back({ph, {evb, e}});
}

static void drain(xrl_ctx ctx)
{
    for (auto& p : ctx->pending) {
        XRL_CUDA(cudaEventSynchronize(p.second.second));
        float ms = 0;
        XRL_CUDA(cudaEventElapsedTime(&ms, p.second.first, p.second.second));
        ctx->phase_ms[p.first] += ms;
        ctx->phase_launches[p.first] += 1;
        ctx->event_pool.push_back(p.second.first);
        ctx->event_pool.push_back(p.second.second);
    }
    ctx->pending.clear();
}

}  // namespace xrl

using namespace xrl;

#define XRL_TRY try {
#define XRL_CATCH                                   \
    }                                               \
    catch (const CudaError& e) { return e.code; }   \
    catch (const std::bad_alloc&) {                 \
        set_error("host out of memory");            \
        return XRL_ENOMEM;                          \
    }

extern "C" {

const char* xrl_last_error(void) { return g_err; }
const char* xrl_version(void) { return "xrl-b200 0.1 (sm_100a, p=10)"; }

xrl_status xrl_ctx_create(int device, void* cuda_stream, int rank, int world, const void* nccl_unique_id,
                          xrl_ctx* out)
{
    if (!out) { set_error("xrl_ctx_create: out is NULL"); return XRL_EINVAL; }
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) { set_error("bad rank/world %d/%d", rank, world); return XRL_EINVAL; }
    if (world > 1 && !nccl_unique_id) { set_error("world > 1 needs an ncclUniqueId"); return XRL_EINVAL; }
    XRL_TRY
        int ndev = 0;
        cudaError_t e = cudaGetDeviceCount(&ndev);
        if (e != cudaSuccess || ndev == 0) {
            set_error("no CUDA device available (%s); this library has no CPU path", cudaGetErrorString(e));
            return XRL_ECUDA;
        }
        XRL_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop;
        XRL_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10) {
            set_error("device %d is sm_%d%d; this library is built for sm_100a only", device, prop.major, prop.minor);
            return XRL_ECUDA;
        }
        // owned by a guard until fully initialised: any failure below (a throwing XRL_CUDA, a failed
        // communicator) releases the streams and events created so far through ctx_release
        struct Guard {
            xrl_ctx c;
            ~Guard() { if (c) { c->dead = true; ctx_release(c); } }
        } guard{new xrl_ctx_s()};
        xrl_ctx c = guard.c;
        c->device = device;
        c->rank = rank;
        c->world = world;
        c->stream = (cudaStream_t)cuda_stream;  // NULL = legacy default stream
        // library-owned streams: `work` (highest priority) runs the FMM chain, `side` (lowest
        // priority) the P2P / near SpMV, so their CTAs fill SMs the chain leaves free
        int prio_lo = 0, prio_hi = 0;
        XRL_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        XRL_CUDA(cudaStreamCreateWithPriority(&c->work, cudaStreamNonBlocking, prio_hi));
        XRL_CUDA(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, prio_lo));
        XRL_CUDA(cudaEventCreateWithFlags(&c->ev_work, cudaEventDisableTiming));
        XRL_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
        XRL_CUDA(cudaEventCreateWithFlags(&c->ev_m2l, cudaEventDisableTiming));
        XRL_CUDA(cudaEventCreateWithFlags(&c->ev_p2p, cudaEventDisableTiming));
        XRL_CUDA(cudaEventCreateWithFlags(&c->ev_near, cudaEventDisableTiming));
        if (const char* e = getenv("XRL_FUSE"); e && e[0] == '0') c->fuse_p2p = false;
        if (const char* e = getenv("XRL_M2L_TF32"); e && e[0] == '1') c->m2l_h16 = false;
        XRL_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
        if (const char* e = getenv("XRL_SCHED")) c->sched = atoi(e);
        if (const char* e = getenv("XRL_SERIAL"); e && e[0] == '1') c->sched = XRL_SCHED_SERIAL;
        if (c->sched < XRL_SCHED_SERIAL || c->sched > XRL_SCHED_LATE) c->sched = XRL_SCHED_FORK;
        upload_constants(c);
        // the exchanges' stream (NCCL on a multi-rank context; the virtual-rank timing pass uses it for the same
        // overlap on a single-rank one)
        XRL_CUDA(cudaStreamCreateWithPriority(&c->comm, cudaStreamNonBlocking, prio_hi));
        XRL_CUDA(cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming));
        XRL_CUDA(cudaEventCreateWithFlags(&c->ev_comm, cudaEventDisableTiming));
        XRL_CUDA(cudaEventCreateWithFlags(&c->ev_p2l, cudaEventDisableTiming));
        if (world > 1) {
            xrl_status st = comm_init(c, nccl_unique_id);
            if (st) return st;
        }
        guard.c = nullptr;
        *out = c;
        return XRL_OK;
    XRL_CATCH
}

xrl_status xrl_ctx_sync(xrl_ctx ctx)
{
    if (!ctx) { set_error("null ctx"); return XRL_EINVAL; }
    XRL_TRY
        XRL_CUDA(cudaSetDevice(ctx->device));
        XRL_CUDA(cudaStreamSynchronize(ctx->stream));
        return XRL_OK;
    XRL_CATCH
}

void xrl_ctx_destroy(xrl_ctx ctx)
{
    if (!ctx) return;
    ctx->dead = true;
    ctx_release(ctx);
}

}  // extern "C"

void xrl::ctx_release(xrl_ctx ctx)
{
    if (!ctx->dead || ctx->refs > 0) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto& p : ctx->pending) { cudaEventDestroy(p.second.first); cudaEventDestroy(p.second.second); }
    for (auto e : ctx->event_pool) cudaEventDestroy(e);
    comm_destroy(ctx);
    if (ctx->side) { cudaStreamSynchronize(ctx->side); cudaStreamDestroy(ctx->side); }
    if (ctx->work) { cudaStreamSynchronize(ctx->work); cudaStreamDestroy(ctx->work); }
    if (ctx->ev_work) cudaEventDestroy(ctx->ev_work);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_m2l) cudaEventDestroy(ctx->ev_m2l);
    if (ctx->ev_p2p) cudaEventDestroy(ctx->ev_p2p);
    if (ctx->ev_near) cudaEventDestroy(ctx->ev_near);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    if (ctx->comm) { cudaStreamSynchronize(ctx->comm); cudaStreamDestroy(ctx->comm); }
    if (ctx->ev_halo) cudaEventDestroy(ctx->ev_halo);
    if (ctx->ev_comm) cudaEventDestroy(ctx->ev_comm);
    if (ctx->ev_p2l) cudaEventDestroy(ctx->ev_p2l);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

extern "C" {

xrl_status xrl_timing_enable(xrl_ctx ctx, int on)
{
    if (!ctx) { set_error("null ctx"); return XRL_EINVAL; }
    ctx->timing = on != 0;
    return XRL_OK;
}

int32_t xrl_timing_count(void) { return PH_COUNT; }
const char* xrl_timing_name(int32_t i) { return (i >= 0 && i < PH_COUNT) ? kPhaseNames[i] : ""; }

xrl_status xrl_timing_get(xrl_ctx ctx, double* ms, int64_t* launches)
{
    if (!ctx) { set_error("null ctx"); return XRL_EINVAL; }
    XRL_TRY
        drain(ctx);
        for (int i = 0; i < PH_COUNT; ++i) {
            if (ms) ms[i] = ctx->phase_ms[i];
            if (launches) launches[i] = ctx->phase_launches[i];
        }
        return XRL_OK;
    XRL_CATCH
}

int64_t xrl_launch_count(xrl_ctx ctx) { return ctx ? ctx->launches : 0; }

xrl_status xrl_ctx_set_sched(xrl_ctx ctx, int32_t mode)
{
    if (!ctx || mode < XRL_SCHED_SERIAL || mode > XRL_SCHED_LATE) {
        set_error("xrl_ctx_set_sched: null context or bad mode %d", mode);
        return XRL_EINVAL;
    }
    ctx->sched = mode;
    return XRL_OK;
}

xrl_status xrl_ctx_set_fuse(xrl_ctx ctx, int32_t on)
{
    if (!ctx) { set_error("xrl_ctx_set_fuse: null context"); return XRL_EINVAL; }
    ctx->fuse_p2p = on != 0;
    return XRL_OK;
}

xrl_status xrl_timing_reset(xrl_ctx ctx)
{
    if (!ctx) { set_error("null ctx"); return XRL_EINVAL; }
    XRL_TRY
        drain(ctx);
        for (int i = 0; i < PH_COUNT; ++i) { ctx->phase_ms[i] = 0; ctx->phase_launches[i] = 0; }
        return XRL_OK;
    XRL_CATCH
}

}  // extern "C"
