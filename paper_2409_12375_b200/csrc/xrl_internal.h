// Internal structures of the XRL B200 library (not part of the ABI).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/xrl.h"
#include "harmonics.h"
#include "operators.h"

namespace xrl {

void set_error(const char* fmt, ...);

struct CudaError {
    xrl_status code;
};

#define XRL_CUDA(expr)                                                                       \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess) {                                                             \
            ::xrl::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e), __FILE__,   \
                             __LINE__, cudaGetErrorString(_e));                              \
            throw ::xrl::CudaError{_e == cudaErrorMemoryAllocation ? XRL_ENOMEM : XRL_ECUDA}; \
        }                                                                                    \
    } while (0)

bool sync_check_enabled();  // XRL_SYNC_CHECK=1: synchronize after every launch (debugging)
#define XRL_LAUNCH_CHECK()                                                                   \
    do {                                                                                     \
        XRL_CUDA(cudaGetLastError());                                                        \
        if (::xrl::sync_check_enabled()) XRL_CUDA(cudaDeviceSynchronize());                  \
    } while (0)

// Simple owning device buffer.
template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) { free(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DBuf() { free(); }
    void alloc(size_t count) {
        free();
        n = count;
        if (count) XRL_CUDA(cudaMalloc(&p, count * sizeof(T)));
    }
    void free() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
};

enum Phase { PH_PACK = 0, PH_P2M, PH_M2M, PH_M2L, PH_P2L, PH_L2L, PH_L2P, PH_P2P, PH_NEAR, PH_COUNT };

struct DeviceOperators {
    DBuf<float> m2l_tc;  // [332: M2L 316, M2M 8, L2L 8][2 (hi, lo)][128 x 128 tf32, tcgen05 canonical K-major]
    DBuf<uint16_t> m2l_h16;  // [316 M2L][2 (hi, lo)][128 x 128 f16, canonical K-major], scaled by 2^m2l_hexp
    int m2l_hexp = 0;
    int m2l_index[343];
};

constexpr int kMuStride = 768;       // floats per box multipole mu[r][k] (r-major, k padded to 128)
constexpr int kOpM2M = 316, kOpL2L = 324, kNOpImg = 332;  // tensor-core operator images: M2L 0..315, M2M, L2L
constexpr int kEllStride = 768;      // floats per box local expansion ell[r][k] (r-major, k padded to 128)
#ifndef XRL_NEAR_SEGLEN
#define XRL_NEAR_SEGLEN 96
#endif
constexpr int kNearSegLen = XRL_NEAR_SEGLEN;  // near SpMV: max union columns per segment (8 lanes each)
constexpr int kNearG = 4;            // near SpMV: rows per row group

}  // namespace xrl

namespace xrl {
// One launch of the translation kernel over several dependent levels (all M2M levels, or all L2L levels):
// blocks [first, first + nblocks) of tr_blocks, level v owning block rows [rows[v], rows[v+1]) of the grid.
struct TransPass {
    int first = 0, nblocks = 0, grid = 1, nlev = 0;
    std::vector<int32_t> rows_h;
    DBuf<int32_t> rows;  // [nlev+1] cumulative block rows per level
    DBuf<int> done;      // [nlev] CTAs done with each level (zeroed per launch)
};
}  // namespace xrl

struct xrl_ctx_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t work = nullptr;      // library-owned high-priority stream (FMM chain of xrl_mvm)
    cudaStream_t side = nullptr;      // library-owned low-priority side stream (near SpMV, P2P)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_work = nullptr, ev_m2l = nullptr, ev_p2p = nullptr;
    cudaEvent_t ev_near = nullptr;    // near-first side stream: the near SpMV is done (the fused P2P adds after it)
    cudaStream_t comm = nullptr;      // library-owned stream of a multi-rank context's NCCL exchanges
    cudaEvent_t ev_halo = nullptr, ev_comm = nullptr, ev_p2l = nullptr;
    bool fuse_p2p = true;             // P2P warps inside the M2L kernel (XRL_FUSE=0: off)
    bool m2l_h16 = true;              // M2L in 3xFP16 (XRL_M2L_TF32=1: 3xTF32, the round-2 kernel)
    bool own_stream = false;
    int rank = 0, world = 1;
    void* nccl_comm = nullptr;        // ncclComm_t when world > 1
    xrl::DeviceOperators ops;
    // timing
    bool timing = false;
    int sched = XRL_SCHED_FORK;       // xrl_ctx_set_sched
    int num_sms = 148;
    int64_t launches = 0;
    int refs = 0;         // live trees
    bool dead = false;    // destroy requested
    double phase_ms[xrl::PH_COUNT] = {};
    int64_t phase_launches[xrl::PH_COUNT] = {};
    cudaEvent_t ev[2 * xrl::PH_COUNT] = {};
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    std::vector<cudaEvent_t> event_pool;
};

struct xrl_tree_s {
    xrl_ctx ctx = nullptr;
    int refs = 0;         // live near handles
    bool dead = false;
    int64_t n = 0;
    int32_t leaf_max = 64, max_depth = 21;
    double lo[3] = {0, 0, 0};   // root cube corner
    double W = 1;               // root cube width
    // per panel, library order
    xrl::DBuf<int32_t> perm;    // library -> original
    xrl::DBuf<int32_t> iperm;   // original -> library
    xrl::DBuf<double> cent;     // [n][3] FP64 centroids
    xrl::DBuf<double> area;     // [n]
    xrl::DBuf<double> dmax;     // [n]
    xrl::DBuf<double> tverts;   // [n][12] panel vertices (library order; 4th = NaN for triangles)
    xrl::DBuf<int4> pvid;       // [n] panel vertex ids (w = -1 for triangles), library order
    xrl::DBuf<float4> loc;      // [n] local coords (W units) relative to leaf centre; w = unused
    xrl::DBuf<int32_t> panel_leaf;  // [n] leaf box of each panel
    // boxes (level order)
    int32_t nbox = 0, nleaf = 0, nlevel = 0;
    std::vector<int32_t> lvl_start;          // host [nlevel+1]
    xrl::DBuf<int32_t> blevel, bix, biy, biz, bparent, bchild, bnchild, bpb, bpe;
    xrl::DBuf<int32_t> leaves;               // [nleaf] leaf box ids
    xrl::DBuf<double> bdmax;                 // [nbox] max D in subtree
    // lists, CSR by target box id
    xrl::DBuf<int64_t> u_ptr, v_ptr, x_ptr, w_ptr;
    xrl::DBuf<int32_t> u_src, v_src, x_src, w_src;
    int64_t nu = 0, nv = 0, nx = 0, nw = 0, np2p = 0;
    // M2L pairs sorted by (offset, target) and their tiles
    xrl::DBuf<int32_t> m2l_tgt, m2l_srcb;    // [nv]
    xrl::DBuf<int4> m2l_tiles;               // (offset, pair begin, pair count <= 21, chunk)
    int32_t n_m2l_tiles = 0;
    xrl::DBuf<int4> m2l_blocks;              // (first tile, #tiles, offset, chunk): runs of one operator
    int32_t n_m2l_blocks = 0;                // (padded: balance_blocks in tree.cu)
    int32_t m2l_grid = 0;                    // persistent grid the block order is balanced for
    // M2M / L2L translation tiles for the tensor-core kernel (all levels concatenated)
    xrl::DBuf<int4> tr_tiles, tr_blocks;
    xrl::DBuf<int32_t> tr_tgt, tr_src;
    std::vector<std::pair<int, int>> m2m_lvl, l2l_lvl;  // per level: (first block, #blocks) before packing
    xrl::TransPass m2m_pass, l2l_pass;                 // the packed multi-level launches
    int64_t n_m2l_subtiles = 0;
    // boxes with non-empty X list, leaves with non-empty W list
    xrl::DBuf<int32_t> x_targets;
    int32_t n_x_targets = 0;
    xrl::DBuf<int2> w_targets;               // (owned leaf, W-list box) pairs (M2P, one CTA each)
    int32_t n_w_targets = 0;
    // parents per level for M2M/L2L: boxes with children, grouped by level
    std::vector<int32_t> par_start;          // host [nlevel+1] offsets into parents
    xrl::DBuf<int32_t> parents;
    // partition: this rank owns panels [p0, p1)
    int32_t part_rank = 0, part_world = 1;
    int32_t p0 = 0, p1 = 0;
    std::vector<int32_t> part_cuts;          // panel offsets of all ranks [world+1]
    std::vector<uint8_t> rel;                // box relevant to this rank
    xrl::DBuf<int32_t> mu_zero, ell_zero;    // boxes whose mu / ell records are zeroed per MVM
    int32_t n_mu_zero = 0, n_ell_zero = 0;
    xrl::DBuf<int32_t> own_leaves;           // owned leaves (Morton order)
    xrl::DBuf<int> p2p_counter;              // P2P leaf-task counter (reset per MVM)
    xrl::DBuf<int4> p2p_tasks;               // P2P tasks (leaf, first target panel, #targets <= 256, 0), longest first
    int32_t n_p2p_tasks = 0;
    int32_t n_own_leaves = 0;
    std::vector<int32_t> l2l_start;          // per-level offsets into l2l_boxes
    xrl::DBuf<int32_t> l2l_boxes;
    // multi-rank exchange plan (exchange.cu; part_world > 1)
    std::vector<int32_t> shared_boxes;       // boxes straddling a cut (partial multipoles, all-reduced)
    xrl::DBuf<int32_t> sh_idx;
    xrl::DBuf<float> sh_buf;                 // [n_shared][kMuStride]
    std::vector<int64_t> let_soff, let_roff; // [world+1] box offsets per peer in the send / receive lists
    xrl::DBuf<int32_t> let_sidx, let_ridx;   // own boxes peers need / peers' boxes this rank needs
    xrl::DBuf<float> let_sbuf, let_rbuf;     // [n][kMuStride]
    std::vector<std::vector<int32_t>> halo_leaves;  // [rank] remote leaves its P2P / P2L read (all ranks)
    // host copies of the mesh (original order) for the topology build
    std::vector<double> h_vert;              // [nv][3]
    std::vector<int32_t> h_tri;              // [n][stride] panel vertex ids (mesh order; -1: no 4th vertex)
    int32_t stride = 3;                      // 3: triangles; 4: hybrid panels pv[n][4] (-1: triangle)
    // MVM scratch
    xrl::DBuf<float> mu;                     // [nbox][kMuStride]  mu[r][k]
    xrl::DBuf<unsigned> mu_max;              // largest |mu| of the MVM (float bits) for the 3xFP16 M2L scale
    xrl::DBuf<float> ell;                    // [nbox][kEllStride] ell[r][k]
    xrl::DBuf<float> xq;                     // [n][8] packed charges
    xrl::DBuf<float> xq2;                    // [n][8] the second triple's charges (xrl_mvm pairs, lazily)
    xrl::DBuf<float2> xtmp, ytmp, xlib, ylib; // host-API staging
    xrl::DBuf<float2> xbuf[2], ybuf[2];       // xrl_mvm_host_batch double buffers
};

struct xrl_near_s {
    xrl_tree tree = nullptr;
    int refs = 0;                                // live operators
    bool dead = false;                           // destroy requested (deferred while refs > 0)
    double eta = 1.5;
    int64_t nnz = 0;
    xrl::DBuf<int64_t> row_ptr;
    xrl::DBuf<int32_t> col;
    xrl::DBuf<float> val;       // N_kl (FP32)
    xrl::DBuf<double> val64;    // P_kl (FP64, before subtraction)
    // row-group format of the owned rows for the SpMV (near.cu build_near_groups): n_entries slots, one per
    // union column of a group of kNearG rows
    int64_t n_segs = 0, n_entries = 0;
    xrl::DBuf<int32_t> seg_grp;   // [n_segs] local row group ((row - p0) / kNearG)
    xrl::DBuf<int32_t> seg_base;  // [n_segs] column base (upper 16 bits)
    xrl::DBuf<int64_t> seg_off;   // [n_segs+1] padded slot offsets (multiples of 4)
    xrl::DBuf<float4> gval;       // [n_entries] the group's kNearG rows' N values (FP32), 0 where absent
    xrl::DBuf<uint16_t> eoff;     // [n_entries] column - base, lane-interleaved per 32 slots
    // halo of x (exchange.cu; part_world > 1): panels peers read from this rank / this rank reads
    std::vector<int64_t> halo_soff, halo_roff;  // [world+1] panel offsets per peer
    xrl::DBuf<int32_t> halo_sidx, halo_ridx;
    xrl::DBuf<float> halo_sbuf, halo_rbuf;      // [n][8] packed charge records
};

struct xrl_topo_s {
    xrl_tree tree = nullptr;
    int refs = 0;                                // live operators
    bool dead = false;                           // destroy requested (deferred while refs > 0)
    int64_t n_edges = 0, n_branches = 0, n_loops = 0, nnz_c = 0;
    int32_t n_ports = 0, n_components = 0;
    int64_t n_vertex_loops = 0, n_fund_loops = 0, n_terminal_loops = 0;
    std::vector<int32_t> perm;                   // library -> mesh order
    std::vector<int32_t> edge_i, edge_j;         // library panel indices, i < j
    std::vector<double> edge_mid;                // [n_edges][3]
    std::vector<int32_t> br_a, br_b;             // branch endpoints (panel or n + super node)
    std::vector<int8_t> br_kind;                 // 0 edge, 1 terminal, 2 port
    std::vector<int64_t> m_ptr;                  // M CSR over loops
    std::vector<int32_t> m_idx;
    std::vector<int8_t> m_val;
    std::vector<int32_t> port_loop;
    std::vector<int8_t> loop_kind;
    std::vector<int64_t> c_ptr_h;                // C = M A_t (host copy, FP64)
    std::vector<int32_t> c_col_h;
    std::vector<double> c_val_h;
    xrl::DBuf<int64_t> cl_ptr, cp_ptr;           // C by loop rows / by panel rows
    xrl::DBuf<int32_t> cl_col, cp_col;
    xrl::DBuf<float> cl_val, cp_val;             // 3 floats per nonzero
    xrl::DBuf<double> cl_val64;                  // FP64 copy for the preconditioner assembly
    xrl::DBuf<double> cp_val64;                  // the same by panel rows (c_l(k) read directly, no row search)
    xrl::DBuf<int32_t> long_rows;                // loops with > 64 panel entries (CTA per row)
    int32_t n_long = 0;
};

namespace xrl {
// Loop-space sharding of a partitioned operator (solver.cu build_loop_partition; SURVEY §8(e) "GMRES
// extras"): this rank owns the contiguous loops [L0, L1) (cuts balanced by the owner of each loop's first
// panel) and the tree's panels [p0, p1); an apply exchanges the loop values its owned panels read (loop
// halo) and the panel values its owned loops read (panel halo).
struct LoopPart {
    int64_t L0 = 0, L1 = 0, nlo = 0, nlh = 0, npl = 0, nph = 0;  // owned / halo loops, owned / halo panels
    std::vector<int64_t> lcut;                     // [world+1] loop cuts
    std::vector<int64_t> lh_soff, lh_roff, ph_soff, ph_roff;  // [world+1] per-peer offsets
    DBuf<int32_t> lh_sidx, ph_sidx;                // owned loops (- L0) / owned panels (- p0) peers read
    DBuf<int64_t> pl_ptr, lp_ptr;                  // owned panel -> loop slots, owned loop -> panel slots
    DBuf<int32_t> pl_col, lp_col, lp_long;
    DBuf<float> pl_val, lp_val;                    // C_t values, 3 per entry
    int32_t n_long = 0;
    DBuf<float2> vext, yext, u, pu, sbuf, rbuf;    // scratch
    int cap = 0;
};
}  // namespace xrl

struct xrl_op_s {
    int refs = 0;                                // live preconditioners
    bool dead = false;                           // destroy requested (deferred while refs > 0)
    xrl_tree tree = nullptr;
    xrl_near near = nullptr;
    xrl_topo topo = nullptr;
    double freq = 0, omega = 0;
    double alpha_im = 0;                         // alpha = j * alpha_im = j omega mu0 / 4 pi
    std::vector<double> zsa_h;                   // Z_s/A per panel (library order), [n][2]
    xrl::DBuf<float2> zsa;                       // device copy
    xrl::DBuf<float2> u, pu;                     // scratch [3*nrhs][n]
    int32_t cap_rhs = 0;
    std::unique_ptr<xrl::LoopPart> part;         // partitioned tree: the loop-space shard (else null)
};

struct xrl_precond_s {
    xrl_op op = nullptr;
    int32_t kind = 0;                            // 0 block-Jacobi (k_block_*), 1 whole Q (precond_exact.cu)
    int32_t ilu = 0;                             // kind 1: 0 exact sparse LU (host), 1 ILU(0) on the GPU
    int32_t qkind = 0;                           // Q: 0 diagonal-of-P (Eq. 10), 1 diagonal-of-L
    void* exact = nullptr;                       // kind 1: factorisation state
    int32_t bs = 64, nblocks = 0;
    std::vector<int32_t> bptr_h;
    xrl::DBuf<int32_t> bptr;                     // block starts (global loop ids, assembly)
    xrl::DBuf<int32_t> bptr_loc;                 // the same relative to the rank's first loop (apply)
    int64_t nl_loc = 0;                          // loops of the vectors the apply sees
    xrl::DBuf<float2> inv;                       // [nblocks][bs][bs]
};

namespace xrl {
// diagonal-of-P preconditioner: d_k = Z_s,k/A_k + j alpha P_kk per panel (library order, FP64)
void precond_diag(xrl_op op, std::vector<double2>& d);
// diag-of-L: L_ee = (sum_t A_t P A_t^T)_ee per edge (host vector, FP64)
void precond_ldiag(xrl_op op, std::vector<double>& lee);
// sparse Q of kind qkind (0 diag-of-P Eq. 10, 1 diag-of-L) on the host: rows rc[a] (ascending), values rv[a]
void assemble_q(xrl_op op, int qkind, std::vector<std::vector<int32_t>>& rc,
                std::vector<std::vector<std::complex<double>>>& rv);
// exact Q^-1 (NEXT f2): build the factorisation into pc->exact, apply it, release it
xrl_status exact_build(xrl_precond pc);
void exact_apply(xrl_precond pc, const float2* v, float2* z, int nrhs);
void exact_free(xrl_precond pc);
// phase timing helpers (no-ops unless enabled)
void phase_begin(xrl_ctx ctx, int ph, cudaEvent_t* evb, cudaStream_t st);
void phase_end(xrl_ctx ctx, int ph, cudaEvent_t evb, cudaStream_t st);
void upload_constants(xrl_ctx ctx);
void ctx_release(xrl_ctx ctx);     // delete if dead and unreferenced
xrl_status comm_init(xrl_ctx ctx, const void* unique_id);
void comm_destroy(xrl_ctx ctx);
// multi-rank exchanges (exchange.cu plans and pack kernels, comm.cu NCCL transport)
void build_let_plan(xrl_tree T, const std::vector<int32_t>& hpb, const std::vector<int32_t>& hpe,
                    const std::vector<int32_t>& hchild, cudaStream_t st);
void build_halo_plan(xrl_tree t, xrl_near N, cudaStream_t st);
void gather_records(int64_t cnt, int w, const int32_t* idx, const float* src, float* dst, cudaStream_t st);
void scatter_records(int64_t cnt, int w, const int32_t* idx, const float* src, float* dst, cudaStream_t st);
void add_into(int64_t cnt, const float* a, float* acc, cudaStream_t st);
xrl_status nccl_exchange(xrl_ctx ctx, const float* sbuf, const std::vector<int64_t>& soff, float* rbuf,
                         const std::vector<int64_t>& roff, int rec_floats, cudaStream_t st);
xrl_status nccl_allreduce_sum(xrl_ctx ctx, float* buf, size_t count, cudaStream_t st);
xrl_status nccl_allreduce_sum_f64(xrl_ctx ctx, double* buf, size_t count, cudaStream_t st);
void tree_release(xrl_tree t);
void topo_release(xrl_topo T);     // delete if dead and unreferenced (then release its tree)
void near_release(xrl_near nr);    // likewise for near fields
std::vector<int64_t> near_row_counts(xrl_tree t, double eta, cudaStream_t st);  // near.cu
void op_release(xrl_op op);        // likewise for operators (then release topology and tree)
}  // namespace xrl
