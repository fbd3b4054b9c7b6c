/*
 * xrl.h -- C-ABI of the B200-native hot path of XRL (arXiv 2409.12375):
 * the FMM-accelerated panel MVM inside the preconditioned GMRES.
 *
 * The operator.  XRL discretises the MQS SIE (Eq. 1) with pulse
 * bases on panels after the centroid-midpoint basis transformation
 * (Eq. 4-5, Alg. 1).  The potential part of Eq. 6
 * with j*omega*mu0/(4 pi) pulled out is the real
 * symmetric panel matrix P, applied three times per loop-space MVM, once per
 * Cartesian current component (Eq. 9), by an FMM over the
 * panel centroids "in the format of particle simulation".
 * This library applies
 *     y_t = P x_t,  t = 1..3  (complex x_t; P real -> 6 real right-hand sides)
 *     P_kk = I(c_k;T_k)/A_k
 *     P_kl = 1/2 [I(c_k;T_l)/A_l + I(c_l;T_k)/A_k]   if d_kl^2 < (eta max(D_k,D_l))^2
 *     P_kl = 1/|c_k - c_l|                            otherwise
 * with I(r;T) = int_T dS'/|r - r'| (analytic), c centroids, A areas, D the
 * longest edge (readings R1-R4).
 *
 * Conventions for every entry point:
 *  - Status: 0 = XRL_OK, > 0 warning, < 0 error; xrl_last_error() returns a
 *    thread-local message for the last failing call.
 *  - Handles are opaque, allocated by the library and released by the matching
 *    *_destroy (NULL-safe).  Host input arrays are borrowed for the duration of
 *    the call and copied.  Device vectors belong to the caller: contiguous,
 *    16-byte aligned, resident on the context's device.  The library never
 *    frees caller memory.
 *  - Asynchrony: xrl_mvm / xrl_precond_apply / order conversions enqueue on the
 *    context stream and return; argument errors are reported synchronously,
 *    asynchronous CUDA faults surface on the next call or at xrl_ctx_sync.
 *    Calls with a _host suffix and xrl_gmres block.
 *  - Concurrency: one in-flight MVM per tree handle (it owns the expansion
 *    scratch).  Handles are immutable after build.
 *  - Vectors passed to the MVM are in "library order" (Morton order of the
 *    centroids; xrl_to_library_order / xrl_from_library_order convert).
 *  - Units: SI (metres); P in 1/m.
 *  - There is no CPU fallback: without a usable sm_100 device every entry point
 *    that needs one returns XRL_ECUDA.
 */
#ifndef XRL_H
#define XRL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t xrl_status;
enum {
    XRL_OK = 0,
    XRL_ENOCONV = 1,       /* some GMRES column did not converge (per-column flags in report) */
    XRL_EINVAL = -1,       /* bad option / argument (p != 10, leaf < 1, eta <= 0, null pointer) */
    XRL_EDIM = -2,         /* vector length / nvec mismatch */
    XRL_EPROVENANCE = -3,  /* handle built from a different tree / context */
    XRL_EGEOM = -4,        /* zero-area triangle, vertex index out of range, coincident centroids */
    XRL_ESINGULAR = -5,    /* preconditioner block pivot below threshold */
    XRL_ENOMEM = -6,
    XRL_ECUDA = -7,
    XRL_ENCCL = -8,
    XRL_ENOFREQ = -9,
    XRL_EUNSUPPORTED = -10
};

/* MVM flags (tests and diagnostics). */
enum {
    XRL_MVM_FULL = 0,        /* y = P x */
    XRL_MVM_NEAR_ONLY = 1,   /* y = N x, N = near CSR (P_kk on the diagonal, P_kl - 1/r off it) */
    XRL_MVM_FAR_ONLY = 2     /* y = sum_{l != k} x_l / |c_k - c_l| (FMM + P2P, no correction) */
};

typedef struct xrl_ctx_s* xrl_ctx;
typedef struct xrl_tree_s* xrl_tree;
typedef struct xrl_near_s* xrl_near;

const char* xrl_last_error(void);
const char* xrl_version(void);

/* Context: device ordinal, CUDA stream the library enqueues on (cudaStream_t;
 * NULL = the legacy default stream, as everywhere in CUDA), rank/world for Morton-range sharding (world == 1 for a
 * single GPU; multi-rank contexts need the 128-byte ncclUniqueId broadcast by
 * the caller, else NULL). */
xrl_status xrl_ctx_create(int device, void* cuda_stream, int rank, int world,
                          const void* nccl_unique_id, xrl_ctx* out);
xrl_status xrl_ctx_sync(xrl_ctx ctx);
/* Destroying a context that still has trees defers the release until the
 * last tree built on it is destroyed (likewise a tree with near handles). */
void xrl_ctx_destroy(xrl_ctx ctx);

/* FMM options.  p: expansion order (only 10 is compiled, PAPER.md silent ->
 * north star p = 10); leaf_max: split a box while it holds more panels
 * (default 64); max_depth: <= 21 (63-bit Morton keys).
 * part_rank / part_world: Morton-range partition of the targets (SURVEY
 * §8(e)).  On a multi-rank context they must equal its rank / world (or be
 * 0 / 0).  On a single-rank context part_world > 1 builds rank part_rank's
 * share ("virtual rank": k such trees on one context run the sharded MVM on
 * one GPU through xrl_mvm_vranks).  0 / 0 = no partition. */
typedef struct {
    int32_t p;
    int32_t leaf_max;
    int32_t max_depth;
    int32_t part_rank;
    int32_t part_world;
} xrl_fmm_opts;

/* Balanced contiguous cuts of n weighted items into `world` ranges:
 * cuts[r] .. cuts[r+1] is range r (int64 [world+1]); the partition rule of
 * the sharded MVM (leaf work estimates in Morton order).  Host function. */
xrl_status xrl_partition_cuts(int64_t n, const double* weights, int32_t world, int64_t* cuts);

/* 128-byte ncclUniqueId for xrl_ctx_create (rank 0 generates it, the caller
 * broadcasts it to the other ranks, e.g. through torch.distributed). */
xrl_status xrl_nccl_unique_id(void* out128);

/* Octree build on the GPU (setup, once per mesh).
 * vert: host FP64 [n_vert][3] (m); tri: host int32 [n_tri][3].
 * Computes centroids/areas/longest edges (PAPER.md:56 centroids are the PEEC
 * nodes), 63-bit Morton keys of the centroids, a stable radix sort, the
 * adaptive octree (split while count > leaf_max) and the U/V/W/X interaction
 * lists.  Errors: XRL_EINVAL, XRL_EGEOM (zero area / bad index), XRL_ECUDA. */
xrl_status xrl_tree_build(xrl_ctx ctx, int64_t n_vert, const double* vert, int64_t n_tri,
                          const int32_t* tri, const xrl_fmm_opts* opts, xrl_tree* out);
/* Hybrid triangle/rectangle meshes ("the hybrid of triangles and
 * rectangles"; NEXT f4): pv host int32 [n_panel][4], pv[k][3] = -1 for a
 * triangle, else a rectangle = planar parallelogram (v0 v1 v2 v3 in cyclic
 * order; XRL_EGEOM if v2 - v1 != v3 - v0 beyond 1e-9 of its diameter).  A
 * rectangle's centroid is the intersection of its diagonals, its D the longer
 * diagonal; the near integrals split it on the diagonal v0-v2.  Otherwise as
 * xrl_tree_build (the loop-space topology accepts triangle meshes only). */
xrl_status xrl_tree_build_poly(xrl_ctx ctx, int64_t n_vert, const double* vert, int64_t n_panel,
                               const int32_t* pv, const xrl_fmm_opts* opts, xrl_tree* out);
void xrl_tree_destroy(xrl_tree tree);

typedef struct {
    int64_t n;            /* panels (global) */
    int64_t n_local;      /* panels owned by this rank */
    int64_t offset;       /* first owned panel in library order */
    int32_t n_boxes, n_leaves, n_levels, p;
    int64_t n_v_pairs;    /* M2L translations */
    int64_t n_x_pairs;    /* P2L (box, leaf) pairs */
    int64_t n_w_pairs;    /* M2P (leaf, box) pairs */
    int64_t n_u_pairs;    /* leaf-leaf P2P pairs (incl. self) */
    int64_t n_p2p;        /* ordered panel pairs done by P2P (self excluded) */
    double root_lo[3];    /* root cube corner (m) */
    double root_width;    /* root cube width W (m) */
    int64_t n_m2l_tiles;     /* 16-pair M2L tiles of this rank */
    int64_t n_m2l_subtiles;  /* tcgen05 MMA groups (one per <= 16-pair tile, N = 96) of this rank */
} xrl_tree_info_t;
xrl_status xrl_tree_info(xrl_tree tree, xrl_tree_info_t* info);

/* perm_host[i] = original panel index of library position i (int32 [n]). */
xrl_status xrl_tree_perm(xrl_tree tree, int32_t* perm_host);

/* Reorder device complex64 vectors [nvec][n]: user (mesh) order <-> library order. */
xrl_status xrl_to_library_order(xrl_tree tree, const void* x_user, void* x_lib, int32_t nvec);
xrl_status xrl_from_library_order(xrl_tree tree, const void* x_lib, void* x_user, int32_t nvec);

/* Box/list export for the coverage audit (tests).  Pass NULL for any array
 * to skip it; sizes from xrl_tree_info.  Boxes are in level order.
 * box_level/ix/iy/iz/parent/pb/pe: int32 [n_boxes]; is_leaf: int32 [n_boxes];
 * *_ptr: int64 [n_boxes+1] CSR by target box, *_src: int32 sources.
 * lists: U (leaf <- box, direct P2P: adjacent leaves, plus adaptive X/W
 * pairs between small boxes evaluated directly), V (box <- box, M2L),
 * X (non-leaf box <- leaf, P2L), W (leaf <- box with > 96 panels, M2P).
 * Every ordered panel pair is covered exactly once by U, W, and the V/X
 * lists of the target's leaf and its ancestors. */
xrl_status xrl_tree_export(xrl_tree tree, int32_t* box_level, int32_t* box_ijk /* [n_boxes][3] */,
                           int32_t* box_parent, int32_t* box_pb, int32_t* box_pe, int32_t* is_leaf,
                           int64_t* u_ptr, int32_t* u_src, int64_t* v_ptr, int32_t* v_src,
                           int64_t* x_ptr, int32_t* x_src, int64_t* w_ptr, int32_t* w_src);

/* Near field (setup, once per mesh; frequency independent).
 * eta: near criterion factor (default 1.5).  For every near pair the FP64
 * analytic single-triangle integrals (Eq. 6 on centroids,
 * PAPER.md:114-116) give N_kl = P_kl - 1/|c_k - c_l| (stored FP32) and
 * N_kk = P_kk; CSR in library order, columns ascending. */
typedef struct {
    double eta;
    int32_t galerkin; /* 0: centroid collocation (the default above); 1: the Galerkin near rule of
                         SPEC.md:345 (NEXT f4) -- self and vertex-adjacent pairs take the mean of
                         I(x; S_l)/A_l over the observation panel (Radon 7-point rule on triangles,
                         2 x 2 Gauss on rectangles), symmetrised the same way; other near pairs unchanged */
} xrl_near_opts;
xrl_status xrl_near_assemble(xrl_tree tree, const xrl_near_opts* opts, xrl_near* out);
void xrl_near_destroy(xrl_near near);
/* Copies the CSR to host buffers (any may be NULL).  row_ptr int64 [n+1],
 * col int32 [nnz], val32 float [nnz] (as used), val64 double [nnz] (P_kl and
 * P_kk in FP64, i.e. the near entries before the 1/r subtraction).  *nnz is
 * always written. */
xrl_status xrl_near_export(xrl_near near, int64_t* row_ptr, int32_t* col, float* val32,
                           double* val64, int64_t* nnz);
/* Sizes of the near field (any pointer may be NULL): nnz of the CSR (all rows), and of the
 * row-group format the SpMV streams for this rank's rows: segments (runs of
 * <= 256 union columns of a group of 4 consecutive rows whose columns share their upper 16
 * bits) and padded slots (one per union column: float4 of the 4 rows' FP32 values + u16 lower
 * column bits; 18 B each). */
xrl_status xrl_near_info(xrl_near near, int64_t* nnz, int64_t* n_segments, int64_t* n_entries);
/* Selected rows of the CSR (tests on full-size meshes): rows host int64 [nrows]
 * (library order); cnt host int64 [nrows] receives each row's length; col,
 * val32, val64 (any may be NULL) receive the rows concatenated in the given
 * order (call once with NULL arrays to size them).  XRL_EINVAL for a row out
 * of range. */
xrl_status xrl_near_export_rows(xrl_near near, int64_t nrows, const int64_t* rows, int64_t* cnt, int32_t* col,
                                float* val32, double* val64);

/* The hot path: y = P x (flags select diagnostic parts).
 * x, y: device complex64 [nvec][n_local] in library order (this rank's slice
 * [offset, offset + n_local) on a multi-rank context), must not alias;
 * nvec a multiple of 3 (each triple of complex components = 6 real RHS through
 * one tree traversal; on a single-rank tree consecutive triples
 * run in pairs whose P2P and near SpMV are one pass for 12 RHS, XRL_PAIR=0
 * turns that off).  Enqueued on the context stream.
 * Multi-rank (plans built at setup from the shared tree and near
 * pattern): each rank packs its own charges, receives the halo of
 * remote charges its P2P / P2L / near rows read (grouped ncclSend/ncclRecv),
 * runs P2M on its own leaves and M2M on its subtrees, all-reduces the partial
 * multipoles of the boxes that straddle a cut, receives the local-essential-
 * tree multipoles (grouped send/recv), then computes its slice of y.  All calls
 * are collective over the context's communicator.  XRL_EUNSUPPORTED for a
 * partitioned tree on a single-rank context (use xrl_mvm_vranks). */
xrl_status xrl_mvm(xrl_tree tree, xrl_near near, const void* x, void* y, int32_t nvec, uint32_t flags);

/* Virtual ranks: the sharded MVM of k trees partitioned 0..k-1 of one mesh
 * (xrl_fmm_opts part_rank = r, part_world = k) built on ONE single-rank
 * context, run in one call on one GPU with the same plans and kernels as the
 * multi-rank xrl_mvm; the exchanges are device copies between the trees'
 * buffers instead of NCCL.  x[r], y[r]: device complex64 [nvec][n_local(r)]
 * (rank r's slice in library order).  The ranks' phases are serialised on the
 * context stream.  rank_ms (host double [k], may be NULL) receives each rank's
 * device time: a timing pass before the real one runs each rank's whole MVM
 * alone on the GPU in the multi-rank order (P2P forked early), the three
 * transports left out; exch_ms (may be NULL) receives the device-copy time of
 * the exchanges -- the inputs of the multi-GPU projection.  k = 1 with an unpartitioned tree
 * is the plain MVM.  Errors: XRL_EINVAL (trees not one k-way partition,
 * aliasing), XRL_EPROVENANCE (near/tree or context mismatch), XRL_EDIM. */
xrl_status xrl_mvm_vranks(int32_t k, const xrl_tree* trees, const xrl_near* nears, const void* const* x,
                          void* const* y, int32_t nvec, uint32_t flags, double* rank_ms, double* exch_ms);

/* Host function (no GPU): the exchange plan of rank `rank` of a `world`-way
 * partition, from a tree and near pattern given as plain host arrays -- the
 * code xrl_tree_build / xrl_near_assemble run on a partitioned tree, exported
 * for CPU multi-process tests.  Boxes b < nbox: panel range [pb[b], pe[b]),
 * child[b] < 0 for leaves; CSR lists by target box (int64 ptr [nbox+1], int32
 * sources): V (M2L), X (P2L source leaves), W (M2P), U (P2P source leaves);
 * near pattern near_ptr int64 [n+1] / near_col int32 (library order); cuts
 * int32 [world+1] panel offsets.  Outputs: *n_shared and shared [n_shared]
 * (boxes straddling a cut); let_roff / let_soff int64 [world+1] and
 * let_ridx / let_sidx (boxes received from / sent to each peer, ascending);
 * halo_roff / halo_soff int64 [world+1] and halo_ridx / halo_sidx (panels).
 * Call once with the index arrays NULL to size them. */
xrl_status xrl_plan_exchange(int32_t nbox, const int32_t* pb, const int32_t* pe, const int32_t* child,
                             const int64_t* v_ptr, const int32_t* v_src, const int64_t* x_ptr,
                             const int32_t* x_src, const int64_t* w_ptr, const int32_t* w_src,
                             const int64_t* u_ptr, const int32_t* u_src, int64_t n, const int64_t* near_ptr,
                             const int32_t* near_col, int32_t world, const int32_t* cuts, int32_t rank,
                             int64_t* n_shared, int32_t* shared, int64_t* let_roff, int32_t* let_ridx,
                             int64_t* let_soff, int32_t* let_sidx, int64_t* halo_roff, int32_t* halo_ridx,
                             int64_t* halo_soff, int32_t* halo_sidx);

/* Per-MVM exchange volume of a partitioned tree (records per triple; 0 on a
 * single-rank tree): halo panels sent / received (32 B each: the 6 RHS + pad),
 * LET boxes sent / received (3 KB each: 6 x 128 floats) and shared boxes
 * all-reduced (3 KB each).  Any pointer may be NULL. */
xrl_status xrl_exchange_info(xrl_tree tree, xrl_near near, int64_t* halo_send, int64_t* halo_recv,
                             int64_t* let_send, int64_t* let_recv, int64_t* shared);

/* End-to-end variant with HOST complex64 buffers [nvec][n] in the mesh's
 * original panel order: H2D copy, reorder, MVM, reorder, D2H copy.  Blocking.
 * On a multi-rank context the host buffers are the rank's slice
 * [nvec][n_local] in library order (H2D, MVM with the NCCL gather, D2H). */
xrl_status xrl_mvm_host(xrl_tree tree, xrl_near near, const void* x_host, void* y_host, int32_t nvec,
                        uint32_t flags);
/* Pipelined end-to-end MVMs over a batch of independent inputs (serving use: many
 * right-hand-side triples, frequency points or requests).  For k = 0 .. nbatch-1:
 * y_host[k] = P x_host[k], each a host complex64 [nvec][n] buffer in mesh order
 * (multi-rank: this rank's [nvec][n_local] slice in library order), every step
 * with its own host->device copy and device->host read, as xrl_mvm_host.  The
 * copies run on two library streams double-buffered against the MVMs, so step
 * k+1's input copy and step k-1's output copy overlap step k's MVM (page-locked
 * host buffers are needed for the overlap; pageable ones still give the right
 * result).  Buffers may repeat across k (inputs are only read; outputs are
 * written in step order).  Blocking; returns when every y_host[k] is written. */
xrl_status xrl_mvm_host_batch(xrl_tree tree, xrl_near near, const void* const* x_host, void* const* y_host,
                              int32_t nvec, int32_t nbatch, uint32_t flags);

/* Kernel scheduling of xrl_mvm on this context (no effect on results beyond
 * FP32 summation order of atomics):
 *   XRL_SCHED_SERIAL (0)  every kernel on the context stream, in order (per-phase
 *                         times are then isolated kernel times; profiling);
 *   XRL_SCHED_FORK (1)    default: the FMM chain (P2M..L2L, L2P) on a library-owned
 *                         high-priority stream, P2P then the near SpMV on a
 *                         low-priority side stream forked after the charge pack,
 *                         joined back into the context stream;
 *   XRL_SCHED_LATE (2)    as 1, side stream forked when the M2L is launched.
 * The XRL_SCHED environment variable, if set, overrides the default at context
 * creation.  Errors: XRL_EINVAL for a null context or unknown mode. */
#define XRL_SCHED_SERIAL 0
#define XRL_SCHED_FORK 1
#define XRL_SCHED_LATE 2
xrl_status xrl_ctx_set_sched(xrl_ctx ctx, int32_t mode);
/* Fused P2P (default on; XRL_FUSE=0 at context creation turns it off): in the
 * forked schedules, three spare warps of the M2L kernel take P2P leaf tasks from
 * the counter the standalone P2P kernel uses (not on trees partitioned more than
 * 2 ways, where the rank's M2L is short).  Results equal the unfused path up
 * to FP32 summation order.  Errors: XRL_EINVAL for a null context. */
xrl_status xrl_ctx_set_fuse(xrl_ctx ctx, int32_t on);

/* Per-phase device timing (CUDA events on the stream each phase runs on) of
 * the MVM kernels, accumulated while enabled.  names: "pack","p2m","m2m","m2l",
 * "p2l","l2l","l2p_m2p","p2p","near".  xrl_timing_get fills ms[i] and
 * launches[i] for i < n (n = xrl_timing_count()). */
xrl_status xrl_timing_enable(xrl_ctx ctx, int on);
int32_t xrl_timing_count(void);
const char* xrl_timing_name(int32_t i);
xrl_status xrl_timing_get(xrl_ctx ctx, double* ms, int64_t* launches);
xrl_status xrl_timing_reset(xrl_ctx ctx);

/* Number of library kernels launched on this context so far (all entry
 * points; used to report gpu_launches of a timed region). */
int64_t xrl_launch_count(xrl_ctx ctx);


/* ------------------------------------------------------------------------
 * Loop-space operator, diagonal-of-P preconditioner and GMRES
 * ------------------------------------------------------------------------ */
typedef struct xrl_topo_s* xrl_topo;
typedef struct xrl_op_s* xrl_op;
typedef struct xrl_precond_s* xrl_precond;

/* A port: two terminal panel sets (panel ids in the mesh's original order).
 * Each terminal is a super-node tied to its panels by zero-impedance
 * branches; the port branch carries the source (SPEC.md:52-55 convention;
 * PAPER.md:90 V_edge = phi_i - phi_j on the excited branch). */
typedef struct {
    int32_t n_plus, n_minus;
    const int32_t* plus;
    const int32_t* minus;
} xrl_port;

typedef struct {
    int64_t n_panels, n_edges, n_branches, n_loops;
    int32_t n_ports, n_components;
    int64_t n_vertex_loops, n_fundamental_loops, n_terminal_loops;
    int64_t nnz_m, nnz_c;
} xrl_topo_info_t;

/* PEEC graph and loop basis (host, setup).  Edges: panels sharing an edge,
 * reference direction from the lower to the higher library index.  CM maps
 * A_t (Alg. 1): A_t(e,i) = (m_e - c_i)_t, A_t(e,j) = (c_j - m_e)_t.
 * Loop matrix M (Eq. 7) from local vertex loops (fundamental
 * cycles if those do not span the cycle space), terminal loops and one port
 * loop per port.  Errors: XRL_EGEOM (non-manifold edge, disconnected
 * terminals), XRL_EINVAL. */
xrl_status xrl_topology_build(xrl_tree tree, int32_t n_ports, const xrl_port* ports, xrl_topo* out);
xrl_status xrl_topology_info(xrl_topo topo, xrl_topo_info_t* info);
/* Host export for tests (any pointer may be NULL).  branch_nodes int32
 * [n_branches][2] (panel ids in mesh order, or -1-s for super-node s);
 * branch_kind int8 (0 edge, 1 terminal, 2 port); edge_mid double [n_edges][3];
 * M as CSR over loops: m_ptr int64 [n_loops+1], m_branch int32, m_sign int8;
 * port_loop int32 [n_ports]; loop_kind int8 (0 vertex, 1 fundamental,
 * 2 terminal, 3 port); C = M A (loop rows): c_ptr int64 [n_loops+1],
 * c_panel int32 (mesh order), c_val double [nnz][3]. */
xrl_status xrl_topology_export(xrl_topo topo, int32_t* branch_nodes, int8_t* branch_kind, double* edge_mid,
                               int64_t* m_ptr, int32_t* m_branch, int8_t* m_sign, int32_t* port_loop,
                               int8_t* loop_kind, int64_t* c_ptr, int32_t* c_panel, double* c_val);
void xrl_topology_destroy(xrl_topo topo);

/* Equivalent surface impedance, Sonnet double-plane model (Eq. 3)
 * read as Z_s = (1+j) R_RF sqrt(f) / (1 - exp(-(1+j) R_RF sqrt(f)/R_DC)),
 * R_DC = 2/(sigma zeta), R_RF = sqrt(pi mu0 / sigma) (reading R12);
 * f = 0 gives the limit R_DC.  Host function. */
xrl_status xrl_esi(double sigma, double zeta, double freq_hz, double* zs_re, double* zs_im);

/* Loop-space operator at one frequency (Eq. 8-9):
 *   A v = M sum_t A_t [ diag(Z_s/A) + alpha P ] A_t^T M^T v,  alpha = j omega mu0/(4 pi)
 * applied as u_t = C_t^T v (C_t = M A_t), P u_t by xrl_mvm, w = sum_t C_t y_t.
 * zs: per-panel complex Z_s (double [n][2], mesh order) or NULL to use
 * xrl_esi(sigma, zeta, freq) for every panel.  Handles are borrowed.
 * On a partitioned tree (part_world > 1) the operator is sharded in loop
 * space: the rank owns the contiguous loops
 * [loop_offset, loop_offset + n_loops_local) (xrl_operator_info; cuts follow
 * the owner of each loop's lowest panel) and every vector of the operator,
 * preconditioner and GMRES calls is that slice; an apply exchanges the loop
 * values its panels read and the panel values its loops read, around the
 * sharded xrl_mvm.  xrl_extract runs on single-rank trees only. */
xrl_status xrl_operator_create(xrl_tree tree, xrl_near near, xrl_topo topo, const double* zs, double sigma,
                               double zeta, double freq_hz, xrl_op* out);
/* w = A v; v, w device complex64 [nrhs][n_loops] (partitioned: [nrhs][n_loops_local], collective over
 * the context's communicator; XRL_EUNSUPPORTED on a virtual rank), must not alias. */
xrl_status xrl_operator_apply(xrl_op op, const void* v, void* w, int32_t nrhs);
/* This rank's loop slice: first loop and count (0 and n_loops on a single-rank operator), and the
 * apply's exchange volume per right-hand side: loop values and panel values sent + received (any
 * pointer may be NULL). */
xrl_status xrl_operator_info(xrl_op op, int64_t* loop_offset, int64_t* n_loops_local, int64_t* loop_halo,
                             int64_t* panel_halo);
/* Virtual ranks: the sharded operator of k operators built on the k trees of one xrl_mvm_vranks
 * partition (one single-rank context), applied in one call with device-copy exchanges; v[r], w[r]:
 * rank r's slices.  k = 1 with a single-rank operator is the plain apply. */
xrl_status xrl_operator_apply_vranks(int32_t k, const xrl_op* ops, const void* const* v, void* const* w, int32_t nrhs);
void xrl_operator_destroy(xrl_op op);

/* Diagonal-of-P preconditioner (Eq. 10-11) in block-Jacobi
 * form (reading R13): Q = sum_t C_t diag(Z_s/A + alpha P_kk) C_t^T,
 * loops cut into consecutive (Morton-ordered) blocks of <= block_size
 * (<= 64; on a sharded operator: of the rank's loops, no communication in
 * the apply), each diagonal block LU-inverted in FP64 and stored complex64.
 * XRL_ESINGULAR if a pivot falls below 1e-13 of the block's largest entry. */
xrl_status xrl_precond_build(xrl_op op, int32_t block_size, xrl_precond* out);
/* Exact diagonal-of-P preconditioner: the same Q, factorised
 * whole, as Eq. 11 applies it (where Pardiso factorises Q once
 * per frequency).  Q is assembled on the host in FP64 complex, ordered by nested
 * dissection (METIS; else approximate minimum degree) and factorised by a host
 * sparse LU with partial pivoting (cuSOLVER low-level csrlu, loaded at run time);
 * xrl_precond_apply then copies v to the host, solves, and copies z back
 * (synchronous).  XRL_EINVAL if cuSOLVER cannot be loaded or n_loops >= 2^31,
 * XRL_ESINGULAR on a zero pivot.  xrl_precond_export rejects this kind. */
xrl_status xrl_precond_build_exact(xrl_op op, xrl_precond* out);
/* Preconditioner of a given kind (Table IV's comparison):
 *   XRL_PRECOND_DIAG_P (0): Eq. 10's Q = Z_s + M sum_t A_t P_d A_t^T M^T;
 *   XRL_PRECOND_DIAG_L (1): the traditional diagonal-of-L preconditioner of
 *     PAPER.md:120-122, Q_L = Z_s + j omega L_d mapped to loops,
 *     Q_L = M [sum_t A_t diag(Z_s/A) A_t^T + alpha diag(L_ee)] M^T with
 *     L_ee the diagonal of the edge-edge matrix sum_t A_t P A_t^T (each edge's
 *     two panels: their P self terms and their mutual near entry).
 * block_size 1..64: block-Jacobi (FP64 Gauss-Jordan per block, complex64
 * storage); -1: the whole Q factorised (as xrl_precond_build_exact); -2: an
 * incomplete LU(0) of the whole Q (reverse Cuthill-McKee order, FP64 complex,
 * factorised on the GPU by cuSPARSE csrilu02 -- no host factorisation), applied
 * by the same two GPU triangular solves.
 * Errors as xrl_precond_build / xrl_precond_build_exact, plus XRL_EINVAL for
 * a bad kind and XRL_EGEOM if an edge's panel pair is missing from the near
 * field. */
#define XRL_PRECOND_DIAG_P 0
#define XRL_PRECOND_DIAG_L 1
xrl_status xrl_precond_build_kind(xrl_op op, int32_t kind, int32_t block_size, xrl_precond* out);
/* z = blockdiag(Q)^-1 v (exact kind: Q^-1 v); device complex64 [nrhs][n_loops]. */
xrl_status xrl_precond_apply(xrl_precond pc, const void* v, void* z, int32_t nrhs);
/* Host export of the block partition and the inverse blocks (tests):
 * block_ptr int32 [n_blocks+1] (loop ranges), inv complex64 [n_blocks][bs][bs]
 * (row-major, rows/cols beyond the block's size are 0). */
xrl_status xrl_precond_export(xrl_precond pc, int32_t* n_blocks, int32_t* block_size, int32_t* block_ptr, void* inv);
void xrl_precond_destroy(xrl_precond pc);

/* Restarted GMRES (restart 50; relative residual 1e-4 above
 * 1 MHz, 1e-6 at or below, reading C-A8), preconditioned on the right (reading
 * R15; the left form of Eq. 11 selectable), one
 * Krylov space per right-hand side, all columns stepping together so every
 * operator call is batched.  CGS2 orthogonalisation; Hessenberg/Givens in FP64.
 * tol <= 0 selects the paper's frequency rule.  b, x: device complex64
 * [nrhs][n_loops] (x holds x0 on entry).  Per-column outputs (host, may be
 * NULL): iters int32, rre double (preconditioned, as converged on),
 * true_rre double (||b - A x|| / ||b||), converged int32.  Blocking; returns
 * XRL_ENOCONV if any column did not converge. */
typedef struct {
    int32_t restart;
    int32_t max_iters;
    double tol;
    int32_t right_precond;  /* 1: right (A M^-1 u = b, x = M^-1 u: GMRES minimises and tests the true
                               residual; used when opts is NULL, reading R15); 0: left,
                               the form of Eq. 11 (tests the preconditioned residual) */
} xrl_gmres_opts;
xrl_status xrl_gmres(xrl_op op, xrl_precond pc, const void* b, void* x, int32_t nrhs, const xrl_gmres_opts* opts,
                     int32_t* iters, double* rre, double* true_rre, int32_t* converged);
/* GMRES over k virtual ranks (the operators / preconditioners of one xrl_mvm_vranks partition; pcs NULL
 * = none): b[r], x[r] rank r's loop slices; the inner products are summed over the ranks (on a multi-rank
 * context xrl_gmres all-reduces them over NCCL instead).  Outputs and errors as xrl_gmres. */
xrl_status xrl_gmres_vranks(int32_t k, const xrl_op* ops, const xrl_precond* pcs, const void* const* b,
                            void* const* x, int32_t nrhs, const xrl_gmres_opts* opts, int32_t* iters, double* rre,
                            double* true_rre, int32_t* converged);

/* Port excitation V_l = M V_branch with `volts` on port `port`'s branch
 * (device complex64 [n_loops], overwritten), and port currents read back from
 * loop currents (I_port = current of the port branch = I_l of its loop):
 * x device complex64 [nrhs][n_loops] -> i_ports host double [nrhs][n_ports][2]. */
xrl_status xrl_port_rhs(xrl_topo topo, int32_t port, double volts, void* b);
xrl_status xrl_port_currents(xrl_topo topo, const void* x, int32_t nrhs, double* i_ports);

/* R/L extraction sweep (PAPER.md:152 solves the loop system at every frequency
 * point and reports R and L).  For each freqs[j] > 0: the operator (xrl_operator_create with zs,
 * sigma, zeta), the diagonal-of-P preconditioner (block-Jacobi with block_size <= 64, 0 = 64; the
 * exact Q^-1 of xrl_precond_build_exact if block_size < 0), one GMRES (opts; NULL =
 * restart 50, the paper's tolerance rule) with the n_ports unit-voltage port excitations as batched
 * right-hand sides, the port currents give the admittance Y[:, q] = I(port q excited), and
 * Z = Y^-1 (FP64), R = Re Z, L = Im Z / (2 pi f).  Host outputs, each may be NULL:
 * z double [n_freq][n_ports][n_ports][2] (re, im), r and l double [n_freq][n_ports][n_ports],
 * iters int32 and true_rre double [n_freq][n_ports].  Handles are borrowed.  Errors: XRL_EINVAL
 * (no ports, n_freq < 1, f <= 0), XRL_ESINGULAR (singular Y), XRL_ENOCONV (some column did not
 * converge; outputs still filled), plus those of the calls above. */
xrl_status xrl_extract(xrl_tree tree, xrl_near near, xrl_topo topo, const double* zs, double sigma, double zeta,
                       int32_t n_freq, const double* freqs, int32_t block_size, const xrl_gmres_opts* opts,
                       double* z, double* r, double* l, int32_t* iters, double* true_rre);

#ifdef __cplusplus
}
#endif

#endif /* XRL_H */
