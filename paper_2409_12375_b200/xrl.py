"""Thin Python binding of libxrl.so (include/xrl.h): argument marshalling only.

Every step of the hot path runs in the CUDA library; there is no CPU fallback.
Device vectors are torch tensors (complex64, contiguous, on the context's
device) passed by data_ptr(); the context runs on the caller's torch stream.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libxrl.so")

XRL_MVM_FULL, XRL_MVM_NEAR_ONLY, XRL_MVM_FAR_ONLY = 0, 1, 2
STATUS = {0: "XRL_OK", 1: "XRL_ENOCONV", -1: "XRL_EINVAL", -2: "XRL_EDIM", -3: "XRL_EPROVENANCE",
          -4: "XRL_EGEOM", -5: "XRL_ESINGULAR", -6: "XRL_ENOMEM", -7: "XRL_ECUDA", -8: "XRL_ENCCL",
          -9: "XRL_ENOFREQ", -10: "XRL_EUNSUPPORTED"}

# symbols declared in include/xrl.h (checked by tests/test_abi.py)
EXPORTS = [
    "xrl_last_error", "xrl_version", "xrl_ctx_create", "xrl_ctx_sync", "xrl_ctx_destroy",
    "xrl_tree_build", "xrl_tree_build_poly", "xrl_tree_destroy", "xrl_tree_info", "xrl_tree_perm", "xrl_to_library_order",
    "xrl_from_library_order", "xrl_tree_export", "xrl_near_assemble", "xrl_near_destroy",
    "xrl_near_export", "xrl_near_export_rows", "xrl_near_info", "xrl_mvm", "xrl_mvm_host", "xrl_mvm_host_batch", "xrl_timing_enable", "xrl_timing_count",
    "xrl_timing_name", "xrl_timing_get", "xrl_timing_reset", "xrl_launch_count", "xrl_ctx_set_sched", "xrl_ctx_set_fuse", "xrl_extract",
    "xrl_topology_build", "xrl_topology_info", "xrl_topology_export", "xrl_topology_destroy", "xrl_esi",
    "xrl_operator_create", "xrl_operator_apply", "xrl_operator_destroy", "xrl_precond_build",
    "xrl_precond_build_exact", "xrl_precond_build_kind", "xrl_precond_apply", "xrl_operator_info",
    "xrl_operator_apply_vranks", "xrl_gmres_vranks", "xrl_precond_export", "xrl_precond_destroy", "xrl_gmres", "xrl_port_rhs",
    "xrl_port_currents", "xrl_partition_cuts", "xrl_nccl_unique_id", "xrl_mvm_vranks", "xrl_exchange_info", "xrl_plan_exchange",
]


class XrlError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class FmmOpts(ctypes.Structure):
    _fields_ = [("p", ctypes.c_int32), ("leaf_max", ctypes.c_int32), ("max_depth", ctypes.c_int32),
                ("part_rank", ctypes.c_int32), ("part_world", ctypes.c_int32)]


class NearOpts(ctypes.Structure):
    _fields_ = [("eta", ctypes.c_double), ("galerkin", ctypes.c_int32)]


class TreeInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("n_local", ctypes.c_int64), ("offset", ctypes.c_int64),
                ("n_boxes", ctypes.c_int32), ("n_leaves", ctypes.c_int32), ("n_levels", ctypes.c_int32),
                ("p", ctypes.c_int32), ("n_v_pairs", ctypes.c_int64), ("n_x_pairs", ctypes.c_int64),
                ("n_w_pairs", ctypes.c_int64), ("n_u_pairs", ctypes.c_int64), ("n_p2p", ctypes.c_int64),
                ("root_lo", ctypes.c_double * 3), ("root_width", ctypes.c_double),
                ("n_m2l_tiles", ctypes.c_int64), ("n_m2l_subtiles", ctypes.c_int64)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["root_lo"] = list(self.root_lo)
        return d


class Port(ctypes.Structure):
    _fields_ = [("n_plus", ctypes.c_int32), ("n_minus", ctypes.c_int32),
                ("plus", ctypes.c_void_p), ("minus", ctypes.c_void_p)]


class TopoInfo(ctypes.Structure):
    _fields_ = [("n_panels", ctypes.c_int64), ("n_edges", ctypes.c_int64), ("n_branches", ctypes.c_int64),
                ("n_loops", ctypes.c_int64), ("n_ports", ctypes.c_int32), ("n_components", ctypes.c_int32),
                ("n_vertex_loops", ctypes.c_int64), ("n_fundamental_loops", ctypes.c_int64),
                ("n_terminal_loops", ctypes.c_int64), ("nnz_m", ctypes.c_int64), ("nnz_c", ctypes.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class GmresOpts(ctypes.Structure):
    _fields_ = [("restart", ctypes.c_int32), ("max_iters", ctypes.c_int32), ("tol", ctypes.c_double),
                ("right_precond", ctypes.c_int32)]


_lib = None


def lib():
    """Load libxrl.so; fails loudly if the CUDA library was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2409_12375_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P, i32, i64, u32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
        pp = ctypes.POINTER(ctypes.c_void_p)
        L.xrl_last_error.restype = ctypes.c_char_p
        L.xrl_version.restype = ctypes.c_char_p
        L.xrl_ctx_create.argtypes = [ctypes.c_int, P, ctypes.c_int, ctypes.c_int, P, pp]
        L.xrl_ctx_sync.argtypes = [P]
        L.xrl_ctx_destroy.argtypes = [P]
        L.xrl_ctx_destroy.restype = None
        L.xrl_tree_build.argtypes = [P, i64, P, i64, P, ctypes.POINTER(FmmOpts), pp]
        L.xrl_tree_build_poly.argtypes = [P, i64, P, i64, P, ctypes.POINTER(FmmOpts), pp]
        L.xrl_tree_destroy.argtypes = [P]
        L.xrl_tree_destroy.restype = None
        L.xrl_tree_info.argtypes = [P, ctypes.POINTER(TreeInfo)]
        L.xrl_tree_perm.argtypes = [P, P]
        L.xrl_to_library_order.argtypes = [P, P, P, i32]
        L.xrl_from_library_order.argtypes = [P, P, P, i32]
        L.xrl_tree_export.argtypes = [P] * 15
        L.xrl_near_assemble.argtypes = [P, ctypes.POINTER(NearOpts), pp]
        L.xrl_near_destroy.argtypes = [P]
        L.xrl_near_destroy.restype = None
        L.xrl_near_export.argtypes = [P, P, P, P, P, P]
        L.xrl_near_export_rows.argtypes = [P, i64, P, P, P, P, P]
        L.xrl_near_info.argtypes = [P, P, P, P]
        L.xrl_mvm.argtypes = [P, P, P, P, i32, u32]
        L.xrl_mvm_host.argtypes = [P, P, P, P, i32, u32]
        L.xrl_mvm_host_batch.argtypes = [P, P, P, P, i32, i32, u32]
        L.xrl_timing_enable.argtypes = [P, ctypes.c_int]
        L.xrl_timing_count.restype = i32
        L.xrl_timing_name.argtypes = [i32]
        L.xrl_timing_name.restype = ctypes.c_char_p
        L.xrl_timing_get.argtypes = [P, P, P]
        L.xrl_timing_reset.argtypes = [P]
        L.xrl_launch_count.argtypes = [P]
        L.xrl_launch_count.restype = i64
        L.xrl_ctx_set_sched.argtypes = [P, i32]
        L.xrl_ctx_set_sched.restype = ctypes.c_int32
        L.xrl_ctx_set_fuse.argtypes = [P, i32]
        L.xrl_ctx_set_fuse.restype = ctypes.c_int32
        L.xrl_extract.argtypes = [P, P, P, P, ctypes.c_double, ctypes.c_double, i32, P, i32, P, P, P, P, P, P]
        L.xrl_extract.restype = ctypes.c_int32
        L.xrl_topology_build.argtypes = [P, i32, P, pp]
        L.xrl_topology_info.argtypes = [P, ctypes.POINTER(TopoInfo)]
        L.xrl_topology_export.argtypes = [P] * 12
        L.xrl_topology_destroy.argtypes = [P]
        L.xrl_topology_destroy.restype = None
        f64 = ctypes.c_double
        L.xrl_esi.argtypes = [f64, f64, f64, P, P]
        L.xrl_operator_create.argtypes = [P, P, P, P, f64, f64, f64, pp]
        L.xrl_operator_apply.argtypes = [P, P, P, i32]
        L.xrl_operator_destroy.argtypes = [P]
        L.xrl_operator_destroy.restype = None
        L.xrl_precond_build.argtypes = [P, i32, pp]
        L.xrl_precond_build_exact.argtypes = [P, pp]
        L.xrl_precond_build_kind.argtypes = [P, i32, i32, pp]
        L.xrl_operator_info.argtypes = [P, P, P, P, P]
        L.xrl_operator_apply_vranks.argtypes = [i32, P, P, P, i32]
        L.xrl_gmres_vranks.argtypes = [i32, P, P, P, P, i32, P, P, P, P, P]
        for name in ("xrl_operator_info", "xrl_operator_apply_vranks", "xrl_gmres_vranks"):
            getattr(L, name).restype = ctypes.c_int32
        L.xrl_precond_apply.argtypes = [P, P, P, i32]
        L.xrl_precond_export.argtypes = [P, P, P, P, P]
        L.xrl_precond_destroy.argtypes = [P]
        L.xrl_precond_destroy.restype = None
        L.xrl_gmres.argtypes = [P, P, P, P, i32, ctypes.POINTER(GmresOpts), P, P, P, P]
        L.xrl_port_rhs.argtypes = [P, i32, f64, P]
        L.xrl_port_currents.argtypes = [P, P, i32, P]
        L.xrl_partition_cuts.argtypes = [i64, P, i32, P]
        L.xrl_nccl_unique_id.argtypes = [P]
        L.xrl_mvm_vranks.argtypes = [i32, P, P, P, P, i32, u32, P, P]
        L.xrl_exchange_info.argtypes = [P, P, P, P, P, P, P]
        L.xrl_plan_exchange.argtypes = [i32] + [P] * 11 + [i64, P, P, i32, P, i32] + [P] * 10
        for name in ("xrl_partition_cuts", "xrl_nccl_unique_id", "xrl_mvm_vranks", "xrl_exchange_info",
                     "xrl_plan_exchange"):
            getattr(L, name).restype = ctypes.c_int32
        for name in ("xrl_topology_build", "xrl_topology_info", "xrl_topology_export", "xrl_esi",
                     "xrl_operator_create", "xrl_operator_apply", "xrl_precond_build", "xrl_precond_build_exact", "xrl_precond_build_kind",
                     "xrl_precond_apply",
                     "xrl_precond_export", "xrl_gmres", "xrl_port_rhs", "xrl_port_currents"):
            getattr(L, name).restype = ctypes.c_int32
        for name in ("xrl_ctx_create", "xrl_ctx_sync", "xrl_tree_build", "xrl_tree_build_poly", "xrl_tree_info", "xrl_tree_perm",
                     "xrl_to_library_order", "xrl_from_library_order", "xrl_tree_export", "xrl_near_assemble",
                     "xrl_near_export", "xrl_mvm", "xrl_mvm_host", "xrl_mvm_host_batch", "xrl_timing_enable", "xrl_timing_get",
                     "xrl_timing_reset"):
            getattr(L, name).restype = ctypes.c_int32
        _lib = L
    return _lib


def check(status):
    if status < 0:
        raise XrlError(status, lib().xrl_last_error().decode())
    return status


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(ctypes.c_void_p)
    return ctypes.c_void_p(a.data_ptr())


def _dev_vec(t, n, name):
    import torch
    if not isinstance(t, torch.Tensor) or t.dtype != torch.complex64 or not t.is_cuda or not t.is_contiguous():
        raise XrlError(-1, f"{name} must be a contiguous complex64 CUDA tensor")
    if t.dim() != 2 or t.shape[1] != n:
        raise XrlError(-2, f"{name} must have shape [nvec, {n}]")
    return t


def partition_cuts(weights, world: int) -> np.ndarray:
    """xrl_partition_cuts: balanced contiguous cuts (int64 [world+1])."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    cuts = np.empty(world + 1, dtype=np.int64)
    check(lib().xrl_partition_cuts(w.size, _ptr(w), world, _ptr(cuts)))
    return cuts


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    check(lib().xrl_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return bytes(buf)


class Context:
    """xrl_ctx_create on `device`, running on torch's current stream (or
    `stream`).  rank/world > 1 needs the same 128-byte ncclUniqueId on every
    rank (see distributed_context)."""

    def __init__(self, device: int = 0, stream=None, rank: int = 0, world: int = 1, nccl_id: bytes | None = None):
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.device = device
        self.stream = stream
        self.rank, self.world = rank, world
        idbuf = None
        if world > 1:
            idbuf = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
        h = ctypes.c_void_p()
        check(lib().xrl_ctx_create(device, ctypes.c_void_p(stream.cuda_stream), rank, world,
                                   ctypes.cast(idbuf, ctypes.c_void_p) if idbuf is not None else None,
                                   ctypes.byref(h)))
        self.h = h

    def sync(self):
        check(lib().xrl_ctx_sync(self.h))

    SCHED_SERIAL, SCHED_FORK, SCHED_LATE = 0, 1, 2

    def set_sched(self, mode: int):
        """xrl_ctx_set_sched: 0 serial (isolated phase times), 1 fork (default), 2 late fork."""
        check(lib().xrl_ctx_set_sched(self.h, int(mode)))

    def set_fuse(self, on: bool):
        """xrl_ctx_set_fuse: P2P leaf tasks also in the M2L kernel's spare warps (default on)."""
        check(lib().xrl_ctx_set_fuse(self.h, int(bool(on))))

    def timing_enable(self, on=True):
        check(lib().xrl_timing_enable(self.h, int(on)))

    def timing_reset(self):
        check(lib().xrl_timing_reset(self.h))

    def timing(self):
        n = lib().xrl_timing_count()
        ms = np.zeros(n)
        cnt = np.zeros(n, dtype=np.int64)
        check(lib().xrl_timing_get(self.h, _ptr(ms), _ptr(cnt)))
        return {lib().xrl_timing_name(i).decode(): (float(ms[i]), int(cnt[i])) for i in range(n)}

    def launch_count(self) -> int:
        return int(lib().xrl_launch_count(self.h))

    def close(self):
        if getattr(self, "h", None):
            lib().xrl_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def distributed_context(device: int = 0, stream=None) -> Context:
    """Context over the torch.distributed process group: rank 0 creates the
    ncclUniqueId, torch.distributed broadcasts it (plumbing only)."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    if world == 1:
        return Context(device, stream)
    buf = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
    if dist.get_backend() == "nccl":
        b = buf.cuda(device)
        dist.broadcast(b, 0)
        buf = b.cpu()
    else:
        dist.broadcast(buf, 0)
    return Context(device, stream, rank, world, bytes(buf.numpy().tobytes()))


class Tree:
    """xrl_tree_build over a triangle mesh (host FP64 verts [nv,3], int32 tris [n,3]); a [n,4] panel array
    (-1 in the last column for triangles, else a rectangle) goes to xrl_tree_build_poly (hybrid mesh)."""

    def __init__(self, ctx: Context, verts, tris, p=10, leaf_max=64, max_depth=21, part_rank=None, part_world=None):
        self.ctx = ctx
        v = np.ascontiguousarray(verts, dtype=np.float64)
        t = np.ascontiguousarray(tris, dtype=np.int32)
        if part_world is None:
            part_rank, part_world = (ctx.rank, ctx.world) if ctx.world > 1 else (0, 0)
        opts = FmmOpts(p, leaf_max, max_depth, part_rank or 0, part_world)
        h = ctypes.c_void_p()
        build = lib().xrl_tree_build_poly if t.shape[1] == 4 else lib().xrl_tree_build
        check(build(ctx.h, v.shape[0], _ptr(v), t.shape[0], _ptr(t), ctypes.byref(opts), ctypes.byref(h)))
        self.h = h
        self.n = t.shape[0]
        i = self.info()
        self.n_local, self.offset = int(i["n_local"]), int(i["offset"])

    def info(self) -> dict:
        ti = TreeInfo()
        check(lib().xrl_tree_info(self.h, ctypes.byref(ti)))
        return ti.as_dict()

    def perm(self) -> np.ndarray:
        out = np.empty(self.n, dtype=np.int32)
        check(lib().xrl_tree_perm(self.h, _ptr(out)))
        return out

    def to_library_order(self, x_user, out=None):
        import torch
        _dev_vec(x_user, self.n, "x_user")
        out = torch.empty_like(x_user) if out is None else out
        check(lib().xrl_to_library_order(self.h, _ptr(x_user), _ptr(out), x_user.shape[0]))
        return out

    def from_library_order(self, x_lib, out=None):
        import torch
        _dev_vec(x_lib, self.n, "x_lib")
        out = torch.empty_like(x_lib) if out is None else out
        check(lib().xrl_from_library_order(self.h, _ptr(x_lib), _ptr(out), x_lib.shape[0]))
        return out

    def export(self) -> dict:
        i = self.info()
        nb = i["n_boxes"]
        a = {k: np.empty(nb, dtype=np.int32) for k in ("level", "parent", "pb", "pe", "is_leaf")}
        a["ijk"] = np.empty((nb, 3), dtype=np.int32)
        for k, cnt in (("u", i["n_u_pairs"]), ("v", i["n_v_pairs"]), ("x", i["n_x_pairs"]), ("w", i["n_w_pairs"])):
            a[k + "_ptr"] = np.empty(nb + 1, dtype=np.int64)
            a[k + "_src"] = np.empty(max(cnt, 1), dtype=np.int32)
        check(lib().xrl_tree_export(self.h, _ptr(a["level"]), _ptr(a["ijk"]), _ptr(a["parent"]), _ptr(a["pb"]),
                                    _ptr(a["pe"]), _ptr(a["is_leaf"]), _ptr(a["u_ptr"]), _ptr(a["u_src"]),
                                    _ptr(a["v_ptr"]), _ptr(a["v_src"]), _ptr(a["x_ptr"]), _ptr(a["x_src"]),
                                    _ptr(a["w_ptr"]), _ptr(a["w_src"])))
        return a

    def close(self):
        if getattr(self, "h", None):
            lib().xrl_tree_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Near:
    """xrl_near_assemble: near-field CSR (library order)."""

    def __init__(self, tree: Tree, eta=1.5, galerkin=False):
        self.tree = tree
        h = ctypes.c_void_p()
        check(lib().xrl_near_assemble(tree.h, ctypes.byref(NearOpts(eta, int(bool(galerkin)))), ctypes.byref(h)))
        self.h = h

    def nnz(self) -> int:
        nnz = ctypes.c_int64()
        check(lib().xrl_near_export(self.h, None, None, None, None, ctypes.byref(nnz)))
        return int(nnz.value)

    def export(self):
        nnz = ctypes.c_int64()
        check(lib().xrl_near_export(self.h, None, None, None, None, ctypes.byref(nnz)))
        n = self.tree.n
        ptr = np.empty(n + 1, dtype=np.int64)
        col = np.empty(max(nnz.value, 1), dtype=np.int32)
        v32 = np.empty(max(nnz.value, 1), dtype=np.float32)
        v64 = np.empty(max(nnz.value, 1), dtype=np.float64)
        check(lib().xrl_near_export(self.h, _ptr(ptr), _ptr(col), _ptr(v32), _ptr(v64), ctypes.byref(nnz)))
        k = nnz.value
        return ptr, col[:k], v32[:k], v64[:k]

    def info(self) -> dict:
        v = [ctypes.c_int64() for _ in range(3)]
        check(lib().xrl_near_info(self.h, *[ctypes.byref(a) for a in v]))
        return dict(zip(("nnz", "n_segments", "n_entries"), [int(a.value) for a in v]))

    def export_rows(self, rows):
        """Selected library-order rows: (ptr, col, v32, v64) over those rows only."""
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        cnt = np.empty(max(rows.size, 1), dtype=np.int64)
        check(lib().xrl_near_export_rows(self.h, rows.size, _ptr(rows), _ptr(cnt), None, None, None))
        ptr = np.zeros(rows.size + 1, dtype=np.int64)
        np.cumsum(cnt[:rows.size], out=ptr[1:])
        k = int(ptr[-1])
        col = np.empty(max(k, 1), dtype=np.int32)
        v32 = np.empty(max(k, 1), dtype=np.float32)
        v64 = np.empty(max(k, 1), dtype=np.float64)
        check(lib().xrl_near_export_rows(self.h, rows.size, _ptr(rows), _ptr(cnt), _ptr(col), _ptr(v32), _ptr(v64)))
        return ptr, col[:k], v32[:k], v64[:k]

    def close(self):
        if getattr(self, "h", None):
            lib().xrl_near_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def mvm(tree: Tree, near: Near, x, y=None, flags=XRL_MVM_FULL):
    """y = P x on the device (library order, complex64 [nvec][n_local]; the
    rank's slice on a multi-rank context)."""
    import torch
    _dev_vec(x, tree.n_local, "x")
    y = torch.empty_like(x) if y is None else _dev_vec(y, tree.n_local, "y")
    check(lib().xrl_mvm(tree.h, near.h, _ptr(x), _ptr(y), x.shape[0], flags))
    return y


def mvm_vranks(trees, nears, xs, ys=None, flags=XRL_MVM_FULL, timing=False):
    """xrl_mvm_vranks: the sharded MVM of k virtual ranks on one GPU.  trees[r] / nears[r]: rank r of a
    k-way partition (Tree(..., part_rank=r, part_world=k)) on one single-rank context; xs[r]: rank r's
    slice [nvec][n_local(r)] (library order).  Returns ys (and, with timing=True, (rank_ms [k],
    exchange_ms))."""
    import torch
    k = len(trees)
    if ys is None:
        ys = [torch.empty_like(x) for x in xs]
    for r in range(k):
        _dev_vec(xs[r], trees[r].n_local, "x")
        _dev_vec(ys[r], trees[r].n_local, "y")
    th = (ctypes.c_void_p * k)(*[t.h.value for t in trees])
    nh = (ctypes.c_void_p * k)(*[n.h.value for n in nears])
    xp = (ctypes.c_void_p * k)(*[x.data_ptr() for x in xs])
    yp = (ctypes.c_void_p * k)(*[y.data_ptr() for y in ys])
    rms = np.zeros(k)
    ems = ctypes.c_double()
    check(lib().xrl_mvm_vranks(k, th, nh, xp, yp, xs[0].shape[0], flags, _ptr(rms) if timing else None,
                               ctypes.byref(ems) if timing else None))
    return (ys, rms, ems.value) if timing else ys


def plan_exchange(tree: dict, near_ptr, near_col, cuts, rank) -> dict:
    """xrl_plan_exchange (host, no GPU): rank `rank`'s exchange plan for a tree given as host arrays
    (dict with pb, pe, child, v_ptr/v_src, x_ptr/x_src, w_ptr/w_src, u_ptr/u_src) and a near pattern."""
    a = {k: np.ascontiguousarray(tree[k], dtype=np.int64 if k.endswith("_ptr") else np.int32)
         for k in ("pb", "pe", "child", "v_ptr", "v_src", "x_ptr", "x_src", "w_ptr", "w_src", "u_ptr", "u_src")}
    for k in ("v_src", "x_src", "w_src", "u_src"):
        if a[k].size == 0:
            a[k] = np.zeros(1, np.int32)
    near_ptr = np.ascontiguousarray(near_ptr, dtype=np.int64)
    near_col = np.ascontiguousarray(near_col, dtype=np.int32)
    cuts = np.ascontiguousarray(cuts, dtype=np.int32)
    world = cuts.size - 1
    nbox = a["pb"].size
    n = near_ptr.size - 1
    nsh = ctypes.c_int64()
    offs = {k: np.zeros(world + 1, np.int64) for k in ("let_roff", "let_soff", "halo_roff", "halo_soff")}

    def call(sh, lr, ls, hr, hs):
        check(lib().xrl_plan_exchange(nbox, *[_ptr(a[k]) for k in ("pb", "pe", "child", "v_ptr", "v_src", "x_ptr",
                                                                     "x_src", "w_ptr", "w_src", "u_ptr", "u_src")],
                                      n, _ptr(near_ptr), _ptr(near_col), world, _ptr(cuts), rank, ctypes.byref(nsh),
                                      _ptr(sh), _ptr(offs["let_roff"]), _ptr(lr), _ptr(offs["let_soff"]), _ptr(ls),
                                      _ptr(offs["halo_roff"]), _ptr(hr), _ptr(offs["halo_soff"]), _ptr(hs)))
    call(None, None, None, None, None)
    out = {"shared": np.zeros(max(nsh.value, 1), np.int32)}
    for k in ("let_r", "let_s", "halo_r", "halo_s"):
        out[k + "idx"] = np.zeros(max(int(offs[k + "off"][-1]), 1), np.int32)
    call(out["shared"], out["let_ridx"], out["let_sidx"], out["halo_ridx"], out["halo_sidx"])
    out["shared"] = out["shared"][:nsh.value]
    for k in ("let_r", "let_s", "halo_r", "halo_s"):
        out[k + "idx"] = out[k + "idx"][:int(offs[k + "off"][-1])]
        out[k + "off"] = offs[k + "off"]
    return out


def exchange_info(tree, near=None) -> dict:
    v = [ctypes.c_int64() for _ in range(5)]
    check(lib().xrl_exchange_info(tree.h, near.h if near is not None else None, *[ctypes.byref(a) for a in v]))
    return dict(zip(("halo_send", "halo_recv", "let_send", "let_recv", "shared"), [int(a.value) for a in v]))


def mvm_host(tree: Tree, near: Near, x_host: np.ndarray, y_host: np.ndarray | None = None, flags=XRL_MVM_FULL):
    """End-to-end y = P x with host complex64 [nvec][n] buffers in mesh order."""
    x_host = np.ascontiguousarray(x_host, dtype=np.complex64)
    if y_host is None:
        y_host = np.empty_like(x_host)
    check(lib().xrl_mvm_host(tree.h, near.h, _ptr(x_host), _ptr(y_host), x_host.shape[0], flags))
    return y_host


def mvm_host_batch(tree: Tree, near: Near, x_list, y_list, flags=XRL_MVM_FULL):
    """xrl_mvm_host_batch: y_list[k] = P x_list[k] for host complex64 [nvec][n] arrays (mesh order), the
    copies pipelined against the MVMs (pinned arrays overlap; entries may repeat)."""
    k = len(x_list)
    assert len(y_list) == k and k > 0
    nvec = x_list[0].shape[0]
    for a in list(x_list) + list(y_list):
        assert a.dtype == np.complex64 and a.flags["C_CONTIGUOUS"] and a.shape == x_list[0].shape
    xp = (ctypes.c_void_p * k)(*[a.ctypes.data for a in x_list])
    yp = (ctypes.c_void_p * k)(*[a.ctypes.data for a in y_list])
    check(lib().xrl_mvm_host_batch(tree.h, near.h, xp, yp, nvec, k, flags))
    return y_list


def esi(sigma: float, zeta: float, freq: float) -> complex:
    """Z_s of Eq. 3, reading R12."""
    re, im = ctypes.c_double(), ctypes.c_double()
    check(lib().xrl_esi(sigma, zeta, freq, ctypes.byref(re), ctypes.byref(im)))
    return complex(re.value, im.value)


class Topology:
    """xrl_topology_build: edges, CM maps (Alg. 1), loop matrix with ports."""

    def __init__(self, tree: Tree, ports=()):
        self.tree = tree
        self._keep = []
        arr = (Port * max(1, len(ports)))()
        for i, (plus, minus) in enumerate(ports):
            p = np.ascontiguousarray(plus, dtype=np.int32)
            m = np.ascontiguousarray(minus, dtype=np.int32)
            self._keep += [p, m]
            arr[i] = Port(p.size, m.size, p.ctypes.data, m.ctypes.data)
        h = ctypes.c_void_p()
        check(lib().xrl_topology_build(tree.h, len(ports), ctypes.cast(arr, ctypes.c_void_p) if ports else None,
                                       ctypes.byref(h)))
        self.h = h
        self.n_ports = len(ports)

    def info(self) -> dict:
        ti = TopoInfo()
        check(lib().xrl_topology_info(self.h, ctypes.byref(ti)))
        return ti.as_dict()

    @property
    def n_loops(self) -> int:
        return int(self.info()["n_loops"])

    def export(self) -> dict:
        i = self.info()
        nb, ne, nl = i["n_branches"], i["n_edges"], i["n_loops"]
        d = {"branch_nodes": np.empty((nb, 2), np.int32), "branch_kind": np.empty(nb, np.int8),
             "edge_mid": np.empty((ne, 3)), "m_ptr": np.empty(nl + 1, np.int64),
             "m_branch": np.empty(max(1, i["nnz_m"]), np.int32), "m_sign": np.empty(max(1, i["nnz_m"]), np.int8),
             "port_loop": np.empty(max(1, i["n_ports"]), np.int32), "loop_kind": np.empty(nl, np.int8),
             "c_ptr": np.empty(nl + 1, np.int64), "c_panel": np.empty(max(1, i["nnz_c"]), np.int32),
             "c_val": np.empty((max(1, i["nnz_c"]), 3))}
        check(lib().xrl_topology_export(self.h, *[_ptr(d[k]) for k in (
            "branch_nodes", "branch_kind", "edge_mid", "m_ptr", "m_branch", "m_sign", "port_loop", "loop_kind",
            "c_ptr", "c_panel", "c_val")]))
        d["m_branch"] = d["m_branch"][:i["nnz_m"]]
        d["m_sign"] = d["m_sign"][:i["nnz_m"]]
        d["c_panel"] = d["c_panel"][:i["nnz_c"]]
        d["c_val"] = d["c_val"][:i["nnz_c"]]
        d["port_loop"] = d["port_loop"][:i["n_ports"]]
        return d

    def port_rhs(self, port: int, volts: float = 1.0, out=None):
        import torch
        out = torch.empty((1, self.n_loops), dtype=torch.complex64, device="cuda") if out is None else out
        check(lib().xrl_port_rhs(self.h, port, volts, _ptr(out)))
        return out

    def port_currents(self, x) -> np.ndarray:
        nrhs = x.shape[0]
        out = np.empty((nrhs, self.n_ports, 2))
        check(lib().xrl_port_currents(self.h, _ptr(x), nrhs, _ptr(out)))
        return out[..., 0] + 1j * out[..., 1]

    def close(self):
        if getattr(self, "h", None):
            lib().xrl_topology_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Operator:
    """xrl_operator_create: loop-space operator of Eq. 8-9 at one frequency."""

    def __init__(self, tree: Tree, near: Near, topo: Topology, freq: float, zs=None, sigma=5.8e7, zeta=1e-4):
        self.tree, self.near, self.topo = tree, near, topo
        z = None
        if zs is not None:
            zs = np.broadcast_to(np.asarray(zs, dtype=np.complex128), (tree.n,))
            z = np.ascontiguousarray(np.stack([zs.real, zs.imag], axis=1))
        h = ctypes.c_void_p()
        check(lib().xrl_operator_create(tree.h, near.h, topo.h, _ptr(z), sigma, zeta, freq, ctypes.byref(h)))
        self.h = h
        self.freq = freq

    def apply(self, v, w=None):
        import torch
        w = torch.empty_like(v) if w is None else w
        check(lib().xrl_operator_apply(self.h, _ptr(v), _ptr(w), v.shape[0]))
        return w

    def loops(self):
        """(first loop, count) of this rank's loop slice (0, n_loops on a single-rank operator)."""
        a, b = ctypes.c_int64(), ctypes.c_int64()
        check(lib().xrl_operator_info(self.h, ctypes.byref(a), ctypes.byref(b), None, None))
        return int(a.value), int(b.value)

    def halo(self):
        """Exchange volume of one apply per right-hand side: (loop values, panel values) sent + received."""
        a, b = ctypes.c_int64(), ctypes.c_int64()
        check(lib().xrl_operator_info(self.h, None, None, ctypes.byref(a), ctypes.byref(b)))
        return int(a.value), int(b.value)

    def close(self):
        if getattr(self, "h", None):
            lib().xrl_operator_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Precond:
    """xrl_precond_build: block-Jacobi diagonal-of-P preconditioner (Eq. 10); exact=True:
    xrl_precond_build_exact, the whole Q factorised (sparse LU, NEXT f2); kind="diag_l": the
    diagonal-of-L baseline of PAPER.md:120-122 (xrl_precond_build_kind); ilu=True: ILU(0) of the whole Q
    on the GPU (cuSPARSE), no host factorisation."""

    KINDS = {"diag_p": 0, "diag_l": 1}

    def __init__(self, op: Operator, block_size: int = 64, exact: bool = False, kind: str = "diag_p",
                 ilu: bool = False):
        self.op = op
        h = ctypes.c_void_p()
        if ilu:  # ILU(0) of the whole Q on the GPU (xrl_precond_build_kind, block_size -2)
            check(lib().xrl_precond_build_kind(op.h, self.KINDS[kind], -2, ctypes.byref(h)))
        elif kind != "diag_p":
            check(lib().xrl_precond_build_kind(op.h, self.KINDS[kind], -1 if exact else block_size, ctypes.byref(h)))
        elif exact:
            check(lib().xrl_precond_build_exact(op.h, ctypes.byref(h)))
        else:
            check(lib().xrl_precond_build(op.h, block_size, ctypes.byref(h)))
        self.h = h

    def apply(self, v, z=None):
        import torch
        z = torch.empty_like(v) if z is None else z
        check(lib().xrl_precond_apply(self.h, _ptr(v), _ptr(z), v.shape[0]))
        return z

    def export(self):
        nb, bs = ctypes.c_int32(), ctypes.c_int32()
        check(lib().xrl_precond_export(self.h, ctypes.byref(nb), ctypes.byref(bs), None, None))
        ptr = np.empty(nb.value + 1, np.int32)
        inv = np.empty((nb.value, bs.value, bs.value), np.complex64)
        check(lib().xrl_precond_export(self.h, None, None, _ptr(ptr), _ptr(inv)))
        return ptr, inv

    def close(self):
        if getattr(self, "h", None):
            lib().xrl_precond_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gmres(op: Operator, pc, b, x=None, restart=50, max_iters=2000, tol=0.0, right=True):
    """xrl_gmres: returns (x, report dict).  tol <= 0 uses PAPER.md:152's rule; right=False selects
    the left-preconditioned form of Eq. 11 (reading R15)."""
    import torch
    x = torch.zeros_like(b) if x is None else x
    nrhs = b.shape[0]
    iters = np.zeros(nrhs, np.int32)
    rre = np.zeros(nrhs)
    trre = np.zeros(nrhs)
    conv = np.zeros(nrhs, np.int32)
    st = lib().xrl_gmres(op.h, pc.h if pc is not None else None, _ptr(b), _ptr(x), nrhs,
                         ctypes.byref(GmresOpts(restart, max_iters, tol, int(right))), _ptr(iters), _ptr(rre), _ptr(trre),
                         _ptr(conv))
    check(st)
    return x, {"iters": iters, "rre": rre, "true_rre": trre, "converged": conv.astype(bool), "status": st}


def operator_apply_vranks(ops, vs, ws=None):
    """xrl_operator_apply_vranks: the sharded loop-space operator of k virtual ranks; vs[r] rank r's slice."""
    import torch
    k = len(ops)
    ws = [torch.empty_like(v) for v in vs] if ws is None else ws
    oh = (ctypes.c_void_p * k)(*[o.h.value for o in ops])
    vp = (ctypes.c_void_p * k)(*[v.data_ptr() for v in vs])
    wp = (ctypes.c_void_p * k)(*[w.data_ptr() for w in ws])
    check(lib().xrl_operator_apply_vranks(k, oh, vp, wp, vs[0].shape[0]))
    return ws


def gmres_vranks(ops, pcs, bs, xs=None, restart=50, max_iters=2000, tol=0.0, right=True):
    """xrl_gmres_vranks: GMRES of k virtual ranks (slices bs[r], xs[r]); returns (xs, report)."""
    import torch
    k = len(ops)
    xs = [torch.zeros_like(b) for b in bs] if xs is None else xs
    nrhs = bs[0].shape[0]
    iters = np.zeros(nrhs, np.int32)
    rre = np.zeros(nrhs)
    trre = np.zeros(nrhs)
    conv = np.zeros(nrhs, np.int32)
    oh = (ctypes.c_void_p * k)(*[o.h.value for o in ops])
    ph = (ctypes.c_void_p * k)(*[p.h.value for p in pcs]) if pcs is not None else None
    bp = (ctypes.c_void_p * k)(*[b.data_ptr() for b in bs])
    xp = (ctypes.c_void_p * k)(*[x.data_ptr() for x in xs])
    st = lib().xrl_gmres_vranks(k, oh, ph, bp, xp, nrhs, ctypes.byref(GmresOpts(restart, max_iters, tol, int(right))),
                                _ptr(iters), _ptr(rre), _ptr(trre), _ptr(conv))
    check(st)
    return xs, {"iters": iters, "rre": rre, "true_rre": trre, "converged": conv.astype(bool), "status": st}


def extract(tree: Tree, near: Near, topo: Topology, freqs, zs=None, sigma=5.8e7, zeta=1e-4, block_size=64,
            restart=50, max_iters=2000, tol=0.0, right=True, exact=False):
    """xrl_extract: R/L sweep.  Returns dict with z [n_freq][P][P] complex, r, l [n_freq][P][P],
    iters, true_rre [n_freq][P] and the status (XRL_ENOCONV is reported, not raised).  exact=True uses
    the exact Q^-1 (xrl_precond_build_exact) instead of the block-Jacobi form."""
    if exact:
        block_size = -1
    freqs = np.ascontiguousarray(freqs, np.float64)
    nf, npt = freqs.size, topo.info()["n_ports"]
    z = np.zeros((nf, npt, npt, 2))
    r = np.zeros((nf, npt, npt))
    l_ = np.zeros((nf, npt, npt))
    it = np.zeros((nf, npt), np.int32)
    tr = np.zeros((nf, npt))
    zsa = None
    if zs is not None:
        zz = np.broadcast_to(np.asarray(zs, dtype=np.complex128), (tree.n,))
        zsa = np.ascontiguousarray(np.stack([zz.real, zz.imag], axis=1))
    st = lib().xrl_extract(tree.h, near.h, topo.h, _ptr(zsa) if zsa is not None else None, sigma, zeta, nf,
                           _ptr(freqs), block_size, ctypes.byref(GmresOpts(restart, max_iters, tol, int(right))), _ptr(z),
                           _ptr(r), _ptr(l_), _ptr(it), _ptr(tr))
    if st < 0:
        check(st)
    return {"freqs": freqs, "z": z[..., 0] + 1j * z[..., 1], "r": r, "l": l_, "iters": it, "true_rre": tr,
            "status": st}
