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
    "xrl_tree_build", "xrl_tree_destroy", "xrl_tree_info", "xrl_tree_perm", "xrl_to_library_order",
    "xrl_from_library_order", "xrl_tree_export", "xrl_near_assemble", "xrl_near_destroy",
    "xrl_near_export", "xrl_mvm", "xrl_mvm_host", "xrl_timing_enable", "xrl_timing_count",
    "xrl_timing_name", "xrl_timing_get", "xrl_timing_reset", "xrl_launch_count",
]


class XrlError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class FmmOpts(ctypes.Structure):
    _fields_ = [("p", ctypes.c_int32), ("leaf_max", ctypes.c_int32), ("max_depth", ctypes.c_int32)]


class NearOpts(ctypes.Structure):
    _fields_ = [("eta", ctypes.c_double)]


class TreeInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("n_local", ctypes.c_int64), ("offset", ctypes.c_int64),
                ("n_boxes", ctypes.c_int32), ("n_leaves", ctypes.c_int32), ("n_levels", ctypes.c_int32),
                ("p", ctypes.c_int32), ("n_v_pairs", ctypes.c_int64), ("n_x_pairs", ctypes.c_int64),
                ("n_w_pairs", ctypes.c_int64), ("n_u_pairs", ctypes.c_int64), ("n_p2p", ctypes.c_int64),
                ("root_lo", ctypes.c_double * 3), ("root_width", ctypes.c_double)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["root_lo"] = list(self.root_lo)
        return d


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
        L.xrl_mvm.argtypes = [P, P, P, P, i32, u32]
        L.xrl_mvm_host.argtypes = [P, P, P, P, i32, u32]
        L.xrl_timing_enable.argtypes = [P, ctypes.c_int]
        L.xrl_timing_count.restype = i32
        L.xrl_timing_name.argtypes = [i32]
        L.xrl_timing_name.restype = ctypes.c_char_p
        L.xrl_timing_get.argtypes = [P, P, P]
        L.xrl_timing_reset.argtypes = [P]
        L.xrl_launch_count.argtypes = [P]
        L.xrl_launch_count.restype = i64
        for name in ("xrl_ctx_create", "xrl_ctx_sync", "xrl_tree_build", "xrl_tree_info", "xrl_tree_perm",
                     "xrl_to_library_order", "xrl_from_library_order", "xrl_tree_export", "xrl_near_assemble",
                     "xrl_near_export", "xrl_mvm", "xrl_mvm_host", "xrl_timing_enable", "xrl_timing_get",
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


class Context:
    """xrl_ctx_create on `device`, running on torch's current stream (or `stream`)."""

    def __init__(self, device: int = 0, stream=None):
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.device = device
        self.stream = stream
        h = ctypes.c_void_p()
        check(lib().xrl_ctx_create(device, ctypes.c_void_p(stream.cuda_stream), 0, 1, None, ctypes.byref(h)))
        self.h = h

    def sync(self):
        check(lib().xrl_ctx_sync(self.h))

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


class Tree:
    """xrl_tree_build over a triangle mesh (host FP64 verts [nv,3], int32 tris [n,3])."""

    def __init__(self, ctx: Context, verts, tris, p=10, leaf_max=64, max_depth=21):
        self.ctx = ctx
        v = np.ascontiguousarray(verts, dtype=np.float64)
        t = np.ascontiguousarray(tris, dtype=np.int32)
        opts = FmmOpts(p, leaf_max, max_depth)
        h = ctypes.c_void_p()
        check(lib().xrl_tree_build(ctx.h, v.shape[0], _ptr(v), t.shape[0], _ptr(t), ctypes.byref(opts),
                                   ctypes.byref(h)))
        self.h = h
        self.n = t.shape[0]

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

    def __init__(self, tree: Tree, eta=1.5):
        self.tree = tree
        h = ctypes.c_void_p()
        check(lib().xrl_near_assemble(tree.h, ctypes.byref(NearOpts(eta)), ctypes.byref(h)))
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
    """y = P x on the device (library order, complex64 [nvec][n])."""
    import torch
    _dev_vec(x, tree.n, "x")
    y = torch.empty_like(x) if y is None else _dev_vec(y, tree.n, "y")
    check(lib().xrl_mvm(tree.h, near.h, _ptr(x), _ptr(y), x.shape[0], flags))
    return y


def mvm_host(tree: Tree, near: Near, x_host: np.ndarray, y_host: np.ndarray | None = None, flags=XRL_MVM_FULL):
    """End-to-end y = P x with host complex64 [nvec][n] buffers in mesh order."""
    x_host = np.ascontiguousarray(x_host, dtype=np.complex64)
    if y_host is None:
        y_host = np.empty_like(x_host)
    check(lib().xrl_mvm_host(tree.h, near.h, _ptr(x_host), _ptr(y_host), x_host.shape[0], flags))
    return y_host
