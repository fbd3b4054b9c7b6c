"""XRL oracle -- TEST INFRASTRUCTURE ONLY (see xrl_oracle.c header).

Plain CPU FP64 implementation of the discrete operator the hot path applies.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  It shares no code with
paper_2409_12375_b200 and never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "xrl_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")

ETA = 1.5  # near criterion factor, reading R3

_lib = None


def _stale() -> bool:
    return not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC)


def build(force: bool = False) -> str:
    """Compile the oracle with gcc: FP64, -ffp-contract=off, OpenMP.

    Safe under concurrent callers (e.g. the spawned ranks of the gloo tests):
    an exclusive file lock serialises the compilers, each writes its own
    per-process temporary and the rename into place is atomic."""
    if not (force or _stale()):
        return _SO
    import fcntl
    with open(_SO + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        try:
            if force or _stale():  # another process may have built it while we waited
                tmp = "%s.%d.tmp" % (_SO, os.getpid())
                cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
                       "-std=c11", "-o", tmp, _SRC, "-lm"]
                subprocess.check_call(cmd)
                os.replace(tmp, _SO)
        finally:
            fcntl.flock(lk, fcntl.LOCK_UN)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        i64, i32, f64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        L.orc_geometry.argtypes = [i64, P, P, i32, P, P, P]
        L.orc_tri_potential.argtypes = [P, P, P, P]
        L.orc_tri_potential.restype = f64
        L.orc_p_entries.argtypes = [i64, P, P, i32, P, P, P, f64, i32, i64, P, i64, P, P]
        L.orc_mvm_rows.argtypes = [i64, P, P, i32, P, P, P, f64, i32, i32, P, i64, P, P, i32]
        L.orc_near_rows.argtypes = [i64, P, P, i32, P, P, P, f64, i32, i64, P, P, P, P, P, P]
        L.orc_panel_potential_ext.argtypes = [P, P, P, i32, i64]
        L.orc_panel_potential_ext.restype = f64
        L.orc_outer_rule_ext.argtypes = [P, P, i32, i64, P, P]
        L.orc_outer_rule_ext.restype = ctypes.c_int
        L.orc_tie_audit.argtypes = [i64, P, P, f64, f64]
        L.orc_tie_audit.restype = i64
        L.orc_tie_audit_rows.argtypes = [i64, P, P, f64, f64, i64, P]
        L.orc_tie_audit_rows.restype = i64
        L.orc_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class Geometry:
    """FP64 per-panel data (centroid, area, diameter D) of a triangle or hybrid triangle/rectangle mesh.
    panels: int32 [n][3] triangles, or [n][4] with -1 in the last column for triangles and a planar
    parallelogram (a, b, c, d in cyclic order) otherwise.  galerkin: the near rule of SPEC.md:345
    (outer quadrature on self and vertex-adjacent pairs) instead of centroid collocation."""

    def __init__(self, verts, tris, galerkin=False):
        self.verts = np.ascontiguousarray(verts, dtype=np.float64)
        self.tris = np.ascontiguousarray(tris, dtype=np.int32)
        n = self.tris.shape[0]
        self.n = n
        self.stride = self.tris.shape[1]
        assert self.stride in (3, 4)
        self.galerkin = int(bool(galerkin))
        self.cent = np.empty((n, 3))
        self.area = np.empty(n)
        self.dmax = np.empty(n)
        lib().orc_geometry(n, _p(self.verts), _p(self.tris), self.stride, _p(self.cent), _p(self.area),
                           _p(self.dmax))


def tri_potential(r, v0, v1, v2) -> float:
    """I(r;T) = int_T dS'/|r-r'| (closed form, FP64)."""
    a = [np.ascontiguousarray(x, dtype=np.float64) for x in (r, v0, v1, v2)]
    return lib().orc_tri_potential(*[_p(x) for x in a])


def panel_potential(r, g: Geometry, k: int) -> float:
    """I(r; S_k) for panel k of g (triangle, or rectangle as its two diagonal triangles)."""
    r = np.ascontiguousarray(r, dtype=np.float64)
    return lib().orc_panel_potential_ext(_p(r), _p(g.verts), _p(g.tris), g.stride, int(k))


def outer_rule(g: Geometry, k: int):
    """The Galerkin outer quadrature of panel k: points [m,3], weights [m] (sum 1)."""
    x = np.empty((7, 3))
    w = np.empty(7)
    m = lib().orc_outer_rule_ext(_p(g.verts), _p(g.tris), g.stride, int(k), _p(x), _p(w))
    return x[:m], w[:m]


def p_entries(g: Geometry, rows, cols, eta=ETA):
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    out = np.empty((rows.size, cols.size))
    lib().orc_p_entries(g.n, _p(g.verts), _p(g.tris), g.stride, _p(g.cent), _p(g.area), _p(g.dmax), eta,
                        g.galerkin, rows.size, _p(rows), cols.size, _p(cols), _p(out))
    return out


def dense_p(g: Geometry, eta=ETA):
    idx = np.arange(g.n, dtype=np.int64)
    return p_entries(g, idx, idx, eta)


def mvm_rows(g: Geometry, x, rows=None, eta=ETA, nthreads=0):
    """y[:, i] = sum_l P[rows[i], l] x[:, l] in FP64.  x: complex [nvec][N]
    (any precision; upcast exactly).  Returns complex128 [nvec][len(rows)]."""
    x = np.asarray(x)
    nvec = x.shape[0]
    xd = np.ascontiguousarray(x.astype(np.complex128)).view(np.float64)
    if rows is None:
        rows = np.arange(g.n, dtype=np.int64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    y = np.empty((nvec, rows.size), dtype=np.complex128)
    lib().orc_mvm_rows(g.n, _p(g.verts), _p(g.tris), g.stride, _p(g.cent), _p(g.area), _p(g.dmax), eta,
                       g.galerkin, nvec, _p(xd), rows.size, _p(rows), _p(y.view(np.float64)), int(nthreads))
    return y


def near_rows(g: Geometry, rows=None, eta=ETA):
    """Near-field rows in CSR form: (ptr, cols, vals, inv_r) where vals are the
    near entries P_kl (self term on the diagonal) and inv_r = 1/|c_k-c_l|
    (0 on the diagonal), columns ascending in the mesh's own panel order."""
    if rows is None:
        rows = np.arange(g.n, dtype=np.int64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    L = lib()
    cnt = np.empty(rows.size, dtype=np.int64)
    L.orc_near_rows(g.n, _p(g.verts), _p(g.tris), g.stride, _p(g.cent), _p(g.area), _p(g.dmax), eta,
                    g.galerkin, rows.size, _p(rows), _p(cnt), None, None, None, None)
    ptr = np.zeros(rows.size + 1, dtype=np.int64)
    np.cumsum(cnt, out=ptr[1:])
    cols = np.empty(ptr[-1], dtype=np.int64)
    vals = np.empty(ptr[-1])
    inv_r = np.empty(ptr[-1])
    L.orc_near_rows(g.n, _p(g.verts), _p(g.tris), g.stride, _p(g.cent), _p(g.area), _p(g.dmax), eta,
                    g.galerkin, rows.size, _p(rows), _p(cnt), _p(ptr), _p(cols), _p(vals), _p(inv_r))
    return ptr, cols, vals, inv_r


def tie_audit(g: Geometry, eta=ETA, rel=1e-9) -> int:
    return int(lib().orc_tie_audit(g.n, _p(g.cent), _p(g.dmax), eta, rel))


def tie_audit_rows(g: Geometry, rows, eta=ETA, rel=1e-9) -> int:
    """Tie audit of the selected target rows against every source panel."""
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    return int(lib().orc_tie_audit_rows(g.n, _p(g.cent), _p(g.dmax), eta, rel, rows.size, _p(rows)))


def num_threads() -> int:
    return int(lib().orc_num_threads())


def rel_l2(y, yref) -> float:
    """Parity metric: ||y - yref||_2 / ||yref||_2 over all components jointly
    (same form as PAPER.md:150 Eq. 12)."""
    y = np.asarray(y, dtype=np.complex128)
    yref = np.asarray(yref, dtype=np.complex128)
    return float(np.linalg.norm(y - yref) / np.linalg.norm(yref))
