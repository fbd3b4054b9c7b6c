"""Seeded, synthetic input generators shared by the oracle tests, the GPU parity
tests and bench.py.

This module holds NONE of the method's arithmetic (no potentials, no FMM, no
near-field criterion): it only emits watertight triangle surface meshes (FP64
vertices in metres, int32 triangles) and the random complex source
coefficients.  Both the oracle (oracle/) and the CUDA path
(paper_2409_12375_b200/) consume these arrays; neither imports the other.

The paper's geometries (coils of Table II, BGA of Table III, HBPOP of Table V;
PAPER.md:160,190,217) are not published, so the five BASELINE.json configs are
procedural stand-ins with the shapes, sizes and density mix BASELINE.json names
(recipes: DESIGN.md "Inputs").
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

UM = 1e-6


@dataclass
class Mesh:
    """Triangle surface mesh.  verts: float64 [nv,3] (m); tris: int32 [nt,3],
    wound counter-clockwise seen from outside (outward normals)."""
    verts: np.ndarray
    tris: np.ndarray
    name: str = ""
    # conductor id per triangle (int32) and port terminal panel sets
    cond: np.ndarray | None = None
    ports: list = field(default_factory=list)  # [(name, plus_ids, minus_ids)]
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.tris.shape[0])


# ---------------------------------------------------------------------------
# low-level helpers
# ---------------------------------------------------------------------------

def _dedupe(points: np.ndarray, quantum: float):
    """Merge vertices that coincide on a grid of `quantum` metres."""
    key = np.round(points / quantum).astype(np.int64)
    _, first, inv = np.unique(key, axis=0, return_index=True, return_inverse=True)
    return points[first], inv.reshape(-1)


def _orient(verts, tris, want_normal):
    """Flip triangles whose winding normal disagrees with want_normal [nt,3]."""
    a, b, c = verts[tris[:, 0]], verts[tris[:, 1]], verts[tris[:, 2]]
    nrm = np.cross(b - a, c - a)
    flip = np.einsum("ij,ij->i", nrm, want_normal) < 0
    t = tris.copy()
    t[flip, 1], t[flip, 2] = tris[flip, 2], tris[flip, 1]
    return t


def quads_to_tris(q):
    """Split quads (a,b,c,d) on the fixed diagonal a-c."""
    q = np.asarray(q)
    return np.concatenate([q[:, [0, 1, 2]], q[:, [0, 2, 3]]], axis=0)


def voxel_surface(occ: np.ndarray, origin, h):
    """Boundary of a union of axis-aligned cells.

    occ: bool [nx,ny,nz]; origin: (3,) m; h: (3,) cell sizes in m.
    Returns (verts, tris) with outward winding; every boundary square is split
    on one fixed diagonal.  Shared grid nodes are merged exactly.
    """
    occ = np.asarray(occ, dtype=bool)
    nx, ny, nz = occ.shape
    pad = np.zeros((nx + 2, ny + 2, nz + 2), dtype=bool)
    pad[1:-1, 1:-1, 1:-1] = occ
    quads, normals = [], []
    # node id of grid node (i,j,k), 0<=i<=nx ...
    def nid(i, j, k):
        return (i * (ny + 1) + j) * (nz + 1) + k

    for axis in range(3):
        for sgn in (+1, -1):
            sh = [0, 0, 0]
            sh[axis] = sgn
            nb = np.roll(pad, shift=-sgn, axis=axis)[1:-1, 1:-1, 1:-1]
            face = occ & ~nb
            i, j, k = np.nonzero(face)
            if i.size == 0:
                continue
            base = [i, j, k]
            base[axis] = base[axis] + (1 if sgn > 0 else 0)
            u, v = [a for a in range(3) if a != axis]
            c0 = list(base)
            c1 = list(base); c1[u] = c1[u] + 1
            c2 = list(base); c2[u] = c2[u] + 1; c2[v] = c2[v] + 1
            c3 = list(base); c3[v] = c3[v] + 1
            q = np.stack([nid(*c0), nid(*c1), nid(*c2), nid(*c3)], axis=1)
            quads.append(q)
            nrm = np.zeros((q.shape[0], 3))
            nrm[:, axis] = sgn
            normals.append(nrm)
    quads = np.concatenate(quads, axis=0)
    normals = np.concatenate(normals, axis=0)
    used, inv = np.unique(quads.reshape(-1), return_inverse=True)
    quads = inv.reshape(-1, 4)
    kk = used % (nz + 1)
    jj = (used // (nz + 1)) % (ny + 1)
    ii = used // ((nz + 1) * (ny + 1))
    verts = np.stack([origin[0] + ii * h[0], origin[1] + jj * h[1], origin[2] + kk * h[2]], axis=1)
    tris = quads_to_tris(quads)
    tris = _orient(verts, tris, np.concatenate([normals, normals], axis=0))
    return verts.astype(np.float64), tris.astype(np.int32)


def voxel_quads(occ: np.ndarray, origin, h):
    """As voxel_surface, but the boundary squares stay rectangles: (verts, quads [n,4], normals [n,3]),
    each quad (a, b, c, d) in cyclic order with (b-a) x (d-a) along the outward normal."""
    occ = np.asarray(occ, dtype=bool)
    nx, ny, nz = occ.shape
    pad = np.zeros((nx + 2, ny + 2, nz + 2), dtype=bool)
    pad[1:-1, 1:-1, 1:-1] = occ

    def nid(i, j, k):
        return (i * (ny + 1) + j) * (nz + 1) + k

    quads, normals = [], []
    for axis in range(3):
        for sgn in (+1, -1):
            nb = np.roll(pad, shift=-sgn, axis=axis)[1:-1, 1:-1, 1:-1]
            i, j, k = np.nonzero(occ & ~nb)
            if i.size == 0:
                continue
            base = [i, j, k]
            base[axis] = base[axis] + (1 if sgn > 0 else 0)
            u, v = [a for a in range(3) if a != axis]
            c1 = list(base); c1[u] = c1[u] + 1
            c2 = list(base); c2[u] = c2[u] + 1; c2[v] = c2[v] + 1
            c3 = list(base); c3[v] = c3[v] + 1
            quads.append(np.stack([nid(*base), nid(*c1), nid(*c2), nid(*c3)], axis=1))
            nrm = np.zeros((i.size, 3))
            nrm[:, axis] = sgn
            normals.append(nrm)
    quads = np.concatenate(quads, axis=0)
    normals = np.concatenate(normals, axis=0)
    used, inv = np.unique(quads.reshape(-1), return_inverse=True)
    quads = inv.reshape(-1, 4)
    kk = used % (nz + 1)
    jj = (used // (nz + 1)) % (ny + 1)
    ii = used // ((nz + 1) * (ny + 1))
    verts = np.stack([origin[0] + ii * h[0], origin[1] + jj * h[1], origin[2] + kk * h[2]], axis=1)
    a, b, d = verts[quads[:, 0]], verts[quads[:, 1]], verts[quads[:, 3]]
    flip = np.einsum("ij,ij->i", np.cross(b - a, d - a), normals) < 0
    quads[flip] = quads[flip][:, [0, 3, 2, 1]]
    return verts.astype(np.float64), quads.astype(np.int32), normals


def bar_hybrid(length=1000 * UM, side=100 * UM, cell=20 * UM) -> Mesh:
    """Config 1 geometry as a hybrid mesh (NEXT f4): the four long faces keep their
    `cell` squares as rectangle panels, the two end caps are split into triangles.  panels int32 [n][4]
    (-1 in the last column for triangles); N = 4 (L/c)(s/c) + 4 (s/c)^2 = 1,100 at the defaults."""
    nx, ny = int(round(length / cell)), int(round(side / cell))
    occ = np.ones((nx, ny, ny), dtype=bool)
    v, q, nrm = voxel_quads(occ, (0.0, 0.0, 0.0), (cell, cell, cell))
    cap = np.abs(nrm[:, 0]) > 0.5
    tri = np.concatenate([q[cap][:, [0, 1, 2]], q[cap][:, [0, 2, 3]]], axis=0)  # same winding as the quad
    panels = np.concatenate([q[~cap], np.concatenate([tri, np.full((tri.shape[0], 1), -1)], axis=1)])
    panels = panels.astype(np.int32)
    cen = np.array([v[p[p >= 0]].mean(axis=0) for p in panels])
    minus = np.nonzero(np.isclose(cen[:, 0], 0.0, atol=1e-3 * cell))[0]
    plus = np.nonzero(np.isclose(cen[:, 0], length, atol=1e-3 * cell))[0]
    return Mesh(v, panels, "bar_hybrid", np.zeros(panels.shape[0], np.int32),
                [("P1", plus.astype(np.int32), minus.astype(np.int32))],
                {"length": length, "side": side, "cell": cell, "rectangles": int((~cap).sum()),
                 "triangles": int(tri.shape[0])})


def merge(parts):
    """Concatenate (verts, tris, cond) parts without merging vertices."""
    vs, ts, cs = [], [], []
    off = 0
    for ci, (v, t) in enumerate(parts):
        vs.append(v)
        ts.append(t + off)
        cs.append(np.full(t.shape[0], ci, dtype=np.int32))
        off += v.shape[0]
    return np.concatenate(vs), np.concatenate(ts).astype(np.int32), np.concatenate(cs)


# ---------------------------------------------------------------------------
# configs
# ---------------------------------------------------------------------------

def bar(length=1000 * UM, side=100 * UM, cell=20 * UM) -> Mesh:
    """Config 1: straight bar [0,L]x[0,s]x[0,s], structured squares of `cell`,
    each split on one fixed diagonal.  N = 2*(4*(L/c)*(s/c) + 2*(s/c)^2)."""
    nx, ny = int(round(length / cell)), int(round(side / cell))
    occ = np.ones((nx, ny, ny), dtype=bool)
    v, t = voxel_surface(occ, (0.0, 0.0, 0.0), (cell, cell, cell))
    cen = v[t].mean(axis=1)
    minus = np.nonzero(np.isclose(cen[:, 0], 0.0, atol=1e-3 * cell))[0]
    plus = np.nonzero(np.isclose(cen[:, 0], length, atol=1e-3 * cell))[0]
    return Mesh(v, t, "bar", np.zeros(t.shape[0], np.int32),
                [("P1", plus.astype(np.int32), minus.astype(np.int32))],
                {"length": length, "side": side, "cell": cell})


def _spiral_cells(n_side, width, pitch, turns):
    """Occupancy [n_side,n_side] of a square spiral (cell units) plus the two
    free-end cell boxes (outer start, inner end)."""
    occ = np.zeros((n_side, n_side), dtype=bool)
    for t in range(turns):
        o = pitch * t
        x0 = max(o - pitch, 0)
        occ[x0:n_side - o, o:o + width] = True                      # bottom, +x
        occ[n_side - o - width:n_side - o, o:n_side - o] = True     # right, +y
        occ[o:n_side - o, n_side - o - width:n_side - o] = True     # top, -x
        occ[o:o + width, o + pitch:n_side - o] = True               # left, -y
    o_last = pitch * (turns - 1)
    start = (0, 0, width)                       # x==0 face, y in [0,width)
    end = (o_last, o_last + pitch, width)       # y==o_last+pitch face, x in [o,o+w)
    return occ, start, end


def coils(outer=1000 * UM, width=20 * UM, thick=5 * UM, pitch=40 * UM, turns=5,
          gap_z=100 * UM, cell=5 * UM) -> Mesh:
    """Config 2: two parallel square spirals (5 turns, outer side 1 mm, trace
    20 um x 5 um, pitch 40 um) stacked with a 100 um vertical gap, meshed on a
    5 um structured grid (squares split in two)."""
    n_side = int(round(outer / cell))
    w, p = int(round(width / cell)), int(round(pitch / cell))
    nt = int(round(thick / cell))
    occ2, start, end = _spiral_cells(n_side, w, p, turns)
    parts, ports = [], []
    off_t = 0
    for ci in range(2):
        z0 = ci * (thick + gap_z)
        occ = np.repeat(occ2[:, :, None], nt, axis=2)
        v, t = voxel_surface(occ, (0.0, 0.0, z0), (cell, cell, cell))
        cen = v[t].mean(axis=1)
        # terminals: outer start face x==0 ; inner end face y == (o+pitch)*cell
        tol = 1e-3 * cell
        s_ids = np.nonzero(np.isclose(cen[:, 0], 0.0, atol=tol) & (cen[:, 1] < w * cell))[0]
        ex0, ey, ewid = end
        e_ids = np.nonzero(np.isclose(cen[:, 1], ey * cell, atol=tol)
                           & (cen[:, 0] > ex0 * cell) & (cen[:, 0] < (ex0 + ewid) * cell)
                           & (np.abs(v[t][:, :, 1] - ey * cell).max(axis=1) < tol))[0]
        parts.append((v, t))
        ports.append((f"coil{ci + 1}", (s_ids + off_t).astype(np.int32), (e_ids + off_t).astype(np.int32)))
        off_t += t.shape[0]
    V, T, C = merge(parts)
    return Mesh(V, T, "coils", C, ports, {"cell": cell})


def icosphere(level=3, radius=1.0):
    """Subdivided icosahedron: 20*4^level triangles, outward winding."""
    ph = (1 + 5 ** 0.5) / 2
    v = np.array([[-1, ph, 0], [1, ph, 0], [-1, -ph, 0], [1, -ph, 0],
                  [0, -1, ph], [0, 1, ph], [0, -1, -ph], [0, 1, -ph],
                  [ph, 0, -1], [ph, 0, 1], [-ph, 0, -1], [-ph, 0, 1]], dtype=np.float64)
    f = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
                  [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
                  [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
                  [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], dtype=np.int64)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    for _ in range(level):
        edges = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]])
        edges = np.sort(edges, axis=1)
        ue, inv = np.unique(edges, axis=0, return_inverse=True)
        inv = inv.reshape(-1)
        mid = v[ue[:, 0]] + v[ue[:, 1]]
        mid /= np.linalg.norm(mid, axis=1, keepdims=True)
        m = inv.reshape(3, -1).T + v.shape[0]  # ab, bc, ca
        v = np.concatenate([v, mid])
        a, b, c = f[:, 0], f[:, 1], f[:, 2]
        ab, bc, ca = m[:, 0], m[:, 1], m[:, 2]
        f = np.concatenate([np.stack([a, ab, ca], 1), np.stack([b, bc, ab], 1),
                            np.stack([c, ca, bc], 1), np.stack([ab, bc, ca], 1)])
    t = _orient(v, f.astype(np.int32), v[f].mean(axis=1))
    return v * radius, t


def perforated_plane(nbx, nby, pitch, hole_r, z0, z1, nseg=16, nring=5):
    """Rectangular plate [0,nbx*pitch]x[0,nby*pitch]x[z0,z1] with one circular
    hole (radius hole_r, nseg-gon) centred in every pitch x pitch cell.  Per
    cell and face: nseg x nring quads from the circle to the cell square; hole
    wall nseg quads; outer rim quads along the plate edge."""
    assert nseg % 4 == 0
    q = nseg // 4
    # square boundary points (counter-clockwise from (+1,-1) corner region),
    # q per side, starting at angle -45 deg corner
    sq = []
    for side in range(4):
        for i in range(q):
            s = -1 + 2 * i / q
            if side == 0:
                sq.append((1.0, s))
            elif side == 1:
                sq.append((-s, 1.0))
            elif side == 2:
                sq.append((-1.0, -s))
            else:
                sq.append((s, -1.0))
    sq = np.array(sq) * 0.5  # unit cell half-width 0.5
    ang = np.arctan2(sq[:, 1], sq[:, 0])
    circ = np.stack([np.cos(ang), np.sin(ang)], 1) * (hole_r / pitch)
    # ring points: r=0..nring, 0 = circle, nring = square
    rings = np.stack([circ + (sq - circ) * (r / nring) for r in range(nring + 1)])  # [nring+1,nseg,2]
    pts, quads, nrm = [], [], []
    npc = (nring + 1) * nseg
    idx = 0
    for bx in range(nbx):
        for by in range(nby):
            cx, cy = (bx + 0.5) * pitch, (by + 0.5) * pitch
            for zf, sgn in ((z1, +1), (z0, -1)):
                p = np.concatenate([(rings.reshape(-1, 2) * pitch + [cx, cy]),
                                    np.full((npc, 1), zf)], axis=1)
                pts.append(p)
                for r in range(nring):
                    for s in range(nseg):
                        s1 = (s + 1) % nseg
                        a = idx + r * nseg + s
                        b = idx + r * nseg + s1
                        c = idx + (r + 1) * nseg + s1
                        d = idx + (r + 1) * nseg + s
                        quads.append((a, b, c, d))
                        nrm.append((0, 0, sgn))
                idx += npc
            # hole wall: circle at z1 (ring 0 of first face) to circle at z0
            top0 = idx - 2 * npc
            bot0 = idx - npc
            for s in range(nseg):
                s1 = (s + 1) % nseg
                quads.append((top0 + s, top0 + s1, bot0 + s1, bot0 + s))
                ang_m = 0.5 * (ang[s] + ang[s1] + (2 * np.pi if ang[s1] < ang[s] else 0))
                nrm.append((-np.cos(ang_m), -np.sin(ang_m), 0))
    pts = np.concatenate(pts)
    # outer rim: plate boundary split into q segments per cell edge
    X, Y = nbx * pitch, nby * pitch
    rim = []
    def seg_list(L, n):
        return np.linspace(0, L, n + 1)
    for (p0, p1, nn) in (((0, 0), (X, 0), (0, -1)), ((X, 0), (X, Y), (1, 0)),
                         ((X, Y), (0, Y), (0, 1)), ((0, Y), (0, 0), (-1, 0))):
        L = np.hypot(p1[0] - p0[0], p1[1] - p0[1])
        ncell = int(round(L / pitch)) * q
        tt = seg_list(1.0, ncell)
        for i in range(ncell):
            a = np.array(p0) + (np.array(p1) - np.array(p0)) * tt[i]
            b = np.array(p0) + (np.array(p1) - np.array(p0)) * tt[i + 1]
            base = len(pts) + len(rim)
            rim.extend([(a[0], a[1], z0), (b[0], b[1], z0), (b[0], b[1], z1), (a[0], a[1], z1)])
            quads.append((base, base + 1, base + 2, base + 3))
            nrm.append((nn[0], nn[1], 0))
    pts = np.concatenate([pts, np.array(rim)])
    quads = np.array(quads, dtype=np.int64)
    nrm = np.array(nrm, dtype=np.float64)
    v, inv = _dedupe(pts, quantum=pitch * 1e-7)
    quads = inv[quads]
    t = quads_to_tris(quads)
    t = _orient(v, t.astype(np.int32), np.concatenate([nrm, nrm]))
    return v, t


def bga(nb=16, pitch=500 * UM, ball_r=150 * UM, hole_r=100 * UM, level=3,
        plane_z=(160 * UM, 180 * UM)) -> Mesh:
    """Configs 3/5: nb x nb icosphere balls (level 3 = 1280 triangles, r=150um,
    500um pitch) centred on z=0 between two plates (20um thick, z in
    [160,180]um and [-180,-160]um) with a coaxial 200um-diameter hole per ball."""
    sv, st = icosphere(level, ball_r)
    parts = []
    for bx in range(nb):
        for by in range(nb):
            parts.append((sv + [(bx + 0.5) * pitch, (by + 0.5) * pitch, 0.0], st))
    z0, z1 = plane_z
    parts.append(perforated_plane(nb, nb, pitch, hole_r, z0, z1))
    parts.append(perforated_plane(nb, nb, pitch, hole_r, -z1, -z0))
    V, T, C = merge(parts)
    return Mesh(V, T, f"bga{nb}", C, [], {"nb": nb})


def _fill_diagonal_contacts(occ: np.ndarray):
    """Cells touching only along an edge (2x2 blocks [[1,0],[0,1]] or
    [[0,1],[1,0]]) make a non-manifold surface; fill the lower-left free cell
    of every such block (repeat until none remain)."""
    while True:
        a, b = occ[:-1, :-1], occ[1:, 1:]
        c, d = occ[1:, :-1], occ[:-1, 1:]
        p1 = a & b & ~c & ~d
        p2 = c & d & ~a & ~b
        if not (p1.any() or p2.any()):
            return
        i, j = np.nonzero(p1)
        occ[i + 1, j] = True
        i, j = np.nonzero(p2)
        occ[i, j] = True


def pop(seed=4242, via_seed=4243, n_traces=2000, n_vias=5000, domain=10e-3,
        len_lo=0.2e-3, len_hi=0.8e-3) -> Mesh:
    """Config 4: package-on-package-like stack.  Two solid ground planes
    (10x10 mm, 10 um thick, 100 um structured grid) at z in [-110,-100] and
    [400,410] um; 4 trace layers (z = 0,100,200,300 um) holding n_traces/4
    seeded Manhattan traces each (20 um wide x 10 um thick, 2-4 axis-aligned
    segments of U[len_lo,len_hi], 20 um panels); n_vias seeded cylinders
    (r = 50 um, 16-gon, one 100 um layer gap, 25 um axial panels, capped)."""
    rng = np.random.default_rng(seed)
    parts = []
    # ground planes
    gp = 100 * UM
    ng = int(round(domain / gp))
    for z in (-110 * UM, 400 * UM):
        occ = np.ones((ng, ng, 1), dtype=bool)
        parts.append(voxel_surface(occ, (0.0, 0.0, z), (gp, gp, 10 * UM)))
    # traces, one occupancy grid per layer
    tc = 20 * UM
    nc = int(round(domain / tc))
    for layer in range(4):
        occ = np.zeros((nc, nc), dtype=bool)
        for _ in range(n_traces // 4):
            x, y = rng.integers(0, nc, size=2)
            nseg = rng.integers(2, 5)
            axis = rng.integers(0, 2)
            for _s in range(nseg):
                L = int(round(rng.uniform(len_lo, len_hi) / tc))
                d = 1 if rng.random() < 0.5 else -1
                if axis == 0:
                    x1 = int(np.clip(x + d * L, 0, nc - 1))
                    lo, hi = min(x, x1), max(x, x1)
                    occ[lo:hi + 1, y] = True
                    x = x1
                else:
                    y1 = int(np.clip(y + d * L, 0, nc - 1))
                    lo, hi = min(y, y1), max(y, y1)
                    occ[x, lo:hi + 1] = True
                    y = y1
                axis ^= 1
        _fill_diagonal_contacts(occ)
        parts.append(voxel_surface(occ[:, :, None], (0.0, 0.0, layer * 100 * UM), (tc, tc, 10 * UM)))
    # vias
    vr = np.random.default_rng(via_seed)
    nseg, nax, r = 16, 4, 50 * UM
    th = 2 * np.pi * np.arange(nseg) / nseg
    ring = np.stack([np.cos(th), np.sin(th)], 1) * r
    for _ in range(n_vias):
        cx, cy = vr.uniform(r, domain - r, size=2)
        g = vr.integers(0, 3)
        z0 = g * 100 * UM + 10 * UM
        zs = z0 + np.arange(nax + 1) * (100 * UM - 10 * UM) / nax
        pts = [np.concatenate([ring + [cx, cy], np.full((nseg, 1), z)], 1) for z in zs]
        pts = np.concatenate(pts + [np.array([[cx, cy, zs[0]], [cx, cy, zs[-1]]])])
        q, nrm = [], []
        for a in range(nax):
            for s in range(nseg):
                s1 = (s + 1) % nseg
                q.append((a * nseg + s, a * nseg + s1, (a + 1) * nseg + s1, (a + 1) * nseg + s))
        q = np.array(q)
        tri = quads_to_tris(q)
        mid = 0.5 * (th + np.roll(th, -1) + np.where(np.arange(nseg) == nseg - 1, 2 * np.pi, 0))
        nq = np.tile(np.stack([np.cos(mid), np.sin(mid), np.zeros(nseg)], 1), (nax, 1))
        nrm = np.concatenate([nq, nq])
        cb, ct = (nax + 1) * nseg, (nax + 1) * nseg + 1
        capb = np.stack([np.full(nseg, cb), np.arange(nseg), (np.arange(nseg) + 1) % nseg], 1)
        capt = np.stack([np.full(nseg, ct), nax * nseg + np.arange(nseg), nax * nseg + (np.arange(nseg) + 1) % nseg], 1)
        tri = np.concatenate([tri, capb, capt])
        nrm = np.concatenate([nrm, np.tile([0, 0, -1.0], (nseg, 1)), np.tile([0, 0, 1.0], (nseg, 1))])
        parts.append((pts, _orient(pts, tri.astype(np.int32), nrm)))
    V, T, C = merge(parts)
    return Mesh(V, T, "pop", C, [], {})


CONFIGS = {1: "bar", 2: "coils", 3: "bga16", 4: "pop", 5: "bga64"}


def make_config(cfg: int, **kw) -> Mesh:
    """BASELINE.json configs[cfg-1]."""
    if cfg == 1:
        return bar(**kw)
    if cfg == 2:
        return coils(**kw)
    if cfg == 3:
        return bga(nb=16, **kw)
    if cfg == 4:
        return pop(**kw)
    if cfg == 5:
        return bga(nb=64, **kw)
    raise ValueError(cfg)


def make_x(cfg: int, n: int, nvec: int = 3) -> np.ndarray:
    """Source coefficients: complex64 [nvec][n], re and im i.i.d. U[-1,1] from
    seed 1000+cfg, in the mesh's original triangle order."""
    rng = np.random.default_rng(1000 + cfg)
    a = rng.random((nvec, n, 2), dtype=np.float64) * 2.0 - 1.0
    return (a[..., 0] + 1j * a[..., 1]).astype(np.complex64)


def small_mesh(kind: str = "cube", **kw) -> Mesh:
    """Tiny meshes for brute-force pins."""
    if kind == "cube":
        n = kw.get("n", 2)
        s = kw.get("side", 1.0)
        occ = np.ones((1, 1, 1), dtype=bool)
        v, t = voxel_surface(np.ones((n, n, n), bool), (0, 0, 0), (s / n,) * 3)
        return Mesh(v, t, "cube")
    if kind == "random":
        rng = np.random.default_rng(kw.get("seed", 0))
        m = kw.get("n", 20)
        v = rng.random((3 * m, 3)) * kw.get("scale", 1.0)
        t = np.arange(3 * m, dtype=np.int32).reshape(m, 3)
        return Mesh(v, t, "random")
    raise ValueError(kind)
