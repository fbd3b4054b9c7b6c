"""Pins of the oracle (oracle/) against things other than itself: closed forms,
an independent polar quadrature (tests/quadrature.py), additivity, isometry
invariance, the point-charge far-field limit, exact symmetry and brute force
on tiny meshes.  CPU only."""
import os

import numpy as np
import pytest

import oracle
from inputs import meshes
from tests.quadrature import tri_potential_quad

GOLD = os.path.join(os.path.dirname(__file__), "golden", "closed_forms.txt")


def golden():
    out = {}
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        k, v = line.split()
        out[k] = float(v)
    return out


def test_closed_form_equilateral():
    g = golden()
    v0, v1, v2 = np.array([0, 0, 0.]), np.array([1, 0, 0.]), np.array([0.5, np.sqrt(3) / 2, 0])
    c = (v0 + v1 + v2) / 3
    A = np.sqrt(3) / 4
    assert oracle.tri_potential(c, v0, v1, v2) / A == pytest.approx(g["equilateral_centroid"], rel=1e-14)
    # scaling: I/A ~ 1/a
    s = 3.7e-5
    assert oracle.tri_potential(c * s, v0 * s, v1 * s, v2 * s) / (A * s * s) == pytest.approx(
        g["equilateral_centroid"] / s, rel=1e-13)


def test_closed_form_unit_square():
    g = golden()
    c = np.array([0.5, 0.5, 0.0])
    a, b, cc, d = [np.array(p, dtype=float) for p in ([0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0])]
    I = oracle.tri_potential(c, a, b, cc) + oracle.tri_potential(c, a, cc, d)
    assert I == pytest.approx(g["unit_square_centre"], rel=1e-14)


def test_far_limit():
    g = golden()
    # unit-area right triangle, observer 100 above its centroid
    L = np.sqrt(2.0)
    v0, v1, v2 = np.array([0, 0, 0.]), np.array([L, 0, 0.]), np.array([0, L, 0.])
    c = (v0 + v1 + v2) / 3
    I = oracle.tri_potential(c + [0, 0, 100.0], v0, v1, v2)
    assert I == pytest.approx(g["far_limit"], rel=2e-5)
    # second-order on-axis term: I = A/d - J/(2 d^3) + O(d^-5), with the polar
    # moment about the centroid of a right triangle J = A (a^2 + b^2) / 18
    J = 1.0 * (L * L + L * L) / 18.0
    for d in (30.0, 100.0):
        I = oracle.tri_potential(c + [0, 0, d], v0, v1, v2)
        assert I == pytest.approx(1.0 / d - J / (2 * d ** 3), rel=3.0 / d ** 4)
    # and the O((size/d)^2) approach to 1/d along an arbitrary direction
    errs = []
    for d in (10.0, 100.0, 1000.0):
        u = np.array([0.3, -0.5, 0.8]); u /= np.linalg.norm(u)
        errs.append(abs(oracle.tri_potential(c + d * u, v0, v1, v2) * d - 1.0))
    assert errs[1] < errs[0] / 50 and errs[2] < errs[1] / 50


def _rand_tri(rng, scale=1.0):
    while True:
        v = rng.normal(size=(3, 3)) * scale
        if np.linalg.norm(np.cross(v[1] - v[0], v[2] - v[0])) > 0.2 * scale * scale:
            return v


@pytest.mark.parametrize("seed", range(6))
def test_against_polar_quadrature(seed):
    """Random triangles, observers: off-plane near/far, coplanar interior,
    coplanar exterior, on the backward extension of an edge line, near an
    edge, at a vertex-adjacent point."""
    rng = np.random.default_rng(seed)
    v = _rand_tri(rng)
    v0, v1, v2 = v
    n = np.cross(v1 - v0, v2 - v0); n /= np.linalg.norm(n)
    c = v.mean(axis=0)
    obs = [
        c + 0.37 * n,                                   # off-plane above centroid
        c + rng.normal(size=3) * 0.5,                   # generic
        c + 3.0 * rng.normal(size=3),                   # farther
        0.2 * v0 + 0.5 * v1 + 0.3 * v2,                 # coplanar interior
        2.0 * v0 - 0.6 * v1 - 0.4 * v2,                 # coplanar exterior
        v0 + 1.7 * (v0 - v1),                           # on edge line, backward extension
        v0 + 1.7 * (v0 - v1) + 1e-3 * n,                # ... slightly off-plane
        0.5 * (v0 + v1) + 1e-4 * (c - 0.5 * (v0 + v1)),  # just inside near an edge midpoint
        v0 + 1e-3 * (c - v0),                           # near a vertex
    ]
    for r in obs:
        got = oracle.tri_potential(r, v0, v1, v2)
        ref = tri_potential_quad(r, v0, v1, v2)
        assert got == pytest.approx(ref, rel=2e-11, abs=1e-13), (r, got, ref)


def test_additivity_midpoint_split():
    """I(T) = sum of I over the 4 midpoint sub-triangles (catches sign/orientation
    errors in the per-edge terms, since inner edges cancel)."""
    rng = np.random.default_rng(11)
    for _ in range(20):
        v0, v1, v2 = _rand_tri(rng)
        m01, m12, m20 = (v0 + v1) / 2, (v1 + v2) / 2, (v2 + v0) / 2
        subs = [(v0, m01, m20), (m01, v1, m12), (m20, m12, v2), (m01, m12, m20)]
        for r in (rng.normal(size=3), (v0 + v1 + v2) / 3, 0.1 * v0 + 0.3 * v1 + 0.6 * v2):
            tot = oracle.tri_potential(r, v0, v1, v2)
            parts = sum(oracle.tri_potential(r, *s) for s in subs)
            assert parts == pytest.approx(tot, rel=1e-12)


def test_isometry_invariance_and_winding():
    rng = np.random.default_rng(5)
    for _ in range(20):
        v = _rand_tri(rng)
        r = rng.normal(size=3)
        q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        t = rng.normal(size=3) * 10
        a = oracle.tri_potential(r, *v)
        b = oracle.tri_potential(q @ r + t, *(q @ x + t for x in v))
        c = oracle.tri_potential(r, v[0], v[2], v[1])  # reversed winding
        assert b == pytest.approx(a, rel=1e-12)
        assert c == pytest.approx(a, rel=1e-13)


def test_geometry():
    m = meshes.bar()
    g = oracle.Geometry(m.verts, m.tris)
    assert g.n == 2100
    # bar surface area 4*1000*100 + 2*100*100 um^2
    assert g.area.sum() == pytest.approx((4 * 1000 * 100 + 2 * 100 * 100) * 1e-12, rel=1e-12)
    assert np.allclose(g.dmax, 20e-6 * np.sqrt(2), rtol=1e-14)
    assert np.allclose(g.cent, m.verts[m.tris].mean(axis=1), rtol=0, atol=1e-18)


def _brute_p(g, eta=oracle.ETA):
    """Dense P from its definition, with every triangle integral done by the
    independent polar quadrature and the near test in numpy."""
    n = g.n
    V = g.verts[g.tris]
    I = np.empty((n, n))  # I[k,l] = I(c_k; T_l)
    for k in range(n):
        for l in range(n):
            I[k, l] = tri_potential_quad(g.cent[k], *V[l], epsrel=1e-12)
    P = np.empty((n, n))
    for k in range(n):
        for l in range(n):
            if k == l:
                P[k, l] = I[k, k] / g.area[k]
                continue
            d = g.cent[k] - g.cent[l]
            d2 = (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]
            t = eta * max(g.dmax[k], g.dmax[l])
            if d2 < t * t:
                P[k, l] = 0.5 * (I[k, l] / g.area[l] + I[l, k] / g.area[k])
            else:
                P[k, l] = 1.0 / np.sqrt(d2)
    return P


def test_dense_p_brute_force_tiny_mesh():
    """Oracle P entries and MVM vs. brute force on a 48-panel cube and a
    stretched box (mixed near / far pairs)."""
    for m in (meshes.small_mesh("cube", n=2),
              meshes.Mesh(*meshes.voxel_surface(np.ones((4, 1, 1), bool), (0, 0, 0), (1.0, 1.0, 1.0)))):
        g = oracle.Geometry(m.verts, m.tris)
        P = oracle.dense_p(g)
        Pb = _brute_p(g)
        near_frac = np.mean(P != 1.0 / np.maximum(np.linalg.norm(g.cent[:, None] - g.cent[None], axis=2), 1e-300))
        assert 0.05 < near_frac < 1.0
        np.testing.assert_allclose(P, Pb, rtol=1e-10, atol=0)
        x = meshes.make_x(1, g.n)
        y = oracle.mvm_rows(g, x)
        yb = (Pb @ x.astype(np.complex128).T).T
        assert oracle.rel_l2(y, yb) < 1e-12


def test_p_symmetric_and_spd_config1():
    """P is exactly symmetric by construction (symmetrised near entries, the
    near test is symmetric) and SPD on config 1 (PAPER.md:124
    positive-definiteness argument)."""
    m = meshes.bar()
    g = oracle.Geometry(m.verts, m.tris)
    P = oracle.dense_p(g)
    assert np.array_equal(P, P.T)
    w = np.linalg.eigvalsh(P)
    assert w.min() > 0
    # congruent triangles: identical self terms; right isosceles leg a:
    # I/A at centroid = 4.814459846328/a, checked by quadrature here
    a = 20e-6
    ref = tri_potential_quad(np.array([a / 3, a / 3, 0]), [0, 0, 0], [a, 0, 0], [0, a, 0]) / (a * a / 2)
    np.testing.assert_allclose(np.diag(P), ref, rtol=1e-10)


def test_mvm_rows_subset_linear_zero():
    m = meshes.bar()
    g = oracle.Geometry(m.verts, m.tris)
    x = meshes.make_x(1, g.n)
    rows = np.array([0, 7, 1000, 2099, 1500], dtype=np.int64)
    y_all = oracle.mvm_rows(g, x)
    y_sub = oracle.mvm_rows(g, x, rows)
    np.testing.assert_array_equal(y_sub, y_all[:, rows])
    assert np.all(oracle.mvm_rows(g, np.zeros_like(x), rows) == 0)
    y2 = oracle.mvm_rows(g, (2.5 * x.astype(np.complex128)), rows)
    np.testing.assert_allclose(y2, 2.5 * y_sub, rtol=1e-13)


def test_near_rows_pattern_and_ties():
    m = meshes.bar()
    g = oracle.Geometry(m.verts, m.tris)
    ptr, cols, vals, inv_r = oracle.near_rows(g)
    # pattern symmetric and contains the diagonal
    S = set()
    for k in range(g.n):
        cs = cols[ptr[k]:ptr[k + 1]]
        assert k in cs
        assert np.all(np.diff(cs) > 0)
        S.update((k, int(l)) for l in cs)
    assert all((l, k) in S for (k, l) in S)
    nnz_per_row = (ptr[-1]) / g.n
    assert 25 < nnz_per_row < 35
    # values equal the dense P entries
    P = oracle.dense_p(g)
    rows = np.repeat(np.arange(g.n), np.diff(ptr))
    np.testing.assert_array_equal(vals, P[rows, cols])
    # no pair within 1e-9 relative of the eta threshold (reading R3)
    assert oracle.tie_audit(g) == 0


# ---------------------------------------------------------------- NEXT f4: rectangles, Galerkin rule

def _square(a, galerkin=False):
    V = np.array([[0, 0, 0], [a, 0, 0], [a, a, 0], [0, a, 0]], dtype=float)
    return oracle.Geometry(V, np.array([[0, 1, 2, 3]], np.int32), galerkin=galerkin)


def test_rectangle_geometry_and_self_term_closed_form():
    """A square panel of side a: centroid at its centre, area a^2, D = the diagonal a sqrt 2, and the
    collocation self term I(centre)/A = 4 ln(1 + sqrt 2)/a (the uniform square's potential at its centre)."""
    a = 2e-5
    g = _square(a)
    assert np.allclose(g.cent[0], [a / 2, a / 2, 0], rtol=0, atol=1e-21)
    assert g.area[0] == pytest.approx(a * a, rel=1e-15)
    assert g.dmax[0] == pytest.approx(a * np.sqrt(2), rel=1e-15)
    assert oracle.dense_p(g)[0, 0] == pytest.approx(4 * np.log(1 + np.sqrt(2)) / a, rel=1e-13)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_rectangle_potential_vs_polar_quadrature(seed):
    """I(r; parallelogram) of a tilted panel against the independent polar quadrature of its two
    triangles (tests/quadrature.py), at off-plane and in-plane observers."""
    rng = np.random.default_rng(seed)
    a0 = rng.normal(size=3)
    e1, e2 = rng.normal(size=3), rng.normal(size=3)
    V = np.array([a0, a0 + e1, a0 + e1 + e2, a0 + e2])
    g = oracle.Geometry(V, np.array([[0, 1, 2, 3]], np.int32))
    n = np.cross(e1, e2)
    for r in (a0 + 0.3 * e1 + 0.6 * e2 + 0.2 * n, a0 + 1.4 * e1 + 0.2 * e2, a0 + 0.5 * e1 + 0.5 * e2 + 2 * n):
        ref = tri_potential_quad(r, V[0], V[1], V[2]) + tri_potential_quad(r, V[0], V[2], V[3])
        assert oracle.panel_potential(r, g, 0) == pytest.approx(ref, rel=1e-9)


def test_outer_rules_polynomial_exactness():
    """Radon's 7-point rule integrates every monomial of degree <= 5 exactly over a triangle; the 2 x 2
    Gauss product rule integrates s^i t^j (i, j <= 3) exactly over a parallelogram."""
    from math import factorial
    V = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 0]])
    g = oracle.Geometry(V, np.array([[0, 1, 2, -1]], np.int32))
    x, w = oracle.outer_rule(g, 0)
    assert len(w) == 7 and w.sum() == pytest.approx(1.0, abs=1e-15)
    for i in range(6):
        for j in range(6 - i):
            exact = factorial(i) * factorial(j) / factorial(i + j + 2) / 0.5  # mean over the unit right triangle
            assert (w * x[:, 0] ** i * x[:, 1] ** j).sum() == pytest.approx(exact, rel=1e-13, abs=1e-16)
    Vq = np.array([[0.0, 0, 0], [2, 0, 0], [3, 1, 0], [1, 1, 0]])  # parallelogram: s e1 + t e2
    gq = oracle.Geometry(Vq, np.array([[0, 1, 2, 3]], np.int32))
    xq, wq = oracle.outer_rule(gq, 0)
    assert len(wq) == 4
    t = xq[:, 1]
    s = (xq[:, 0] - t) / 2
    for i in range(4):
        for j in range(4):
            assert (wq * s ** i * t ** j).sum() == pytest.approx(1 / ((i + 1) * (j + 1)), rel=1e-13)


def test_galerkin_self_terms_against_exact_double_integrals():
    """Galerkin self terms (1/A^2) int int dS dS'/|r - r'|: the unit-square closed form
    4 ln(1 + sqrt 2) - (4/3)(sqrt 2 - 1) (per side a: / a), and for a right triangle a 2-D adaptive
    quadrature of the analytic inner integral.  The outer rules land within 3 % (2 x 2 Gauss, square:
    +2.2 %) and 1 % (7 points, triangle: +0.5 %) of the exact values, more than 5x closer than the
    centroid collocation (+19 %, +20 %)."""
    from scipy.integrate import dblquad
    a = 3e-5
    exact = (4 * np.log(1 + np.sqrt(2)) - 4.0 / 3.0 * (np.sqrt(2) - 1)) / a
    pg = oracle.dense_p(_square(a, galerkin=True))[0, 0]
    pc = oracle.dense_p(_square(a))[0, 0]
    assert abs(pg - exact) / exact < 0.03 and abs(pg - exact) < abs(pc - exact) / 5
    V = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 0]])
    gt = oracle.Geometry(V, np.array([[0, 1, 2, -1]], np.int32), galerkin=True)
    gc = oracle.Geometry(V, np.array([[0, 1, 2, -1]], np.int32))
    val, _ = dblquad(lambda y, x: oracle.panel_potential([x, y, 0.0], gc, 0), 0, 1, 0, lambda x: 1 - x,
                     epsabs=1e-10, epsrel=1e-9)
    exact_t = val / 0.25  # (1/A^2) with A = 1/2
    pg_t, pc_t = oracle.dense_p(gt)[0, 0], oracle.dense_p(gc)[0, 0]
    assert abs(pg_t - exact_t) / exact_t < 0.01 and abs(pg_t - exact_t) < abs(pc_t - exact_t) / 5


def test_hybrid_mesh_p_symmetric_and_far_entries():
    """Hybrid bar (rectangles + triangles): P symmetric (both near rules), far entries 1/r, and the
    Galerkin rule touches only self and vertex-adjacent near pairs."""
    m = meshes.bar_hybrid(length=200e-6, side=40e-6, cell=20e-6)
    g = oracle.Geometry(m.verts, m.tris)
    gg = oracle.Geometry(m.verts, m.tris, galerkin=True)
    P, Pg = oracle.dense_p(g), oracle.dense_p(gg)
    assert np.allclose(P, P.T, rtol=1e-13, atol=0) and np.allclose(Pg, Pg.T, rtol=1e-13, atol=0)
    d = np.linalg.norm(g.cent[:, None] - g.cent[None], axis=2)
    far = d >= oracle.ETA * np.maximum(g.dmax[:, None], g.dmax[None])
    np.fill_diagonal(far, False)
    assert np.array_equal(P[far], 1 / d[far]) and np.array_equal(Pg[far], P[far])
    pv = [set(r[r >= 0]) for r in m.tris]
    diff = np.argwhere(Pg != P)
    assert all(k == l or pv[k] & pv[l] for k, l in diff)
    assert len(diff) > m.n


def test_galerkin_adjacent_rectangle_triangle_pair_against_double_integral():
    """Pins the Galerkin near rule on a vertex/edge-adjacent pair of DIFFERENT panel types (rectangle k on
    a long face, triangle l on the end cap, sharing an edge; A_k = 2 A_l): the oracle's symmetrised entry
    1/2 [rule_k I(.; S_l)/A_l + rule_l I(.; S_k)/A_k] must approximate the exact Galerkin entry
    (1/(A_k A_l)) int_{S_k} int_{S_l} dS dS'/|r - r'| to the outer rules' accuracy (< 3 %).  The exact value
    is an independent nested quadrature: scipy dblquad over S_k of the polar-coordinate inner integral
    (tests/quadrature.py) over S_l.  Swapping A_k and A_l in either term moves the entry by ~25-50 % and a
    wrong rule/panel pairing by more, so a normalisation slip fails here."""
    from scipy.integrate import dblquad
    from tests.quadrature import tri_potential_quad
    m = meshes.bar_hybrid(length=200e-6, side=40e-6, cell=20e-6)
    gg = oracle.Geometry(m.verts, m.tris, galerkin=True)
    quads = [k for k in range(m.n) if m.tris[k, 3] >= 0]
    tris = [k for k in range(m.n) if m.tris[k, 3] < 0]
    pair = None
    for k in quads:
        sk = set(m.tris[k])
        for l in tris:
            if len(sk & set(m.tris[l, :3])) == 2:
                pair = (k, l)
                break
        if pair:
            break
    k, l = pair
    V = m.verts
    a, b, c, d = (V[i] for i in m.tris[k])
    ta, tb, tc = (V[i] for i in m.tris[l, :3])
    Ak = np.linalg.norm(np.cross(b - a, d - a))
    Al = 0.5 * np.linalg.norm(np.cross(tb - ta, tc - ta))
    assert Ak == pytest.approx(2 * Al, rel=1e-12)

    def inner(r):
        return tri_potential_quad(r, ta, tb, tc, epsrel=1e-8)
    val, err = dblquad(lambda t, s: inner(a + s * (b - a) + t * (d - a)), 0, 1, 0, 1, epsabs=0, epsrel=1e-5)
    exact = val * Ak / (Ak * Al)  # ds dt = dS / A_k
    pg = oracle.p_entries(gg, [k], [l])[0, 0]
    assert pg == pytest.approx(oracle.p_entries(gg, [l], [k])[0, 0], rel=1e-13)
    print("galerkin rect-tri pair", pg, exact, (pg - exact) / exact)
    assert abs(pg - exact) / exact < 0.03
    # collocation for contrast: the centroid entry is farther from the Galerkin value
    gc = oracle.Geometry(m.verts, m.tris)
    pc = oracle.p_entries(gc, [k], [l])[0, 0]
    assert abs(pg - exact) < abs(pc - exact)
