"""Pins of the loop-space oracle (oracle/loop_oracle.py): Eq. 3 limits, the
loop basis (KCL, cycle rank), a hand-worked 2-panel strip, operator
structure, and the DC partial self-inductance of the bar (config 1) against
its closed form.  CPU only."""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from inputs import meshes
from oracle import loop_oracle as lo


def test_esi_limits():
    s, z = 5.8e7, 35e-6
    rdc = 2 / (s * z)
    assert lo.esi(s, z, 0.0) == pytest.approx(rdc, rel=1e-15)
    # f -> 0: Z_s = R_DC x/(1 - e^-x) = R_DC (1 + x/2 + O(x^2)), x = (1+j) R_RF sqrt(f)/R_DC
    rrf = np.sqrt(np.pi * lo.MU0 / s)
    for f in (1e-3, 1e-1):
        x = (1 + 1j) * rrf * np.sqrt(f) / rdc
        assert abs(lo.esi(s, z, f) / rdc - (1 + x / 2)) < 2 * abs(x) ** 2
    zs = lo.esi(s, z, 1e13)                                      # exp term -> 0
    assert zs == pytest.approx((1 + 1j) * rrf * np.sqrt(1e13), rel=1e-12)
    # at 1 GHz the skin depth (2.09 um) << thickness: Z_s ~ (1+j)/(sigma delta)
    delta = 1 / np.sqrt(np.pi * 1e9 * lo.MU0 * s)
    assert lo.esi(s, z, 1e9) == pytest.approx((1 + 1j) / (s * delta), rel=1e-3)
    re = [lo.esi(s, z, f).real for f in np.logspace(0, 11, 23)]
    assert np.all(np.diff(re) >= 0)


def test_two_panel_strip_by_hand():
    """SPEC.md:152/213 strip: two triangles, one port (+ panel 0, - panel 1):
    N_nodes = 4, N_b = 4, one loop through port, terminal and interior branch."""
    v = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], float)
    t = np.array([[0, 1, 2], [0, 2, 3]])
    br, kinds = lo.build_graph(t, [([0], [1])])
    assert len(br) == 4 and list(kinds) == [0, 1, 1, 2]
    M, ends, nn = lo.loop_basis(2, br, kinds)
    assert M.shape == (1, 4) and nn == 4
    assert lo.kcl_residual(M, ends, nn) == 0
    assert set(np.abs(M.toarray().ravel())) == {1}
    cent = v[t].mean(axis=1)
    A = lo.cm_maps(v, t, cent, br)
    # edge 0 -> 2 shared, midpoint (0.5, 0.5, 0): A(e,0) = m - c0, A(e,1) = c1 - m
    m = np.array([0.5, 0.5, 0.0])
    for k in range(3):
        assert A[k][0, 0] == pytest.approx((m - cent[0])[k])
        assert A[k][0, 1] == pytest.approx((cent[1] - m)[k])


def test_loop_basis_counts_and_kcl():
    m = meshes.bar()
    br, kinds = lo.build_graph(m.tris, [(m.ports[0][1], m.ports[0][2])])
    M, ends, nn = lo.loop_basis(m.n, br, kinds)
    assert lo.kcl_residual(M, ends, nn) == 0
    assert M.shape[0] == len(br) - nn + 1
    # rows independent
    assert np.linalg.matrix_rank(M.toarray()) == M.shape[0]
    # the port branch lies in exactly one loop
    pb = np.nonzero(kinds == 2)[0][0]
    assert M[:, pb].nnz == 1


@pytest.fixture(scope="module")
def bar_dense():
    m = meshes.bar()
    g = oracle.Geometry(m.verts, m.tris)
    return m, g, oracle.dense_p(g)


def test_bar_dc_inductance_closed_form(bar_dense):
    """North star: DC bar partial self-inductance.  Surface current at DC is
    uniform around the perimeter, so the discrete model approaches the thin-
    walled tube (perimeter GMD): 0.519 nH for 1000 x 100 x 100 um.  Z_s = R_DC
    (reading R12).  R must equal R_DC * length / perimeter."""
    m, g, P = bar_dense
    sigma, zeta = 5.8e7, 100e-6
    rdc = 2 / (sigma * zeta)
    f = 1e3
    Z, info = lo.port_impedance(m.verts, m.tris, g.cent, g.area, P, [(m.ports[0][1], m.ports[0][2])], rdc, f)
    L = Z[0, 0].imag / (2 * np.pi * f)
    Lt = lo.bar_partial_inductance_tube(1e-3, 1e-4)
    assert info["kcl"] == 0
    assert abs(L - Lt) / Lt < 0.02, (L, Lt)
    assert Z[0, 0].real == pytest.approx(rdc * 1e-3 / 4e-4, rel=5e-3)


def test_loop_system_structure(bar_dense):
    m, g, P = bar_dense
    br, kinds = lo.build_graph(m.tris, [(m.ports[0][1], m.ports[0][2])])
    M, ends, nn = lo.loop_basis(m.n, br, kinds)
    A = lo.cm_maps(m.verts, m.tris, g.cent, br)
    phys = sp.diags((kinds == 0).astype(float))
    C = [M @ phys @ A[t] for t in range(3)]
    zsa = np.full(m.n, 3.4e-4) / g.area
    Z0 = lo.loop_system(C, P, zsa, 0.0)
    Z1 = lo.loop_system(C, P, zsa, 1j * 1e-4)
    # omega = 0: resistive part only (real); complex symmetric always
    assert np.all(Z0.imag == 0)
    assert np.allclose(Z1, Z1.T, rtol=0, atol=1e-12 * np.abs(Z1).max())
    # the potential part is symmetric positive definite on this mesh (P SPD)
    Lp = lo.loop_system(C, P, np.zeros(m.n), 1.0)
    assert np.linalg.eigvalsh(0.5 * (Lp + Lp.T).real).min() > 0


def test_hybrid_bar_loop_oracle_dc_inductance():
    """NEXT f4 on the loop oracle: the hybrid bar (rectangles on the long faces, triangles on the caps)
    has the closed-surface edge count E = V + F - 2, a KCL-exact loop basis, and its DC partial
    inductance matches the thin-walled-tube closed form (like the all-triangle bar)."""
    m = meshes.bar_hybrid()
    e = lo.interior_edges(m.tris)
    assert len(e) == m.verts.shape[0] + m.n - 2
    g = oracle.Geometry(m.verts, m.tris)
    P = oracle.dense_p(g)
    rdc = 2 / (5.8e7 * 1e-4)
    Z, info = lo.port_impedance(m.verts, m.tris, g.cent, g.area, P, [(m.ports[0][1], m.ports[0][2])], rdc, 1e3)
    assert info["kcl"] < 1e-12
    L = Z[0, 0].imag / (2 * np.pi * 1e3)
    Lt = lo.bar_partial_inductance_tube(1e-3, 1e-4)
    print("hybrid bar L", L, "tube", Lt)
    assert abs(L - Lt) / Lt < 0.02
