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


# ---------------------------------------------------------------- C7: the Eq. 10 preconditioner oracle

def _bar_system():
    m = meshes.bar()
    g = oracle.Geometry(m.verts, m.tris)
    P = oracle.dense_p(g)
    br, kinds = lo.build_graph(m.tris, [(m.ports[0][1], m.ports[0][2])])
    M, ends, nn = lo.loop_basis(m.n, br, kinds)
    A = lo.cm_maps(m.verts, m.tris, g.cent, br)
    phys = sp.diags((kinds == 0).astype(float))
    A = [phys @ A[t] for t in range(3)]
    C = [M @ A[t] for t in range(3)]
    return m, g, P, M, A, C


@pytest.fixture(scope="module")
def bar_system():
    return _bar_system()


def test_precond_omega_zero_is_resistive_part(bar_system):
    """SPEC.md:443 (C7): at omega = 0 the diagonal-of-P Q of Eq. 10 is the ESI part Z_s of Eq. 8 exactly:
    it equals the dense loop system (an independent dense product, loop_system) with alpha = 0, for any
    P; the diagonal-of-L Q_L reduces to the same matrix."""
    m, g, P, M, A, C = bar_system
    zsa = lo.esi(5.8e7, 100e-6, 0.0) / g.area
    Q = lo.precond_q(C, zsa, 0.0, np.diag(P)).toarray()
    Z0 = lo.loop_system(C, P, zsa, 0.0)
    assert np.abs(Q - Z0).max() <= 1e-12 * np.abs(Z0).max()
    QL = lo.precond_q_diag_l(M, A, zsa, 0.0, P).toarray()
    assert np.abs(QL - Z0).max() <= 1e-12 * np.abs(Z0).max()


def test_precond_one_loop_strip_by_hand():
    """SPEC.md:442 (C7): the 2-panel strip of unit right triangles T0 = (0,0),(1,0),(0,1) and
    T1 = (1,0),(1,1),(0,1) with a port (+ on T0, - on T1) has one loop; Q is 1 x 1 and, by hand,
    Q = sum_t [(m - c0)_t^2 d0 + (m - c1)_t^2 d1] = (d0 + d1)/18 with the shared-edge midpoint
    m = (1/2, 1/2), centroids (1/3, 1/3), (2/3, 2/3), and d_k = Z_s/A_k + alpha P_kk,
    A_k = 1/2, P_kk = 4.814459846328 (the right-isosceles centroid self term, golden pin 2).
    So apply(v) = 18 v / (d0 + d1)."""
    v = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0]], float)
    t = np.array([[0, 1, 2], [1, 3, 2]], np.int32)
    g = oracle.Geometry(v, t)
    br, kinds = lo.build_graph(t, [([0], [1])])
    M, ends, nn = lo.loop_basis(2, br, kinds)
    assert M.shape[0] == 1
    A = lo.cm_maps(v, t, g.cent, br)
    C = [M @ A[k] for k in range(3)]
    zs, alpha = 0.37 + 0.11j, 2.5j
    pkk = np.array([4.814459846328, 4.814459846328])
    d = zs / 0.5 + alpha * pkk
    q_hand = (d[0] + d[1]) / 18.0
    Q = lo.precond_q(C, np.full(2, zs) / g.area, alpha, np.diag(oracle.dense_p(g)))
    assert Q.shape == (1, 1)
    assert abs(Q[0, 0] - q_hand) <= 1e-11 * abs(q_hand)
    vv = np.array([[1.0 + 2.0j]])
    z = lo.precond_apply(C, np.full(2, zs) / g.area, alpha, np.diag(oracle.dense_p(g)), [0, 1], vv)
    assert abs(z[0, 0] - vv[0, 0] / q_hand) <= 1e-11 * abs(vv[0, 0] / q_hand)


def test_precond_whole_block_round_trip(bar_system):
    """SPEC.md:460 (C7): with one block (the exact Q^-1 of Eq. 11), apply(Q x) = x to 1e-9, where Q x is
    formed by the dense product sum_t C_t (diag(zsa) + alpha diag(P_kk)) C_t^T (loop_system with the
    diagonal of P), independent of precond_q's sparse assembly; the diag-of-L Q_L likewise against its
    dense edge-space product M (sum_t A_t diag(zsa) A_t^T + alpha diag(sum_t A_t P A_t^T)) M^T."""
    m, g, P, M, A, C = bar_system
    f = 1e8
    zsa = lo.esi(5.8e7, 100e-6, f) / g.area
    alpha = 1j * 2 * np.pi * f * lo.MU0 / (4 * np.pi)
    nl = M.shape[0]
    rng = np.random.default_rng(11)
    x = rng.normal(size=(2, nl)) + 1j * rng.normal(size=(2, nl))
    Qd = lo.loop_system(C, np.diag(np.diag(P)), zsa, alpha)
    z = lo.precond_apply(C, zsa, alpha, np.diag(P), [0, nl], (Qd @ x.T).T)
    assert np.linalg.norm(z - x) <= 1e-9 * np.linalg.norm(x)
    Md = M.toarray()
    Ad = [A[t].toarray() for t in range(3)]
    Le = sum(Ad[t] @ P @ Ad[t].T for t in range(3))
    Zs = sum(Ad[t] @ np.diag(zsa) @ Ad[t].T for t in range(3))
    QLd = Md @ (Zs + alpha * np.diag(np.diag(Le))) @ Md.T
    QL = lo.precond_q_diag_l(M, A, zsa, alpha, P)
    assert np.abs(QL.toarray() - QLd).max() <= 1e-12 * np.abs(QLd).max()
    zl = lo.block_solve(QL, [0, nl], (QLd @ x.T).T)
    assert np.linalg.norm(zl - x) <= 1e-9 * np.linalg.norm(x)


def test_precond_blocks_solve_their_diagonal_blocks(bar_system):
    """Block-Jacobi (reading C-A10): for a 64-loop partition, each output block z_B solves Q_BB z_B = v_B
    with Q_BB cut from the dense product (not from precond_q)."""
    m, g, P, M, A, C = bar_system
    f = 1e6
    zsa = lo.esi(5.8e7, 100e-6, f) / g.area
    alpha = 1j * 2 * np.pi * f * lo.MU0 / (4 * np.pi)
    nl = M.shape[0]
    bptr = list(range(0, nl, 64)) + [nl]
    v = np.random.default_rng(2).normal(size=(1, nl)) + 0j
    z = lo.precond_apply(C, zsa, alpha, np.diag(P), bptr, v)
    Qd = lo.loop_system(C, np.diag(np.diag(P)), zsa, alpha)
    for a, b in zip(bptr[:-1], bptr[1:]):
        r = Qd[a:b, a:b] @ z[0, a:b] - v[0, a:b]
        assert np.linalg.norm(r) <= 1e-10 * np.linalg.norm(v[0, a:b])


def test_precond_pattern_frequency_invariant(bar_system):
    """SPEC.md:467 (C7): Q's sparsity pattern is the same at every frequency (only values change); the
    diag-of-L source matrix before the loop mapping is diagonal (N_e entries) while diag-of-P
    couples the edges of each panel."""
    m, g, P, M, A, C = bar_system
    pats = []
    for f in (1e3, 1e6, 1e9, 1e10):
        zsa = lo.esi(5.8e7, 100e-6, f) / g.area
        alpha = 1j * 2 * np.pi * f * lo.MU0 / (4 * np.pi)
        Q = lo.precond_q(C, zsa, alpha, np.diag(P))
        Q.eliminate_zeros()
        Q.sort_indices()
        pats.append((Q.indptr.copy(), Q.indices.copy()))
    for ip, ix in pats[1:]:
        assert np.array_equal(ip, pats[0][0]) and np.array_equal(ix, pats[0][1])
    nphys = A[0].getnnz(axis=1).astype(bool).sum()
    Ad = [A[t].toarray() for t in range(3)]
    edge_p = sum(Ad[t] @ np.diag(np.diag(P)) @ Ad[t].T for t in range(3))
    assert np.count_nonzero(edge_p) > nphys  # diag-of-P: same-panel edges coupled
