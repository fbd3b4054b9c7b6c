"""XRL loop-space ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Plain FP64 numpy/scipy implementation of what SURVEY §8(a) a14-a17 compute,
following the paper step by step, on small meshes:

  * esi():          Eq. 3, reading R12 (R_RF = sqrt(pi mu0/sigma))
  * cm_maps():      Algorithm 1 for a given branch list
  * loop_basis():   loop matrix M of Eq. 7 by fundamental
                    cycles of a BFS spanning tree, port branches forced into
                    the co-tree (independent of the library's vertex loops)
  * loop_system():  Eq. 7-9: M sum_t A_t (diag(Z_s/A) + alpha P) A_t^T M^T,
                    alpha = j omega mu0/(4 pi), P the oracle's dense P
  * port_impedance(): dense solve (numpy LU) and Z_port = V / I_port
  * precond_q():     Eq. 10 Q = sum_t C_t diag(Z_s/A + alpha P_kk) C_t^T
  * precond_q_diag_l(): the diagonal-of-L baseline of PAPER.md:120-122
  * precond_apply() / block_solve(): Eq. 11 with Q's diagonal blocks inverted
                    (numpy LU), applied block-wise (one block = the exact Q^-1)

It never imports paper_2409_12375_b200.  Library data (branch orientation,
loop matrix, block partition) enters only as plain input arrays where the
test compares basis-dependent quantities.
"""
from __future__ import annotations

from collections import deque

import numpy as np
import scipy.sparse as sp

MU0 = 4e-7 * np.pi


def esi(sigma: float, zeta: float, f: float) -> complex:
    """Z_s = (1+j) R_RF sqrt(f) / (1 - exp(-(1+j) R_RF sqrt(f) / R_DC)),
    R_DC = 2/(sigma zeta), R_RF = sqrt(pi mu0 / sigma); f = 0 -> R_DC."""
    rdc = 2.0 / (sigma * zeta)
    if f == 0:
        return complex(rdc)
    rrf = np.sqrt(np.pi * MU0 / sigma)
    a = (1 + 1j) * rrf * np.sqrt(f)
    return complex(a / (1 - np.exp(-a / rdc)))


def _corners(t):
    """Vertex ids of a panel row ([3] triangle, or [4] with -1 for a triangle)."""
    return [int(v) for v in t if v >= 0]


def interior_edges(tris):
    """Interior edges of a triangle or hybrid triangle/rectangle mesh: list of (p, q, va, vb), p < q
    panels."""
    tris = np.asarray(tris)
    d = {}
    for p, t in enumerate(tris):
        c = _corners(t)
        for e in range(len(c)):
            a, b = c[e], c[(e + 1) % len(c)]
            k = (min(a, b), max(a, b))
            d.setdefault(k, []).append(p)
    out = []
    for (a, b), ps in d.items():
        if len(ps) == 2:
            out.append((min(ps), max(ps), a, b))
        elif len(ps) > 2:
            raise ValueError("non-manifold edge")
    out.sort()
    return out


def cm_maps(verts, tris, cent, branches):
    """Algorithm 1: for each physical branch (a -> b) between panels a and b
    sharing an edge with midpoint m: A_t(e, a) = (m - c_a)_t (rho_a points
    along the current), A_t(e, b) = -(m - c_b)_t.  Returns 3 sparse
    [n_branches x n_panels] matrices (rows of non-physical branches empty)."""
    verts = np.asarray(verts)
    tris = np.asarray(tris)
    n = tris.shape[0]
    rows, cols, vals = [], [], [[], [], []]
    for e, (a, b) in enumerate(branches):
        if a < 0 or b < 0:
            continue
        common = sorted(set(_corners(tris[a])) & set(_corners(tris[b])))
        assert len(common) == 2
        m = 0.5 * (verts[common[0]] + verts[common[1]])
        ra = m - cent[a]
        rb = m - cent[b]
        for p, r, s in ((a, ra, 1.0), (b, rb, -1.0)):
            rows.append(e)
            cols.append(p)
            for t in range(3):
                vals[t].append(s * r[t])
    return [sp.csr_matrix((vals[t], (rows, cols)), shape=(len(branches), n)) for t in range(3)]


def build_graph(tris, ports):
    """Branches: interior edges (p -> q, p < q), then per port terminal
    branches (S+ -> k for k in plus, k -> S- for k in minus) and the port
    branch S- -> S+.  Super-node s is encoded as -1-s."""
    br = [(p, q) for (p, q, _, _) in interior_edges(tris)]
    kinds = [0] * len(br)
    for i, (plus, minus) in enumerate(ports):
        sp_, sm_ = -1 - 2 * i, -2 - 2 * i
        for k in plus:
            br.append((sp_, int(k)))
            kinds.append(1)
        for k in minus:
            br.append((int(k), sm_))
            kinds.append(1)
        br.append((sm_, sp_))
        kinds.append(2)
    return br, np.array(kinds)


def loop_basis(n_panels, branches, kinds):
    """Fundamental cycles of a BFS spanning forest (port branches never in the
    tree).  Returns sparse M [n_loops x n_branches] with entries +-1."""
    nodes = {}

    def nid(x):
        if x not in nodes:
            nodes[x] = len(nodes)
        return nodes[x]
    for i in range(n_panels):
        nid(i)
    ends = [(nid(a), nid(b)) for a, b in branches]
    nn = len(nodes)
    adj = [[] for _ in range(nn)]
    for e, (a, b) in enumerate(ends):
        if kinds[e] == 2:
            continue
        adj[a].append(e)
        adj[b].append(e)
    par = [-1] * nn
    depth = [-1] * nn
    for r in range(nn):
        if depth[r] >= 0:
            continue
        depth[r] = 0
        q = deque([r])
        while q:
            u = q.popleft()
            for e in adj[u]:
                a, b = ends[e]
                o = b if a == u else a
                if depth[o] < 0:
                    depth[o] = depth[u] + 1
                    par[o] = e
                    q.append(o)
    tree = set(e for e in par if e >= 0)
    rows, cols, vals = [], [], []
    nl = 0
    for e, (a, b) in enumerate(ends):
        if e in tree:
            continue
        # traverse e from a to b, then the tree path from b back to a
        path = [(e, 1)]
        x, y = b, a
        up_x, up_y = [], []
        while x != y:
            if depth[x] >= depth[y]:
                pe = par[x]
                pa, pb = ends[pe]
                up_x.append((pe, 1 if pa == x else -1))
                x = pb if pa == x else pa
            else:
                pe = par[y]
                pa, pb = ends[pe]
                py = pb if pa == y else pa
                up_y.append((pe, 1 if pa == py else -1))
                y = py
        path += up_x + up_y[::-1]
        for be, s in path:
            rows.append(nl)
            cols.append(be)
            vals.append(s)
        nl += 1
    M = sp.csr_matrix((vals, (rows, cols)), shape=(nl, len(branches)))
    return M, ends, nn


def kcl_residual(M, ends, n_nodes):
    """max |B M^T| with B the node-branch incidence matrix (+1 tail, -1 head)."""
    nb = len(ends)
    r, c, v = [], [], []
    for e, (a, b) in enumerate(ends):
        r += [a, b]
        c += [e, e]
        v += [1, -1]
    B = sp.csr_matrix((v, (r, c)), shape=(n_nodes, nb))
    return float(abs(B @ M.T).max()) if M.shape[0] else 0.0


def loop_system(C, P, zsa, alpha):
    """Z_loop = sum_t C_t (diag(zsa) + alpha P) C_t^T (dense, complex128)."""
    Z = 0
    for t in range(3):
        Ct = C[t].toarray() if sp.issparse(C[t]) else C[t]
        Z = Z + Ct @ ((np.diag(zsa) + alpha * P) @ Ct.T)
    return Z


def port_impedance(verts, tris, cent, area, P, ports, zs, freq):
    """Z matrix of the ports (Y = I/V with the other ports shorted, Z = Y^-1)
    from a dense FP64 solve of the loop system with the oracle's own basis."""
    branches, kinds = build_graph(tris, ports)
    M, ends, nn = loop_basis(len(tris), branches, kinds)
    A = cm_maps(verts, tris, cent, branches)
    phys = sp.diags((kinds == 0).astype(float))
    C = [M @ phys @ A[t] for t in range(3)]
    alpha = 1j * 2 * np.pi * freq * MU0 / (4 * np.pi)
    zsa = np.broadcast_to(np.asarray(zs, dtype=complex), (len(tris),)) / area
    Z = loop_system(C, P, zsa, alpha)
    pb = np.nonzero(kinds == 2)[0]
    Y = np.zeros((len(pb), len(pb)), dtype=complex)
    for q, b in enumerate(pb):
        V = M[:, b].toarray().ravel().astype(complex)
        I = np.linalg.solve(Z, V)
        Ib = M.T @ I
        Y[:, q] = Ib[pb]
    return np.linalg.inv(Y), {"n_loops": M.shape[0], "kcl": kcl_residual(M, ends, nn)}


def precond_q(C, zsa, alpha, pkk):
    """Eq. 10, the diagonal-of-P preconditioner as a sparse
    matrix: Q = Z_s + M (sum_t A_t P_d A_t^T) M^T with the jw mu0/4pi factor
    alpha on the P_d term (reading C-A7) and Z_s = M (sum_t A_t diag(Z_s/A)
    A_t^T) M^T the ESI part of Eq. 8, i.e. with C_t = M A_t,
        Q = sum_t C_t diag(zsa + alpha P_kk) C_t^T."""
    d = np.asarray(zsa) + alpha * np.asarray(pkk)
    Q = 0
    for t in range(3):
        Ct = sp.csr_matrix(C[t])
        Q = Q + Ct @ sp.diags(d) @ Ct.T
    return sp.csr_matrix(Q)


def precond_q_diag_l(M, A, zsa, alpha, P):
    """The traditional diagonal-of-L preconditioner:
    Q_L = Z_s + jw L_d with L_d "formed by the diagonal entries of the
    edge-edge interaction matrix" L = sum_t A_t P A_t^T (the edge matrix of
    Eq. 5/7 with mu0/4pi pulled out, reading C-A7), mapped to loops like
    Eq. 7:  Q_L = M [ sum_t A_t diag(zsa) A_t^T + alpha diag(L_ee) ] M^T.
    A: the 3 branch x panel maps of Algorithm 1 (physical branches only);
    P: the dense (or any indexable) panel matrix -- only the entries P_ij of
    the two panels of each edge are used."""
    Zs = 0
    for t in range(3):
        At = sp.csr_matrix(A[t])
        Zs = Zs + At @ sp.diags(np.asarray(zsa)) @ At.T
    nb = A[0].shape[0]
    Ld = np.zeros(nb)
    for t in range(3):
        At = sp.csr_matrix(A[t])
        for e in range(nb):
            cols = At.indices[At.indptr[e]:At.indptr[e + 1]]
            vals = At.data[At.indptr[e]:At.indptr[e + 1]]
            Ld[e] += sum(vals[a] * vals[b] * P[cols[a], cols[b]] for a in range(len(cols)) for b in range(len(cols)))
    M = sp.csr_matrix(M)
    return sp.csr_matrix(M @ (Zs + alpha * sp.diags(Ld)) @ M.T)


def block_solve(Q, block_ptr, v):
    """z_B = Q_BB^{-1} v_B for each block [block_ptr[i], block_ptr[i+1]) of a
    sparse Q (dense LU per block, numpy).  v: [..., N_l]."""
    Q = sp.csr_matrix(Q)
    z = np.zeros_like(v, dtype=complex)
    for i in range(len(block_ptr) - 1):
        a, b = block_ptr[i], block_ptr[i + 1]
        QB = Q[a:b, a:b].toarray()
        z[..., a:b] = np.linalg.solve(QB, v[..., a:b].T).T
    return z


def precond_apply(C, zsa, alpha, pkk, block_ptr, v):
    """Eq. 10-11 in block-Jacobi form (reading C-A10): z_B = Q_BB^{-1} v_B
    with Q of precond_q; block_ptr = [0, N_l] is the exact Q^{-1} v."""
    return block_solve(precond_q(C, zsa, alpha, pkk), block_ptr, v)


def bar_partial_inductance_tube(length, side):
    """Closed-form partial self-inductance of a thin-walled square tube of
    perimeter GMD g = 2^(1/4) e^((pi-6)/4) side: L = mu0 l/(2 pi) [ln(2l/g) - 1 + g/l]."""
    g = 2 ** 0.25 * np.exp((np.pi - 6) / 4) * side
    return MU0 * length / (2 * np.pi) * (np.log(2 * length / g) - 1 + g / length)
