"""Multi-rank path on CPU (gloo, world size 2 and 3): the partition rule the
library uses (xrl_partition_cuts, a host function), and the library's
exchange plans (xrl_plan_exchange, the host code a partitioned tree / near
build runs) driving a real multi-process exchange: the halo of charges by
point-to-point send/recv, the shared-box all-reduce and the LET send/recv of
(monopole) multipoles, after which every value a rank's P2P, P2L, near rows,
M2L and M2P read must be complete; a monopole FMM computed rank by rank from
exactly those values equals the single-process one.  The CUDA kernels of the
sharded MVM are checked on one GPU by test_virtual_ranks_equal_single_gpu."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_partition_cuts_rule():
    from paper_2409_12375_b200 import xrl
    w = np.array([1, 1, 1, 1, 10, 1, 1, 1], float)
    c = xrl.partition_cuts(w, 2)
    assert c[0] == 0 and c[-1] == len(w) and np.all(np.diff(c) >= 0)
    assert c[1] in (4, 5)
    c = xrl.partition_cuts(np.ones(10), 3)
    assert list(np.diff(c)) in ([3, 4, 3], [4, 3, 3], [3, 3, 4])
    assert list(xrl.partition_cuts(np.ones(2), 4)[[0, -1]]) == [0, 2]


# ---------------------------------------------------------------- exchange plans through a real exchange

def _uniform_tree(cent, depth):
    """A uniform octree of the points at `depth` (empty boxes dropped), panels in Morton order: host arrays
    in the layout xrl_plan_exchange takes (boxes in level order; U = adjacent leaves incl. self, V = the
    non-adjacent children of the parent's neighbours; no X / W lists in a uniform tree).  Returns
    (perm, tree dict, box centres, box levels)."""
    lo = cent.min(0)
    W = (cent.max(0) - lo).max() * (1 + 1e-9)
    q = np.minimum(((cent - lo) / W * (1 << depth)).astype(np.int64), (1 << depth) - 1)
    key = np.zeros(len(cent), np.int64)
    for bit in range(depth):
        for d in range(3):
            key |= ((q[:, d] >> bit) & 1) << (3 * bit + d)
    perm = np.argsort(key, kind="stable")
    key = key[perm]
    boxes = []  # (level, ijk, pb, pe)
    for lev in range(depth + 1):
        k = key >> (3 * (depth - lev))
        starts = np.flatnonzero(np.r_[True, k[1:] != k[:-1]])
        ends = np.r_[starts[1:], len(k)]
        for a, b in zip(starts, ends):
            ijk = q[perm[a]] >> (depth - lev)
            boxes.append((lev, tuple(int(v) for v in ijk), int(a), int(b)))
    idx = {(l, ijk): i for i, (l, ijk, _, _) in enumerate(boxes)}
    nb = len(boxes)
    pb = np.array([b[2] for b in boxes], np.int32)
    pe = np.array([b[3] for b in boxes], np.int32)
    child = np.full(nb, -1, np.int32)
    for i, (l, ijk, _, _) in enumerate(boxes):
        if l < depth:
            for c in range(8):
                cijk = tuple(2 * ijk[d] + ((c >> d) & 1) for d in range(3))
                j = idx.get((l + 1, cijk))
                if j is not None and (child[i] < 0 or j < child[i]):
                    child[i] = j
    nbrs = [(dx, dy, dz) for dx in (-1, 0, 1) for dy in (-1, 0, 1) for dz in (-1, 0, 1)]
    V, U = [[] for _ in range(nb)], [[] for _ in range(nb)]
    for i, (l, ijk, _, _) in enumerate(boxes):
        if l >= 2:
            pijk = tuple(v >> 1 for v in ijk)
            for d in nbrs:
                for c in range(8):
                    cijk = tuple(2 * (pijk[e] + d[e]) + ((c >> e) & 1) for e in range(3))
                    j = idx.get((l, cijk))
                    if j is not None and max(abs(cijk[e] - ijk[e]) for e in range(3)) > 1:
                        V[i].append(j)
        if l == depth:
            for d in nbrs:
                j = idx.get((l, tuple(ijk[e] + d[e] for e in range(3))))
                if j is not None:
                    U[i].append(j)
    def csr(lists):
        ptr = np.zeros(nb + 1, np.int64)
        ptr[1:] = np.cumsum([len(x) for x in lists])
        return ptr, np.array([v for x in lists for v in sorted(x)], np.int32)
    t = {"pb": pb, "pe": pe, "child": child}
    t["v_ptr"], t["v_src"] = csr(V)
    t["u_ptr"], t["u_src"] = csr(U)
    t["x_ptr"], t["x_src"] = csr([[] for _ in range(nb)])
    t["w_ptr"], t["w_src"] = csr([[] for _ in range(nb)])
    centre = np.array([lo + (np.array(b[1]) + 0.5) * W / (1 << b[0]) for b in boxes])
    return perm, t, centre, np.array([b[0] for b in boxes])


def _plan_problem():
    import oracle
    from inputs import meshes
    m = meshes.bar()  # 2,100 panels, elongated: boxes straddle every cut at several levels
    g = oracle.Geometry(m.verts, m.tris)
    perm, t, centre, lev = _uniform_tree(g.cent, 4)
    iperm = np.empty_like(perm)
    iperm[perm] = np.arange(m.n)
    optr, ocol, _, _ = oracle.near_rows(g, perm)  # near rows in library order, columns in mesh order
    ncol = iperm[ocol].astype(np.int32)
    q = meshes.make_x(1, m.n)[0].real.astype(np.float64)[perm]  # one real charge per panel, library order
    return m, g.cent[perm], t, centre, lev, optr, ncol, q


def _monopole_fmm(t, cent, centre, q, mono, rows):
    """y_k = sum over U-list leaves of q_l / r (l != k) + sum over the V lists of the leaf and its ancestors
    of mono(s) / |c_k - centre(s)| (a monopole FMM: enough to check that every value read is the right
    one)."""
    nb = len(t["pb"])
    par = np.full(nb, -1)
    for b in range(nb):
        if t["child"][b] >= 0:
            c = t["child"][b]
            while c < nb and t["pb"][c] >= t["pb"][b] and t["pe"][c] <= t["pe"][b]:
                if par[c] < 0 and c != b:
                    par[c] = b
                c += 1
    leaf_of = {}
    for b in range(nb):
        if t["child"][b] < 0:
            for p in range(t["pb"][b], t["pe"][b]):
                leaf_of[p] = b
    y = np.zeros(len(rows))
    for i, k in enumerate(rows):
        L = leaf_of[k]
        for s in t["u_src"][t["u_ptr"][L]:t["u_ptr"][L + 1]]:
            for l in range(t["pb"][s], t["pe"][s]):
                if l != k:
                    y[i] += q[l] / np.linalg.norm(cent[k] - cent[l])
        a = L
        while a >= 0:
            for s in t["v_src"][t["v_ptr"][a]:t["v_ptr"][a + 1]]:
                y[i] += mono[s] / np.linalg.norm(cent[k] - centre[s])
            a = par[a]
    return y


def _plan_worker(rank, world, port, q_out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2409_12375_b200 import xrl
        m, cent, t, centre, lev, nptr, ncol, q = _plan_problem()
        nb = len(t["pb"])
        leaves = np.flatnonzero(t["child"] < 0)
        leaves = leaves[np.argsort(t["pb"][leaves])]
        w = (t["pe"][leaves] - t["pb"][leaves]).astype(float)
        lc = xrl.partition_cuts(w, world)
        cuts = np.array([t["pb"][leaves[c]] if c < len(leaves) else m.n for c in lc], np.int32)
        plan = xrl.plan_exchange(t, nptr, ncol, cuts, rank)
        c0, c1 = int(cuts[rank]), int(cuts[rank + 1])
        # local charges: own panels only
        x = np.full(m.n, np.nan)
        x[c0:c1] = q[c0:c1]

        def exchange(sbuf, soff, rbuf, roff, rec):
            reqs = []
            for p in range(world):
                if p == rank:
                    continue
                if soff[p + 1] > soff[p]:
                    reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(sbuf[soff[p] * rec:soff[p + 1] * rec])), p))
            for p in range(world):
                if p == rank:
                    continue
                if roff[p + 1] > roff[p]:
                    buf = torch.zeros(int(roff[p + 1] - roff[p]) * rec, dtype=torch.float64)
                    dist.recv(buf, p)
                    rbuf[roff[p] * rec:roff[p + 1] * rec] = buf.numpy()
            for r_ in reqs:
                r_.wait()

        # halo of x
        rbuf = np.zeros(max(int(plan["halo_roff"][-1]), 1))
        exchange(x[plan["halo_sidx"]], plan["halo_soff"], rbuf, plan["halo_roff"], 1)
        x[plan["halo_ridx"]] = rbuf[:len(plan["halo_ridx"])]
        # upward pass on the own panels only: partial monopoles of the relevant boxes
        mono = np.full(nb, np.nan)
        rel = (t["pb"] < c1) & (t["pe"] > c0)
        for b in np.flatnonzero(rel):
            a, e = max(t["pb"][b], c0), min(t["pe"][b], c1)
            mono[b] = q[a:e].sum()  # P2M + M2M of the own panels (linear: the partial sum)
        # shared boxes: all-reduce of the partial sums
        sh = plan["shared"]
        part = torch.from_numpy(np.where(rel[sh], mono[sh], 0.0).copy())
        dist.all_reduce(part)
        mono[sh] = part.numpy()
        # LET
        rb = np.zeros(max(int(plan["let_roff"][-1]), 1))
        exchange(mono[plan["let_sidx"]], plan["let_soff"], rb, plan["let_roff"], 1)
        mono[plan["let_ridx"]] = rb[:len(plan["let_ridx"])]
        # every value this rank's kernels read must be present and exact
        own_leaves = [L for L in leaves if c0 <= t["pb"][L] < c1]
        bad = 0
        for L in own_leaves:
            for s in t["u_src"][t["u_ptr"][L]:t["u_ptr"][L + 1]]:
                bad += int(np.any(x[t["pb"][s]:t["pe"][s]] != q[t["pb"][s]:t["pe"][s]]))
        for k in range(c0, c1):
            cols = ncol[nptr[k]:nptr[k + 1]]
            bad += int(np.any(x[cols] != q[cols]))
        truth = np.array([q[t["pb"][b]:t["pe"][b]].sum() for b in range(nb)])
        for b in np.flatnonzero(rel):
            for s in t["v_src"][t["v_ptr"][b]:t["v_ptr"][b + 1]]:
                bad += int(not np.isclose(mono[s], truth[s], rtol=1e-12, atol=1e-12))
        rows = np.arange(c0, c1, 7)
        y = _monopole_fmm(t, cent, centre, np.nan_to_num(x, nan=1e300), np.nan_to_num(mono, nan=1e300), rows)
        out = [None] * world
        dist.all_gather_object(out, (rank, c0, c1, bad, rows, y, len(sh), int(plan["let_roff"][-1]),
                                     int(plan["halo_roff"][-1])))
        if rank == 0:
            q_out.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_plans_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_plan_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m, cent, t, centre, lev, nptr, ncol, qq = _plan_problem()
    truth = np.array([qq[t["pb"][b]:t["pe"][b]].sum() for b in range(len(t["pb"]))])
    for (rank, c0, c1, bad, rows, y, nsh, nlet, nhalo) in out:
        print("rank", rank, "panels", c1 - c0, "shared", nsh, "LET recv", nlet, "halo recv", nhalo, "bad", bad)
        assert bad == 0
        assert nsh > 0 and nlet > 0 and nhalo > 0
        yref = _monopole_fmm(t, cent, centre, qq, truth, rows)
        assert np.allclose(y, yref, rtol=1e-12, atol=0)
