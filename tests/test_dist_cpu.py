"""Multi-rank path on CPU (gloo, world size 2): the partition rule the library
uses (xrl_partition_cuts, a host function) and the sharded data flow of the
MVM -- gather the owned slices of x, apply the owned rows of P, concatenate
-- emulated with the oracle's dense P.  The GPU kernels of the restricted
passes are checked on one GPU by test_virtual_partition_concat_equals_full."""
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


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from inputs import meshes
        from paper_2409_12375_b200 import xrl
        m = meshes.small_mesh("cube", n=3)  # 108 panels
        g = oracle.Geometry(m.verts, m.tris)
        P = oracle.dense_p(g)
        rng = np.random.default_rng(0)
        w = rng.random(m.n) + 0.5           # per-item work (same on every rank)
        cuts = xrl.partition_cuts(w, world)
        lo, hi = int(cuts[rank]), int(cuts[rank + 1])
        x = meshes.make_x(1, m.n)
        xs = torch.from_numpy(x[:, lo:hi].copy())
        # gather variable-size slices: broadcast each rank's slice (as the NCCL group does)
        full = torch.zeros((3, m.n), dtype=torch.complex64)
        for r in range(world):
            a, b = int(cuts[r]), int(cuts[r + 1])
            buf = xs.clone() if r == rank else torch.zeros((3, b - a), dtype=torch.complex64)
            buf = torch.view_as_real(buf).contiguous()
            dist.broadcast(buf, r)
            full[:, a:b] = torch.view_as_complex(buf)
        y_local = (P[lo:hi] @ full.numpy().astype(np.complex128).T).T
        out = [None] * world
        dist.all_gather_object(out, (lo, hi, y_local, float(w[lo:hi].sum())))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def test_partition_cuts_rule():
    from paper_2409_12375_b200 import xrl
    w = np.array([1, 1, 1, 1, 10, 1, 1, 1], float)
    c = xrl.partition_cuts(w, 2)
    assert c[0] == 0 and c[-1] == len(w) and np.all(np.diff(c) >= 0)
    assert c[1] in (4, 5)
    c = xrl.partition_cuts(np.ones(10), 3)
    assert list(np.diff(c)) in ([3, 4, 3], [4, 3, 3], [3, 3, 4])
    assert list(xrl.partition_cuts(np.ones(2), 4)[[0, -1]]) == [0, 2]


def test_sharded_mvm_dataflow_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import oracle
    from inputs import meshes
    m = meshes.small_mesh("cube", n=3)
    g = oracle.Geometry(m.verts, m.tris)
    P = oracle.dense_p(g)
    x = meshes.make_x(1, m.n).astype(np.complex128)
    yref = (P @ x.T).T
    ys = sorted(out, key=lambda t: t[0])
    assert ys[0][0] == 0 and ys[-1][1] == m.n
    assert all(ys[i][1] == ys[i + 1][0] for i in range(world - 1))
    y = np.concatenate([t[2] for t in ys], axis=1)
    assert np.abs(y - yref).max() <= 1e-6 * np.abs(yref).max()
    works = [t[3] for t in ys]
    assert max(works) / min(works) < 1.2
