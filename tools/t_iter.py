"""GMRES iteration time t_iter (operator + preconditioner apply + orthogonalisation per
step) on configs 1, 2 and 4 at 1 GHz with one random loop RHS (seed 1404): block-Jacobi and exact Q^-1."""
import os
import sys
import time
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from inputs import meshes  # noqa: E402
from paper_2409_12375_b200 import xrl  # noqa: E402

ctx = xrl.Context(0)
for cfg, leaf in ((1, 64), (2, 128), (4, 352)):
    m = meshes.make_config(cfg)
    tree = xrl.Tree(ctx, m.verts, m.tris, leaf_max=leaf)
    near = xrl.Near(tree)
    topo = xrl.Topology(tree, [])
    op = xrl.Operator(tree, near, topo, 1e9, sigma=5.8e7, zeta=10e-6)
    nl = topo.n_loops
    rng = np.random.default_rng(1404)
    b = torch.from_numpy((rng.random((1, nl)) - 0.5 + 1j * (rng.random((1, nl)) - 0.5)).astype(np.complex64)).cuda()
    for kind in ("block", "exact"):
        t0 = time.perf_counter()
        pc = xrl.Precond(op, 64, exact=(kind == "exact"))
        torch.cuda.synchronize()
        setup = time.perf_counter() - t0
        xrl.gmres(op, pc, b, max_iters=2, tol=1e-30)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, rep = xrl.gmres(op, pc, b, max_iters=40, restart=50, tol=1e-30)
        e1.record()
        torch.cuda.synchronize()
        it = int(rep["iters"][0])
        print(f"cfg {cfg} panels {m.n} loops {nl} {kind:5s} precond setup {setup:.2f}s  t_iter "
              f"{e0.elapsed_time(e1) / max(it, 1):.2f} ms over {it} iterations", flush=True)
