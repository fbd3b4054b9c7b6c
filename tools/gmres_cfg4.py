"""Config 4 GMRES convergence probe: exact Q^-1 vs right block-Jacobi, random loop RHS (seed 1404)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from inputs import meshes  # noqa: E402
from paper_2409_12375_b200 import xrl  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 300
m = meshes.make_config(cfg)
ctx = xrl.Context(0)
tree = xrl.Tree(ctx, m.verts, m.tris, leaf_max=512)
near = xrl.Near(tree)
topo = xrl.Topology(tree, [])
nl = topo.n_loops
print("config", cfg, "panels", tree.info()["n"], "loops", nl, flush=True)
rng = np.random.default_rng(1404)
b = torch.from_numpy((rng.random((1, nl)) - 0.5 + 1j * (rng.random((1, nl)) - 0.5)).astype(np.complex64)).cuda()
for f in [1e9]:
    op = xrl.Operator(tree, near, topo, f, sigma=5.8e7, zeta=10e-6)
    for mode in ["exact", "right"]:
        t0 = time.time()
        pc = None if mode == "none" else xrl.Precond(op, 64, exact=(mode == "exact"))
        torch.cuda.synchronize()
        print(f"f={f:g} {mode} preconditioner setup {time.time() - t0:.1f}s", flush=True)
        for restart in [50]:
            t0 = time.time()
            x, rep = xrl.gmres(op, pc, b, max_iters=iters, restart=restart, right=(mode != "left"))
            torch.cuda.synchronize()
            print(f"f={f:g} {mode:5s} restart={restart} iters={rep['iters'][0]} rre={rep['rre'][0]:.3e} "
                  f"true_rre={rep['true_rre'][0]:.3e} {time.time() - t0:.1f}s", flush=True)
