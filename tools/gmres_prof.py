"""A few GMRES iterations on config 4 (for an ncu launch list of the loop-space kernels).
    python tools/gmres_prof.py [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from inputs import meshes  # noqa: E402
from paper_2409_12375_b200 import xrl  # noqa: E402

it = int(sys.argv[1]) if len(sys.argv) > 1 else 5
m = meshes.make_config(4)
ctx = xrl.Context(0)
tree = xrl.Tree(ctx, m.verts, m.tris, leaf_max=384)
near = xrl.Near(tree)
topo = xrl.Topology(tree, [])
op = xrl.Operator(tree, near, topo, 1e9, sigma=5.8e7, zeta=10e-6)
pc = xrl.Precond(op, 64)
rng = np.random.default_rng(1404)
nl = topo.n_loops
b = torch.from_numpy((rng.random((1, nl)) - 0.5 + 1j * (rng.random((1, nl)) - 0.5)).astype(np.complex64)).cuda()
xrl.gmres(op, pc, b, max_iters=it, tol=1e-30)
torch.cuda.synchronize()
print("ok")
