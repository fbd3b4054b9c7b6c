"""Run a few MVMs of a config (for ncu captures): python tools/prof_mvm.py [cfg] [iters] [leaf]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from inputs import meshes  # noqa: E402
from paper_2409_12375_b200 import xrl  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
leaf = int(sys.argv[3]) if len(sys.argv) > 3 else 64
m = meshes.make_config(cfg)
ctx = xrl.Context(0)
tree = xrl.Tree(ctx, m.verts, m.tris, leaf_max=leaf)
near = xrl.Near(tree)
x = tree.to_library_order(torch.from_numpy(meshes.make_x(cfg, m.n)).cuda())
y = torch.empty_like(x)
for _ in range(iters):
    xrl.mvm(tree, near, x, y)
torch.cuda.synchronize()
print("ok", tree.info())
