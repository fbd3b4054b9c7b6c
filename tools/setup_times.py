"""Setup wall times of the tree and near-field builds (XRL_SETUP_TIMES=1 prints the tree's sections).
    XRL_SETUP_TIMES=1 python tools/setup_times.py [cfg] [leaf]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from inputs import meshes  # noqa: E402
from paper_2409_12375_b200 import xrl  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
leaf = int(sys.argv[2]) if len(sys.argv) > 2 else 384
t0 = time.perf_counter()
m = meshes.make_config(cfg)
t1 = time.perf_counter()
ctx = xrl.Context(0)
torch.cuda.synchronize()
t2 = time.perf_counter()
for rep in range(2):
    t3 = time.perf_counter()
    tree = xrl.Tree(ctx, m.verts, m.tris, leaf_max=leaf)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    near = xrl.Near(tree)
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(f"rep {rep}: mesh {t1 - t0:.2f} s, context {t2 - t1:.2f} s, tree {t4 - t3:.3f} s, near {t5 - t4:.3f} s", flush=True)
    del near, tree
