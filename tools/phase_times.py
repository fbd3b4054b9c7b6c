"""Isolated per-phase times (serial schedule, CUDA events per phase) of a config's MVM:
    python tools/phase_times.py [cfg] [leaf] [iters]   -> one JSON line {phase: ms per launch}"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from inputs import meshes  # noqa: E402
from paper_2409_12375_b200 import xrl  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
leaf = int(sys.argv[2]) if len(sys.argv) > 2 else 384
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 10
m = meshes.make_config(cfg)
ctx = xrl.Context(0)
tree = xrl.Tree(ctx, m.verts, m.tris, leaf_max=leaf)
near = xrl.Near(tree)
x = tree.to_library_order(torch.from_numpy(meshes.make_x(cfg, m.n)).cuda())
y = torch.empty_like(x)
ctx.set_sched(ctx.SCHED_SERIAL)
for _ in range(3):
    xrl.mvm(tree, near, x, y)
torch.cuda.synchronize()
ctx.timing_reset()
ctx.timing_enable(True)
for _ in range(iters):
    xrl.mvm(tree, near, x, y)
torch.cuda.synchronize()
ctx.timing_enable(False)
ph = ctx.timing()
print(json.dumps({"tag": os.environ.get("TAG", ""), **{k: round(v[0] / max(v[1], 1), 4) for k, v in ph.items()}}))
