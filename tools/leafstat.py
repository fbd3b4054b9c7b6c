import sys, numpy as np
sys.path.insert(0, '.')
from inputs import meshes
from paper_2409_12375_b200 import xrl
m = meshes.make_config(4)
ctx = xrl.Context(0)
tree = xrl.Tree(ctx, m.verts, m.tris, leaf_max=352)
ex = tree.export()
leaves = np.nonzero(ex["is_leaf"])[0]
T = (ex["pe"] - ex["pb"])
up, us = ex["u_ptr"], ex["u_src"]
src = np.array([T[us[up[b]:up[b+1]]].sum() for b in leaves])
Tl = T[leaves]
work = Tl * src
tot = work.sum()
for lo, hi in [(0,8),(8,16),(16,32),(32,64),(64,128),(128,256),(256,400)]:
    sel = (Tl > lo) & (Tl <= hi)
    print(f"T in ({lo},{hi}]: leaves {sel.sum():6d}  work share {work[sel].sum()/tot:6.3f}  mean sources {src[sel].mean() if sel.any() else 0:8.0f}")
print("total pairs", tot)
