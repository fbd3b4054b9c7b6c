"""Which lists make the halo of x (config 4, 2-way partition): remote leaves read by the P2P (U lists of the
rank's own leaves) and by the P2L (X lists of its relevant boxes), counted in panels.
    python tools/halo_diag.py [cfg] [world] [leaf]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from inputs import meshes  # noqa: E402
from paper_2409_12375_b200 import xrl  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
leaf = int(sys.argv[3]) if len(sys.argv) > 3 else 384
m = meshes.make_config(cfg)
ctx = xrl.Context(0)
tr = xrl.Tree(ctx, m.verts, m.tris, leaf_max=leaf, part_rank=0, part_world=world)
ex = tr.export()
info = tr.info()
c0, c1 = info["offset"], info["offset"] + info["n_local"]
pb, pe, leafm, lev = ex["pb"], ex["pe"], ex["is_leaf"].astype(bool), ex["level"]
rel = (pb < c1) & (pe > c0)
own = (pb >= c0) & (pe <= c1)
def lst(k, b):
    return ex[k + "_src"][ex[k + "_ptr"][b]:ex[k + "_ptr"][b + 1]]
U, X = set(), set()
for b in np.nonzero(rel)[0]:
    for s in lst("x", b):
        if not own[s]:
            X.add(int(s))
    if leafm[b] and own[b]:
        for s in lst("u", b):
            if not own[s]:
                U.add(int(s))
sz = lambda S: int(sum(pe[s] - pb[s] for s in S))
print("rank 0 of", world, "owns", c1 - c0, "panels; leaves", int(leafm.sum()))
print("U-list remote leaves", len(U), "panels", sz(U), " levels", np.bincount(lev[list(U)]) if U else [])
print("X-list remote leaves", len(X), "panels", sz(X), " levels", np.bincount(lev[list(X)]) if X else [])
big = sorted(U, key=lambda s: -(pe[s] - pb[s]))[:10]
print("largest U leaves (level, size):", [(int(lev[s]), int(pe[s] - pb[s])) for s in big])
print("exchange_info", xrl.exchange_info(tr, xrl.Near(tr)))
# spatial picture: box ijk scaled to the finest level, for own leaves with remote U neighbours and the remote leaves
ijk, L = ex["ijk"], ex["level"]
def ctr(b):
    s = 2.0 ** -L[b]
    return (ijk[b] + 0.5) * s
bnd = [b for b in np.nonzero(leafm & own)[0] if any(not own[s] for s in lst("u", b))]
print("own leaves", int((leafm & own).sum()), "with remote U neighbours", len(bnd))
cb = np.array([ctr(b) for b in bnd]); cr = np.array([ctr(s) for s in U])
for nm, a in (("own boundary", cb), ("remote U", cr)):
    print(nm, "x range", a[:, 0].min().round(3), a[:, 0].max().round(3), "y range", a[:, 1].min().round(3),
          a[:, 1].max().round(3), "z range", a[:, 2].min().round(4), a[:, 2].max().round(4))
own_c = np.array([ctr(b) for b in np.nonzero(leafm & own)[0]])
print("own leaves y quantiles", np.quantile(own_c[:, 1], [0, .25, .5, .75, 1]).round(3), "x", np.quantile(own_c[:, 0], [0, .5, 1]).round(3))
