"""Component-wise accuracy diagnosis on config 4 sampled rows (test infrastructure: GPU path vs the oracle).
    python tests/diag_cfg4.py [cfg] [leaf]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from inputs import meshes
from tests.gpu_helpers import cuda_setup, run_mvm
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
leaf = int(sys.argv[2]) if len(sys.argv) > 2 else 64
m = meshes.make_config(cfg)
ctx, tree, near = cuda_setup(m, leaf_max=leaf)
x = meshes.make_x(cfg, m.n)
rows = np.random.default_rng(7).choice(m.n, size=256, replace=False)
g = oracle.Geometry(m.verts, m.tris)
yfull = run_mvm(tree, near, x)
ynear = run_mvm(tree, near, x, flags=1)
yfar = run_mvm(tree, near, x, flags=2)
ref = oracle.mvm_rows(g, x, rows)
ptr, cols, vals, inv_r = oracle.near_rows(g, rows)
rr = np.repeat(np.arange(len(rows)), np.diff(ptr))
corr = vals - inv_r
nref = np.zeros((3, len(rows)), complex)
for v in range(3):
    np.add.at(nref[v], rr, corr * x[v, cols].astype(complex))
c = g.cent
far = np.zeros((3, len(rows)), complex)
xc = x.astype(complex)
for i, k in enumerate(rows):
    d = np.linalg.norm(c - c[k], axis=1); d[k] = np.inf
    far[:, i] = (xc / d).sum(axis=1)
print("full", oracle.rel_l2(yfull[:, rows], ref))
print("near-only", oracle.rel_l2(ynear[:, rows], nref))
print("far-only", oracle.rel_l2(yfar[:, rows], far))
print("consistency ref - (near+far)", oracle.rel_l2(nref + far, ref))
e = np.abs(yfar[:, rows] - far).sum(axis=0) / np.abs(far).sum(axis=0)
worst = np.argsort(e)[-5:]
print("worst far rows", rows[worst], e[worst])
print(tree.info())
