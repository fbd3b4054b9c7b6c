"""Parity of the CUDA path at BASELINE.json's full sizes (configs 2-5), through the C-ABI, against the
FP64 oracle on sampled rows (S = 4096 rows, seed 7; config 2 in full).

  * the full MVM (<= 2e-5 relative L2, BASELINE north star) at the bench's launch configuration;
  * the near-field SpMV alone (XRL_MVM_NEAR_ONLY) against the oracle's near rows (<= 1e-6);
  * the near pattern bit for bit and the FP64 near values to 1e-11 on sampled rows, and the tie audit
    (no pair within 1e-9 of the eta threshold, C3) on the same rows;
  * the Morton order of the library permutation, recomputed here from the FP64 centroids;
  * a leaf larger than 32,767 panels (the P2P task encoding)."""
import numpy as np
import pytest

import oracle
from inputs import meshes
from tests.gpu_helpers import cuda_setup, oracle_rows, run_mvm

pytestmark = pytest.mark.gpu

TOL_FULL = 2e-5
TOL_NEAR = 1e-6
S_ROWS = 4096
BENCH_LEAF = 384  # bench.py's launch configuration (leaf_max)

_cache = {}


def _setup(cfg, leaf):
    """One tree/near per (cfg, leaf) for the module (cfg 5 takes ~10 s to build)."""
    key = (cfg, leaf)
    if key not in _cache:
        for k in list(_cache):  # keep one large mesh resident at a time
            if k[0] != cfg:
                del _cache[k]
        m = meshes.make_config(cfg)
        ctx, tree, near = cuda_setup(m, leaf_max=leaf)
        _cache[key] = (m, ctx, tree, near, oracle.Geometry(m.verts, m.tris))
    return _cache[key]


def _rows(n):
    return np.sort(np.random.default_rng(7).choice(n, size=min(S_ROWS, n), replace=False))


@pytest.mark.parametrize("cfg,leaf", [(3, BENCH_LEAF), (3, 64), (4, BENCH_LEAF), (4, 64), (5, BENCH_LEAF)])
def test_full_mvm_4096_rows(cfg, leaf):
    m, ctx, tree, near, g = _setup(cfg, leaf)
    x = meshes.make_x(cfg, m.n)
    y = run_mvm(tree, near, x)
    rows = _rows(m.n)
    yref = oracle.mvm_rows(g, x, rows)
    err = oracle.rel_l2(y[:, rows], yref)
    per = [oracle.rel_l2(y[t, rows], yref[t]) for t in range(3)]
    rowmax = float(np.max(np.abs(y[:, rows] - yref)) / np.max(np.abs(yref)))
    print(f"cfg{cfg} leaf {leaf} rows {rows.size}: rel L2 {err:.3e} per-comp {per} max-row {rowmax:.3e}")
    assert err <= TOL_FULL


def test_full_mvm_config2_every_row():
    """Config 2 (131,072 panels) against the oracle's full O(N^2) direct sum (1.7e10 pairs)."""
    m, ctx, tree, near, g = _setup(2, BENCH_LEAF)
    x = meshes.make_x(2, m.n)
    y = run_mvm(tree, near, x)
    yref = oracle.mvm_rows(g, x)
    err = oracle.rel_l2(y, yref)
    print("cfg2 full rel L2", err, [oracle.rel_l2(y[t], yref[t]) for t in range(3)])
    assert err <= TOL_FULL


def _near_ref(g, x, rows):
    """Oracle near-only product on `rows`: sum_l (P_kl - 1/r_kl) x_l + P_kk x_k (C4 correction term)."""
    optr, ocol, oval, oinv_r = oracle.near_rows(g, rows)
    corr = oval - oinv_r
    yref = np.zeros((x.shape[0], rows.size), dtype=np.complex128)
    ri = np.repeat(np.arange(rows.size), np.diff(optr))
    for v in range(x.shape[0]):
        np.add.at(yref[v], ri, corr * x[v, ocol].astype(np.complex128))
    return yref, (optr, ocol, oval)


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_near_spmv_pattern_and_ties_sampled(cfg):
    """Near-only SpMV <= 1e-6 vs the oracle's CSR x on 4096 sampled rows; the same rows' GPU pattern equals
    the oracle's bit for bit, FP64 values to 1e-11, and the tie audit of those rows is 0."""
    m, ctx, tree, near, g = _setup(cfg, BENCH_LEAF)
    x = meshes.make_x(cfg, m.n)
    rows = _rows(m.n)
    y = run_mvm(tree, near, x, flags=1)
    yref, (optr, ocol, oval) = _near_ref(g, x, rows)
    err = oracle.rel_l2(y[:, rows], yref)
    nnz_row = np.diff(optr).mean()
    print(f"cfg{cfg} near-only rel L2 {err:.3e} ({nnz_row:.1f} nnz/row on the sample)")
    assert err <= TOL_NEAR
    # pattern and values, library order -> mesh order
    perm = tree.perm()
    iperm = np.empty_like(perm)
    iperm[perm] = np.arange(m.n, dtype=perm.dtype)
    ptr, col, v32, v64 = near.export_rows(iperm[rows])
    for i, k in enumerate(rows):
        gc = perm[col[ptr[i]:ptr[i + 1]]]
        order = np.argsort(gc)
        oc = ocol[optr[i]:optr[i + 1]]
        assert np.array_equal(gc[order], oc), (cfg, k)
        # FP64 to 1e-11: the GPU integrals are FMA-contracted, the oracle is -ffp-contract=off, and the
        # log/atan edge terms cancel for separated pairs (observed <= 1.24e-12; FP32 storage is 6e-8)
        np.testing.assert_allclose(v64[ptr[i]:ptr[i + 1]][order], oval[optr[i]:optr[i + 1]], rtol=1e-11)
    assert oracle.tie_audit_rows(g, rows) == 0


@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_permutation_is_stable_morton_sort(cfg):
    """The library order is the stable sort of the 63-bit Morton keys of the FP64 centroids (K2/K3): the
    keys are recomputed here from the oracle's centroids and the tree's root cube -- q_d =
    floor((c_d - lo_d) (1/W) 2^21) clamped to [0, 2^21 - 1], bits interleaved x, y, z from the lowest --
    and must be non-decreasing along perm, with equal keys in ascending original index."""
    m = meshes.make_config(cfg)
    ctx, tree, near = cuda_setup(m, leaf_max=BENCH_LEAF)
    g = oracle.Geometry(m.verts, m.tris)
    info = tree.info()
    lo = np.array(info["root_lo"])
    invW = 1.0 / info["root_width"]
    q = np.floor((g.cent - lo) * invW * float(1 << 21)).astype(np.int64)
    q = np.clip(q, 0, (1 << 21) - 1).astype(np.uint64)
    key = np.zeros(m.n, dtype=np.uint64)
    for bit in range(21):
        for d in range(3):
            key |= ((q[:, d] >> np.uint64(bit)) & np.uint64(1)) << np.uint64(3 * bit + d)
    perm = tree.perm()
    assert np.array_equal(np.sort(perm), np.arange(m.n))
    kp = key[perm]
    assert np.all(kp[1:] >= kp[:-1])
    tie = kp[1:] == kp[:-1]
    assert np.all(perm[1:][tie] > perm[:-1][tie])
    # and it is exactly numpy's stable argsort of the keys
    assert np.array_equal(perm, np.argsort(key, kind="stable"))


def test_leaf_above_32767_panels():
    """a leaf with more than 32,767 targets (config 3 with leaf_max above N: one leaf of all
    508,928 panels, no far field) -- the P2P tasks carry the first target as an absolute index, so every
    target is written."""
    from paper_2409_12375_b200 import xrl
    m = meshes.make_config(3)
    ctx = xrl.Context(0)
    tree = xrl.Tree(ctx, m.verts, m.tris, leaf_max=1 << 20, max_depth=1)
    near = xrl.Near(tree)
    ex = tree.export()
    leaves = np.nonzero(ex["is_leaf"])[0]
    assert (ex["pe"][leaves] - ex["pb"][leaves]).max() > 32767
    x = meshes.make_x(3, m.n)
    y = run_mvm(tree, near, x)
    rows = np.random.default_rng(7).choice(m.n, size=512, replace=False)
    g = oracle.Geometry(m.verts, m.tris)
    err = oracle.rel_l2(y[:, rows], oracle.mvm_rows(g, x, rows))
    print("max_depth 1 leaves", ex["pe"][leaves] - ex["pb"][leaves], err)
    assert err <= TOL_FULL


def _ctx_tree(cfg, leaf, env):
    """A fresh context/tree/near with environment switches read at context creation (XRL_M2L_TF32)."""
    import os
    from paper_2409_12375_b200 import xrl
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        m = meshes.make_config(cfg)
        ctx = xrl.Context(0)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    tree = xrl.Tree(ctx, m.verts, m.tris, leaf_max=leaf)
    return m, ctx, tree, xrl.Near(tree)


def test_m2l_fp16_matches_tf32():
    """The default 3xFP16 M2L (scaled operands) and the 3xTF32 one agree to FP32 rounding of the far field
    (both keep 22 significand bits per product)."""
    m, _, t16, n16 = _ctx_tree(3, 64, {"XRL_M2L_TF32": "0"})
    _, _, t32, n32 = _ctx_tree(3, 64, {"XRL_M2L_TF32": "1"})
    x = meshes.make_x(3, m.n)
    y16 = run_mvm(t16, n16, x, flags=2)  # XRL_MVM_FAR_ONLY: the FMM part alone
    y32 = run_mvm(t32, n32, x, flags=2)
    d = oracle.rel_l2(y16, y32)
    print("far-only rel L2 fp16 vs tf32 M2L:", d)
    assert d <= 1e-6


def test_m2l_fp16_skewed_charges():
    """Charges spanning 16 decades across the mesh (one power-of-2 scale for all multipoles of the MVM):
    the MVM stays within the north-star bound of the oracle on sampled rows."""
    m, ctx, tree, near, g = _setup(3, BENCH_LEAF)
    x = meshes.make_x(3, m.n)
    z = m.verts[m.tris].mean(axis=1)[:, 2]
    s = 10.0 ** (-16.0 * (z - z.min()) / max(z.max() - z.min(), 1e-30))
    x = (x * s[None, :]).astype(np.complex64)
    y = run_mvm(tree, near, x)
    rows = _rows(m.n)
    yref = oracle.mvm_rows(g, x, rows)
    err = oracle.rel_l2(y[:, rows], yref)
    print("skewed charges rel L2", err)
    assert err <= TOL_FULL
