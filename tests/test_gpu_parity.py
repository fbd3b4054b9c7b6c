"""Parity of the CUDA path (through the C-ABI) against the FP64 oracle.

Tolerances (BASELINE.json north star): full MVM relative L2 <= 2e-5 at p = 10
over all 3 complex components jointly; near-field SpMV alone <= 1e-6.  Index
work (near pattern, permutation, list coverage) is compared bit for bit."""
import numpy as np
import pytest

import oracle
from inputs import meshes
from tests.gpu_helpers import cuda_setup, oracle_rows, run_mvm

pytestmark = pytest.mark.gpu

TOL_FULL = 2e-5
TOL_NEAR = 1e-6


@pytest.fixture(scope="module")
def bar_setup():
    m = meshes.bar()
    ctx, tree, near = cuda_setup(m)
    return m, ctx, tree, near


def test_permutation_and_info(bar_setup):
    """perm is a permutation (the Morton order itself is checked in test_gpu_fullsize.py)."""
    m, ctx, tree, near = bar_setup
    perm = tree.perm()
    assert np.array_equal(np.sort(perm), np.arange(m.n))
    info = tree.info()
    assert info["n"] == m.n and info["p"] == 10


def _coverage(ex, n):
    """For every leaf, count how often each source panel is covered by
    U (P2P), W (M2P) and V/X of the leaf and all its ancestors."""
    nb = ex["level"].shape[0]
    par = ex["parent"]
    pb, pe = ex["pb"], ex["pe"]
    def panels(b):
        return np.arange(pb[b], pe[b])
    bad = 0
    for b in np.nonzero(ex["is_leaf"])[0]:
        cnt = np.zeros(n, dtype=np.int32)
        for s in ex["u_src"][ex["u_ptr"][b]:ex["u_ptr"][b + 1]]:
            cnt[panels(s)] += 1
        for w in ex["w_src"][ex["w_ptr"][b]:ex["w_ptr"][b + 1]]:
            cnt[panels(w)] += 1
        a = b
        while a >= 0:
            for s in ex["v_src"][ex["v_ptr"][a]:ex["v_ptr"][a + 1]]:
                cnt[panels(s)] += 1
            for s in ex["x_src"][ex["x_ptr"][a]:ex["x_ptr"][a + 1]]:
                cnt[panels(s)] += 1
            a = par[a]
        bad += int(np.sum(cnt != 1))
    return bad


@pytest.mark.parametrize("kind", ["bar", "bga2", "clustered"])
def test_tree_lists_cover_every_pair_once(kind):
    """SPEC.md:381 coverage audit: near + far lists cover all N^2 ordered
    panel pairs exactly once (adaptive U/V/W/X lists)."""
    if kind == "bar":
        m = meshes.bar()
        lm = 16
    elif kind == "bga2":
        m = meshes.bga(nb=2)
        lm = 24
    else:
        # two dense clusters + sparse background: exercises W/X lists
        rng = np.random.default_rng(3)
        parts = []
        for c, s, k in (((0, 0, 0), 1e-5, 300), ((3e-4, 1e-4, 0), 1e-5, 300), ((1e-4, 2e-4, 1e-4), 3e-4, 200)):
            v = rng.normal(size=(3 * k, 3)) * s + np.array(c)
            parts.append(v)
        v = np.concatenate(parts)
        m = meshes.Mesh(v, np.arange(v.shape[0], dtype=np.int32).reshape(-1, 3))
        lm = 8
    ctx, tree, near = cuda_setup(m, leaf_max=lm)
    ex = tree.export()
    info = tree.info()
    assert info["n_levels"] >= 3
    # leaves partition the panels, leaves respect leaf_max (depth cap not reached here)
    leaves = np.nonzero(ex["is_leaf"])[0]
    sizes = ex["pe"][leaves] - ex["pb"][leaves]
    assert sizes.sum() == m.n and sizes.max() <= lm
    assert _coverage(ex, m.n) == 0
    print(kind, {k: info[k] for k in ("n_u_pairs", "n_v_pairs", "n_x_pairs", "n_w_pairs")})


def _clustered_mesh():
    rng = np.random.default_rng(3)
    parts = []
    for c, s, k in (((0, 0, 0), 1e-5, 300), ((3e-4, 1e-4, 0), 1e-5, 300), ((1e-4, 2e-4, 1e-4), 3e-4, 200)):
        parts.append(rng.normal(size=(3 * k, 3)) * s + np.array(c))
    v = np.concatenate(parts)
    return meshes.Mesh(v, np.arange(v.shape[0], dtype=np.int32).reshape(-1, 3))


@pytest.mark.parametrize("leaf_max", [4, 8, 16])
def test_adaptive_lists_parity(leaf_max):
    """Strongly non-uniform point set with small leaves: exercises kept
    P2L/M2P pairs and X/W pairs converted to direct P2P (incl. non-leaf W
    boxes expanded into their leaves)."""
    m = _clustered_mesh()
    ctx, tree, near = cuda_setup(m, leaf_max=leaf_max)
    x = meshes.make_x(2, m.n)
    err = oracle.rel_l2(run_mvm(tree, near, x), oracle_rows(m, x))
    print("clustered leaf", leaf_max, err, tree.info())
    assert err <= TOL_FULL


def test_near_pattern_and_values_match_oracle(bar_setup):
    m, ctx, tree, near = bar_setup
    perm = tree.perm()
    ptr, col, v32, v64 = near.export()
    g = oracle.Geometry(m.verts, m.tris)
    optr, ocol, oval, oinv_r = oracle.near_rows(g)
    # map GPU rows/cols (library order) to mesh order
    for i in range(m.n):
        k = perm[i]
        gc = np.sort(perm[col[ptr[i]:ptr[i + 1]]])
        oc = ocol[optr[k]:optr[k + 1]]
        assert np.array_equal(gc, oc), i
    # values: FP64 near entries agree to rounding; FP32 correction = P - 1/r
    rows_lib = np.repeat(np.arange(m.n), np.diff(ptr))
    k_m = perm[rows_lib]
    l_m = perm[col]
    P = oracle.dense_p(g)
    np.testing.assert_allclose(v64, P[k_m, l_m], rtol=1e-12)
    d = np.linalg.norm(g.cent[k_m] - g.cent[l_m], axis=1)
    corr = np.where(k_m == l_m, P[k_m, l_m], P[k_m, l_m] - 1.0 / np.where(d > 0, d, 1))
    np.testing.assert_allclose(v32, corr, rtol=2e-7, atol=1e-7 * np.abs(P).max())


def test_near_only_spmv(bar_setup):
    m, ctx, tree, near = bar_setup
    x = meshes.make_x(1, m.n)
    y = run_mvm(tree, near, x, flags=1)
    g = oracle.Geometry(m.verts, m.tris)
    optr, ocol, oval, oinv_r = oracle.near_rows(g)
    rows = np.repeat(np.arange(m.n), np.diff(optr))
    corr = oval - oinv_r
    yref = np.zeros((3, m.n), dtype=np.complex128)
    for v in range(3):
        np.add.at(yref[v], rows, corr * x[v, ocol].astype(np.complex128))
    err = oracle.rel_l2(y, yref)
    print("near-only rel L2", err)
    assert err <= TOL_NEAR


def test_full_mvm_config1(bar_setup):
    m, ctx, tree, near = bar_setup
    x = meshes.make_x(1, m.n)
    y = run_mvm(tree, near, x)
    yref = oracle_rows(m, x)
    err = oracle.rel_l2(y, yref)
    print("cfg1 full rel L2", err)
    assert err <= TOL_FULL


def test_far_only_vs_direct_inverse_r(bar_setup):
    m, ctx, tree, near = bar_setup
    x = meshes.make_x(1, m.n)
    y = run_mvm(tree, near, x, flags=2)
    c = m.verts[m.tris].mean(axis=1)
    d = np.linalg.norm(c[:, None] - c[None], axis=2)
    np.fill_diagonal(d, np.inf)
    yref = (1.0 / d) @ x.astype(np.complex128).T
    err = oracle.rel_l2(y, yref.T)
    print("far-only rel L2", err)
    assert err <= TOL_FULL


def test_special_cases(bar_setup):
    m, ctx, tree, near = bar_setup
    x = np.zeros((3, m.n), dtype=np.complex64)
    assert np.all(run_mvm(tree, near, x) == 0)
    x = meshes.make_x(1, m.n)
    y1 = run_mvm(tree, near, x)
    y2 = run_mvm(tree, near, (2 * x).astype(np.complex64))
    assert np.allclose(y2, 2 * y1, rtol=1e-6, atol=1e-6 * np.abs(y1).max())
    # two triples in one call == two calls
    # (M2L accumulates with atomics: results agree to FP32 rounding, not bitwise)
    x6 = np.concatenate([x, x[::-1].copy()])
    y6 = run_mvm(tree, near, x6)
    assert oracle.rel_l2(y6[:3], y1) < 1e-6
    assert oracle.rel_l2(y6[3:], run_mvm(tree, near, x[::-1].copy())) < 1e-6


def test_single_leaf_exact():
    """N <= leaf_max: no multipoles, y = P2P + CSR."""
    m = meshes.small_mesh("cube", n=2)  # 48 panels
    ctx, tree, near = cuda_setup(m, leaf_max=64)
    assert tree.info()["n_levels"] == 1
    x = meshes.make_x(1, m.n)
    y = run_mvm(tree, near, x)
    yref = oracle_rows(m, x)
    assert oracle.rel_l2(y, yref) < 1e-6


@pytest.mark.parametrize("leaf_max", [8, 30, 200])
def test_leaf_sizes_ragged(leaf_max):
    m = meshes.bar()
    ctx, tree, near = cuda_setup(m, leaf_max=leaf_max)
    x = meshes.make_x(1, m.n)
    y = run_mvm(tree, near, x)
    err = oracle.rel_l2(y, oracle_rows(m, x))
    print("leaf", leaf_max, err)
    assert err <= TOL_FULL


def test_host_api_e2e(bar_setup):
    from paper_2409_12375_b200 import xrl
    m, ctx, tree, near = bar_setup
    x = meshes.make_x(1, m.n)
    y_dev = run_mvm(tree, near, x)
    y_host = xrl.mvm_host(tree, near, x)
    assert oracle.rel_l2(y_host, y_dev) < 1e-6


@pytest.mark.parametrize("cfg,nrows,leaf", [(2, 1024, 64), (4, 256, 512)])
def test_full_mvm_sampled_rows(cfg, nrows, leaf):
    """Other leaf sizes on sampled rows (the 4096-row and full config-2 checks at the bench's leaf (384) are
    in test_gpu_fullsize.py)."""
    m = meshes.make_config(cfg)
    ctx, tree, near = cuda_setup(m, leaf_max=leaf)
    x = meshes.make_x(cfg, m.n)
    y = run_mvm(tree, near, x)
    rows = np.random.default_rng(7).choice(m.n, size=nrows, replace=False)
    yref = oracle_rows(m, x, rows)
    err = oracle.rel_l2(y[:, rows], yref)
    print(f"cfg{cfg} sampled rel L2", err, tree.info())
    assert err <= TOL_FULL


@pytest.mark.parametrize("cfg,world,leaf", [(1, 2, 64), (1, 3, 16), (2, 4, 64), (2, 8, 384), (3, 8, 384)])
def test_virtual_ranks_equal_single_gpu(cfg, world, leaf):
    """Sharded MVM on one GPU through xrl_mvm_vranks: k trees partitioned 0..k-1, each with
    its own charges only; the halo of x, the shared-box multipole all-reduce and the LET exchange run as
    device copies between the trees.  The concatenated rank slices equal the single-GPU MVM to 1e-6 (FP32
    summation order) and the oracle on sampled rows; every exchange list is non-trivial for k > 1."""
    import torch
    from paper_2409_12375_b200 import xrl
    m = meshes.make_config(cfg)
    ctx, tree, near = cuda_setup(m, leaf_max=leaf)
    x = meshes.make_x(cfg, m.n)
    xl = tree.to_library_order(torch.from_numpy(x).cuda())
    y_full = xrl.mvm(tree, near, xl).cpu().numpy()
    trees, nears, xs, off = [], [], [], 0
    for r in range(world):
        tr = xrl.Tree(ctx, m.verts, m.tris, leaf_max=leaf, part_rank=r, part_world=world)
        trees.append(tr)
        nears.append(xrl.Near(tr))
        assert tr.offset == off and tr.n_local > 0
        xs.append(xl[:, off:off + tr.n_local].contiguous())
        off += tr.n_local
    assert off == m.n
    ys, rank_ms, exch_ms = xrl.mvm_vranks(trees, nears, xs, timing=True)
    y_cat = torch.cat(ys, dim=1).cpu().numpy()
    err = oracle.rel_l2(y_cat, y_full)
    info = [xrl.exchange_info(t, n) for t, n in zip(trees, nears)]
    print("virtual ranks", cfg, world, err, [t.n_local for t in trees], info, rank_ms, exch_ms)
    assert err < 1e-6
    assert sum(i["halo_send"] for i in info) == sum(i["halo_recv"] for i in info) > 0
    if m.n > 10000:
        assert sum(i["let_send"] for i in info) == sum(i["let_recv"] for i in info) > 0
        assert info[0]["shared"] > 0
        rows = np.random.default_rng(7).choice(m.n, size=256, replace=False)
        perm = tree.perm()
        y_user = np.empty_like(y_cat)
        y_user[:, perm] = y_cat
        assert oracle.rel_l2(y_user[:, rows], oracle_rows(m, x, rows)) <= TOL_FULL
    assert np.all(rank_ms > 0)
    # the other flags go through the same exchanges
    yn = torch.cat(xrl.mvm_vranks(trees, nears, xs, flags=1), dim=1).cpu().numpy()
    assert oracle.rel_l2(yn, xrl.mvm(tree, near, xl, flags=1).cpu().numpy()) < 1e-6


# ---------------------------------------------------------------- NEXT f4: hybrid meshes, Galerkin near rule

def _near_vs_oracle(m, tree, near, galerkin):
    perm = tree.perm()
    ptr, col, v32, v64 = near.export()
    g = oracle.Geometry(m.verts, m.tris, galerkin=galerkin)
    optr, ocol, oval, _ = oracle.near_rows(g)
    for i in range(m.n):
        k = perm[i]
        order = np.argsort(perm[col[ptr[i]:ptr[i + 1]]])
        assert np.array_equal(perm[col[ptr[i]:ptr[i + 1]]][order], ocol[optr[k]:optr[k + 1]]), i
        np.testing.assert_allclose(v64[ptr[i]:ptr[i + 1]][order], oval[optr[k]:optr[k + 1]], rtol=1e-12)


@pytest.mark.parametrize("galerkin", [False, True])
def test_hybrid_mesh_near_and_full_mvm(galerkin):
    """Hybrid bar (1,000 rectangles + 100 triangles, xrl_tree_build_poly): near pattern bit for bit and
    FP64 near values to 1e-12 against the oracle, full MVM within the north-star tolerance; with the
    Galerkin near rule as well."""
    m = meshes.bar_hybrid()
    ctx, tree, near = cuda_setup(m, galerkin=galerkin)
    _near_vs_oracle(m, tree, near, galerkin)
    x = meshes.make_x(1, m.n)
    err = oracle.rel_l2(run_mvm(tree, near, x), oracle_rows(m, x, galerkin=galerkin))
    print("hybrid galerkin", galerkin, "full", err)
    assert err <= TOL_FULL


def test_galerkin_near_rule_triangle_mesh(bar_setup):
    """The Galerkin rule on the triangle bar: near values match the oracle's, full MVM within tolerance."""
    m = bar_setup[0]
    ctx, tree, near = cuda_setup(m, galerkin=True)
    _near_vs_oracle(m, tree, near, True)
    x = meshes.make_x(2, m.n)
    err = oracle.rel_l2(run_mvm(tree, near, x), oracle_rows(m, x, galerkin=True))
    print("bar galerkin full", err)
    assert err <= TOL_FULL


def test_hybrid_mesh_errors():
    """A rectangle that is not a parallelogram is XRL_EGEOM; triangles-only [n][4] input equals the
    [n][3] path bit for bit."""
    from paper_2409_12375_b200 import xrl
    m = meshes.bar_hybrid()
    ctx, tree, near = cuda_setup(m)
    bad = m.verts.copy()
    bad[m.tris[0, 2]] += np.array([1e-6, 0, 0])  # breaks the first rectangle (and its neighbours)
    with pytest.raises(xrl.XrlError) as e:
        xrl.Tree(ctx, bad, m.tris)
    assert e.value.code == -4
    mb = meshes.bar()
    t4 = np.concatenate([mb.tris, np.full((mb.n, 1), -1, np.int32)], axis=1)
    c3, tr3, n3 = cuda_setup(mb)
    tr4 = xrl.Tree(c3, mb.verts, t4)
    n4 = xrl.Near(tr4)
    a, b = n3.export(), n4.export()
    assert all(np.array_equal(u, v) for u, v in zip(a, b))


@pytest.mark.parametrize("npanel", [1, 2, 5, 7, 11])
def test_degenerate_tiny_meshes(npanel):
    """Degenerate sizes: 1, 2, 5, 7 and 11 panels (a single leaf, no far field, the self term alone for
    N = 1; the near SpMV's last row group of 4 rows partial); also leaf_max = 1 (every panel its own leaf,
    the deepest tree).  The near-only product is checked against the oracle's CSR as well."""
    rng = np.random.default_rng(npanel)
    V = rng.normal(size=(3 * npanel, 3)) * 1e-4
    T = np.arange(3 * npanel, dtype=np.int32).reshape(-1, 3)
    m = meshes.Mesh(V, T)
    for leaf in (64, 1):
        ctx, tree, near = cuda_setup(m, leaf_max=leaf)
        x = meshes.make_x(1, m.n)
        err = oracle.rel_l2(run_mvm(tree, near, x), oracle_rows(m, x))
        print("tiny", npanel, leaf, err)
        assert err < 1e-6
        optr, ocol, oval, oinv_r = oracle.near_rows(oracle.Geometry(m.verts, m.tris))
        rows = np.repeat(np.arange(m.n), np.diff(optr))
        yref = np.zeros((3, m.n), dtype=np.complex128)
        for v in range(3):
            np.add.at(yref[v], rows, (oval - oinv_r) * x[v, ocol].astype(np.complex128))
        assert oracle.rel_l2(run_mvm(tree, near, x, flags=1), yref) <= TOL_NEAR


def test_host_batch_pipelined_equals_single_calls(bar_setup):
    """xrl_mvm_host_batch: 5 different inputs through the double-buffered pipeline (buffers repeated in
    the pointer lists too) give the same outputs as 5 blocking xrl_mvm_host calls."""
    import torch
    from paper_2409_12375_b200 import xrl
    m, ctx, tree, near = bar_setup
    xs = [torch.from_numpy(meshes.make_x(10 + k, m.n)).pin_memory().numpy() for k in range(5)]
    ys = [torch.empty((3, m.n), dtype=torch.complex64).pin_memory().numpy() for _ in range(5)]
    xrl.mvm_host_batch(tree, near, xs, ys)
    for k in range(5):
        ref = xrl.mvm_host(tree, near, xs[k])
        assert oracle.rel_l2(ys[k], ref) < 1e-6, k
    # repeated buffers: 6 steps over 2 inputs and 2 outputs; the last writes win
    y2 = [np.empty((3, m.n), np.complex64) for _ in range(2)]
    xrl.mvm_host_batch(tree, near, [xs[k % 2] for k in range(6)], [y2[k % 2] for k in range(6)])
    for k in range(2):
        assert oracle.rel_l2(y2[k], ys[k]) < 1e-6


@pytest.mark.parametrize("cfg,leaf", [(1, 16), (2, 352)])
def test_schedules_agree(cfg, leaf):
    """Fused P2P tasks (default), unfused, serial and late-fork schedules give the same y up to FP32
    summation order, and the fused result matches the oracle on sampled rows."""
    from paper_2409_12375_b200 import xrl
    m = meshes.make_config(cfg)
    ctx, tree, near = cuda_setup(m, leaf_max=leaf)
    x = meshes.make_x(cfg, m.n)
    y0 = run_mvm(tree, near, x)
    out = {}
    for name, sched, fuse in (("unfused", 1, False), ("serial", 0, True), ("late", 2, True)):
        ctx.set_sched(sched)
        ctx.set_fuse(fuse)
        out[name] = run_mvm(tree, near, x)
    ctx.set_sched(1)
    ctx.set_fuse(True)
    for name, y in out.items():
        err = oracle.rel_l2(y, y0)
        print(cfg, name, err)
        assert err < 1e-6, name
    rows = np.random.default_rng(7).choice(m.n, size=min(256, m.n), replace=False)
    assert oracle.rel_l2(y0[:, rows], oracle_rows(m, x, rows)) <= TOL_FULL


@pytest.mark.parametrize("cfg,leaf,nvec", [(1, 16, 6), (2, 64, 9), (2, 384, 12)])
@pytest.mark.parametrize("flags", [0, 1, 2])
def test_paired_triples_equal_single_triples(cfg, leaf, nvec, flags):
    """xrl_mvm with nvec = 6k runs the triples in pairs (one P2P / near pass for 12 right-hand sides,
    k_p2p12 / k_near_rg<2>); each triple of the result equals the same triple run alone (nvec = 3) up to
    the FP32 summation order, for the full, near-only and far-only products, and the paired full product
    matches the oracle on sampled rows (north-star bound)."""
    import torch
    from paper_2409_12375_b200 import xrl
    m = meshes.make_config(cfg)
    ctx, tree, near = cuda_setup(m, leaf_max=leaf)
    rng = np.random.default_rng(17)
    x = (rng.standard_normal((nvec, m.n)) + 1j * rng.standard_normal((nvec, m.n))).astype(np.complex64)
    y = run_mvm(tree, near, x, flags=flags)
    for v in range(0, nvec, 3):
        y1 = run_mvm(tree, near, np.ascontiguousarray(x[v:v + 3]), flags=flags)
        err = np.linalg.norm(y[v:v + 3] - y1) / np.linalg.norm(y1)
        assert err < 2e-6, (v, err)
    if flags == 0:
        rows = np.sort(rng.choice(m.n, size=min(256, m.n), replace=False))
        g = oracle.Geometry(m.verts, m.tris)
        yref = oracle.mvm_rows(g, x[3:6], rows)
        assert oracle.rel_l2(y[3:6, rows], yref) <= 2e-5


@pytest.mark.parametrize("align", ["corner", "centre"])
def test_root_placements_agree(align, tmp_path):
    """The root cube placement (the cost-model search, or XRL_ROOT_ALIGN=corner / centre) changes
    the tree, not the product: config 2's MVM with a forced placement (fresh process, the variable is read
    once) matches the oracle on sampled rows and the searched tree's result to FP32 accuracy."""
    import os
    import subprocess
    import sys
    m = meshes.make_config(2)
    ctx, tree, near = cuda_setup(m, leaf_max=64)
    x = meshes.make_x(2, m.n)
    y = run_mvm(tree, near, x)
    out = tmp_path / "y.npy"
    code = ("import sys, numpy as np; sys.path.insert(0, %r)\n"
            "from inputs import meshes\nfrom tests.gpu_helpers import cuda_setup, run_mvm\n"
            "m = meshes.make_config(2); ctx, tree, near = cuda_setup(m, leaf_max=64)\n"
            "np.save(%r, run_mvm(tree, near, meshes.make_x(2, m.n)))\n"
            "print(tree.info()['root_lo'])\n") % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), str(out))
    env = dict(os.environ, XRL_ROOT_ALIGN=align)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    print(align, "root_lo", r.stdout.strip(), "searched", tree.info()["root_lo"])
    y2 = np.load(out)
    assert oracle.rel_l2(y2, y) < 1e-5
    rows = np.random.default_rng(3).choice(m.n, size=256, replace=False)
    assert oracle.rel_l2(y2[:, rows], oracle_rows(m, x, rows)) <= TOL_FULL
