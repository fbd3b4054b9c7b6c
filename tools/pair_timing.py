"""Two triples per traversal (xrl_mvm nvec = 6: k_p2p12 / k_near_rg<2>) against one triple (nvec = 3), and
the 2-port loop-space operator apply against the 1-port one.

    python tools/pair_timing.py [--config 4] [--leaf 384] [--reps 20] [--out file.json]"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from inputs import meshes  # noqa: E402
from paper_2409_12375_b200 import xrl  # noqa: E402


def timed(ctx, fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        fn()
        e1.record(ctx.stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--leaf", type=int, default=384)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    m = meshes.make_config(a.config)
    ctx = xrl.Context(0)
    tree = xrl.Tree(ctx, m.verts, m.tris, leaf_max=a.leaf)
    near = xrl.Near(tree)
    rng = np.random.default_rng(5)
    x = torch.from_numpy((rng.standard_normal((12, m.n)) + 1j * rng.standard_normal((12, m.n))).astype(np.complex64)).cuda()
    xl = tree.to_library_order(x)
    y = torch.empty_like(xl)
    res = {"config": a.config, "n_panels": m.n, "leaf_max": a.leaf}
    res["mvm_1_triple_ms"] = timed(ctx, lambda: xrl.mvm(tree, near, xl[:3], y[:3]), a.reps)
    res["mvm_2_triples_paired_ms"] = timed(ctx, lambda: xrl.mvm(tree, near, xl[:6], y[:6]), a.reps)
    res["mvm_2_triples_separate_ms"] = timed(ctx, lambda: (xrl.mvm(tree, near, xl[:3], y[:3]),
                                                           xrl.mvm(tree, near, xl[3:6], y[3:6])), a.reps)
    res["mvm_4_triples_paired_ms"] = timed(ctx, lambda: xrl.mvm(tree, near, xl, y), a.reps)
    res["pair_ratio"] = res["mvm_2_triples_paired_ms"] / res["mvm_1_triple_ms"]
    # isolated phase times (serial schedule): one triple vs a pair
    for name, nv in (("phases_1_triple", 3), ("phases_pair", 6)):
        ctx.set_sched(ctx.SCHED_SERIAL)
        xrl.mvm(tree, near, xl[:nv], y[:nv])
        torch.cuda.synchronize()
        ctx.timing_reset()
        ctx.timing_enable(True)
        for _ in range(5):
            xrl.mvm(tree, near, xl[:nv], y[:nv])
        torch.cuda.synchronize()
        ctx.timing_enable(False)
        res[name] = {k: v[0] / 5 for k, v in ctx.timing().items()}
        ctx.set_sched(ctx.SCHED_FORK)
    # loop-space operator: 1 vs 2 right-hand sides (a 2-port solve applies both per GMRES step)
    topo = xrl.Topology(tree, [])
    op = xrl.Operator(tree, near, topo, 1e9, sigma=5.8e7, zeta=10e-6)
    nl = topo.n_loops
    u = torch.from_numpy((rng.standard_normal((2, nl)) + 1j * rng.standard_normal((2, nl))).astype(np.complex64)).cuda()
    w = torch.empty_like(u)
    res["op_1_rhs_ms"] = timed(ctx, lambda: op.apply(u[:1], w[:1]), a.reps)
    res["op_2_rhs_ms"] = timed(ctx, lambda: op.apply(u, w), a.reps)
    res["op_ratio"] = res["op_2_rhs_ms"] / res["op_1_rhs_ms"]
    js = json.dumps(res, indent=1)
    print(js)
    if a.out:
        open(a.out, "w").write(js + "\n")


if __name__ == "__main__":
    main()
