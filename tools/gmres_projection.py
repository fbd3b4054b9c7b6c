"""GMRES iteration time of config 4 at 1/2/4/8 GPUs, projected from virtual ranks on one GPU (BASELINE config
4: "MVM and GMRES iteration time at 1/2/4/8 GPUs"; SURVEY §8(d) t_iter).

The sharded loop-space GMRES (xrl_gmres_vranks: k operators on the k trees of a partition, rank-local block
diag-of-P preconditioners, inner products summed over the ranks) runs a fixed number of iterations on one GPU
with the ranks serialised; its time per iteration divided by k is the mean rank's device time per iteration.
The projection multiplies that by the MVM's measured rank imbalance and adds the exposed communication per
iteration: the MVM's (tools/vrank_projection.py model), two loop-space halo exchanges of the operator (loop
values, panel values: volumes from the plans) and 2 x CGS2 passes + 1 norm of FP64 all-reduces, 15 us each.

    python tools/gmres_projection.py [--ks 1,2,4,8] [--iters 20] [--out file.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from inputs import meshes  # noqa: E402
from paper_2409_12375_b200 import xrl  # noqa: E402

LAT = 15e-6


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--leaf", type=int, default=384)
    ap.add_argument("--ks", default="1,2,4,8")
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--freq", type=float, default=1e9)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    m = meshes.make_config(a.config)
    ctx = xrl.Context(0)
    res = {"config": a.config, "n_panels": m.n, "freq_hz": a.freq, "iters": a.iters, "ks": {}}
    b_full = None
    for k in [int(v) for v in a.ks.split(",")]:
        t0 = time.perf_counter()
        trees, nears, topos, ops, pcs = [], [], [], [], []
        for r in range(k):
            kw = dict(part_rank=r, part_world=k) if k > 1 else {}
            tr = xrl.Tree(ctx, m.verts, m.tris, leaf_max=a.leaf, **kw)
            nr = xrl.Near(tr)
            tp = xrl.Topology(tr, [])
            op = xrl.Operator(tr, nr, tp, a.freq, sigma=5.8e7, zeta=10e-6)
            trees.append(tr); nears.append(nr); topos.append(tp); ops.append(op)
            pcs.append(xrl.Precond(op, 64))
        setup = time.perf_counter() - t0
        nl = topos[0].n_loops
        if b_full is None:
            rng = np.random.default_rng(1404)
            b_full = torch.from_numpy((rng.random((1, nl)) - 0.5 + 1j * (rng.random((1, nl)) - 0.5))
                                      .astype(np.complex64)).cuda()
        sl = [o.loops() for o in ops]
        bs = [b_full[:, s0:s0 + c].contiguous() for s0, c in sl]
        xrl.gmres_vranks(ops, pcs, bs, max_iters=a.iters, tol=1e-30)  # warm-up (Krylov basis allocated)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, rep = xrl.gmres_vranks(ops, pcs, bs, max_iters=a.iters, tol=1e-30)
        e1.record()
        torch.cuda.synchronize()
        it = int(rep["iters"][0])
        ms_iter_all = e0.elapsed_time(e1) / max(it, 1)
        if k == 1:  # the single-GPU solver itself (xrl_gmres), beside the one-rank xrl_gmres_vranks
            xrl.gmres(ops[0], pcs[0], bs[0], max_iters=a.iters, tol=1e-30)
            torch.cuda.synchronize()
            e0.record()
            _, rep1 = xrl.gmres(ops[0], pcs[0], bs[0], max_iters=a.iters, tol=1e-30)
            e1.record()
            torch.cuda.synchronize()
            res["xrl_gmres_ms_per_iter"] = e0.elapsed_time(e1) / max(int(rep1["iters"][0]), 1)
        # MVM projection inputs of this partition
        xs = []
        off = 0
        for t in trees:
            xs.append(torch.zeros((3, t.n_local), dtype=torch.complex64, device="cuda"))
        ys = [torch.empty_like(v) for v in xs]
        runs = [xrl.mvm_vranks(trees, nears, xs, ys, timing=True)[1] for _ in range(3)] if k > 1 else [[1.0]]
        rk = np.median(np.array(runs), axis=0)
        imb = float(rk.max() / rk.mean())
        info = [xrl.exchange_info(t, n) for t, n in zip(trees, nears)] if k > 1 else []
        # exposed communication per iteration: MVM (LET + shared + 2 latencies; the halo overlaps the up pass),
        # the operator's loop / panel halos (8 B per loop value, 24 B per panel value, one RHS), 5 all-reduces
        comm = 0.0
        if k > 1:
            mu = max(3072 * max(i["let_send"], i["let_recv"]) + 2 * 3072 * i["shared"] for i in info) / 900e9
            op_halo = 2 * LAT + max(8 * o.halo()[0] + 24 * o.halo()[1] for o in ops) / 900e9
            comm = mu + 2 * LAT + op_halo + 5 * LAT
        proj = ms_iter_all / k * imb + 1e3 * comm
        res["ks"][k] = {"gmres_iters": it, "ms_per_iter_all_ranks_on_one_gpu": ms_iter_all, "mvm_rank_imbalance": imb,
                        "comm_ms_per_iter": 1e3 * comm, "projected_ms_per_iter": proj, "setup_s": round(setup, 1),
                        "n_loops": nl, "loops_per_rank": [c for _, c in sl]}
        print(json.dumps({k: res["ks"][k]}), flush=True)
        del pcs, ops, topos, nears, trees, xs, ys, bs
        torch.cuda.empty_cache()
    t1 = res["ks"].get(1, {}).get("projected_ms_per_iter")
    for k, v in res["ks"].items():
        if t1:
            v["speedup"] = t1 / v["projected_ms_per_iter"]
    js = json.dumps(res, indent=1)
    print(js)
    if a.out:
        open(a.out, "w").write(js + "\n")


if __name__ == "__main__":
    main()
