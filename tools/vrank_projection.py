"""Multi-GPU projection of the sharded MVM from virtual ranks on ONE GPU.

Only one B200 is available to this build, so the k-GPU time is projected from measurements of the real
sharded code path: k trees partitioned 0..k-1 of the same mesh run through xrl_mvm_vranks (the same
plans, exchanges and kernels as the multi-rank xrl_mvm; exchanges as device copies).  Each rank's phase
groups run alone on the whole GPU with the production (forked, fused) schedule, so its measured device
time is what one GPU would spend on that rank's share.  The projection is
    t(k) = max_r t_rank(r) + t_comm(k),
    t_comm = max(0, t_halo - t_up) + (max(LET sent, received) + 2 x shared bytes of the busiest rank) / 900 GB/s
             + 2 x 15 us,
    t_halo = max(halo sent, received) of the busiest rank / 900 GB/s (NVLink 5, per direction) + 15 us:
the halo of x overlaps the up pass (xrl_mvm issues it on its comm stream while P2M / M2M read only the rank's
own charges), the shared-box all-reduce and the LET exchange are on the critical path.  The single-GPU references are the
same driver at k = 1 and xrl_mvm itself.

    python tools/vrank_projection.py [--config 4] [--leaf 384] [--ks 1,2,4,8] [--reps 5] [--out file.json]
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from inputs import meshes  # noqa: E402
from paper_2409_12375_b200 import xrl  # noqa: E402

NVLINK_GBS = 900.0
LAT_S = 15e-6


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--leaf", type=int, default=384)
    ap.add_argument("--ks", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    m = meshes.make_config(a.config)
    ctx = xrl.Context(0)
    x_user = torch.from_numpy(meshes.make_x(a.config, m.n)).cuda()
    # single-GPU reference with the default schedule
    tree = xrl.Tree(ctx, m.verts, m.tris, leaf_max=a.leaf)
    near = xrl.Near(tree)
    xl = tree.to_library_order(x_user)
    y = torch.empty_like(xl)
    for _ in range(3):
        xrl.mvm(tree, near, xl, y)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        xrl.mvm(tree, near, xl, y)
        e1.record(ctx.stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    t_fork = statistics.median(ts)
    del near, tree, y
    torch.cuda.empty_cache()
    res = {"config": a.config, "n_panels": m.n, "leaf_max": a.leaf, "t1_forked_ms": t_fork,
           "model": "t(k) = max_r t_rank(r) + max(0, t_halo - t_up) + (max(LET sent, recv) + 2 shared bytes) / 900 GB/s + 2 x 15 us", "ks": {}}
    for k in [int(v) for v in a.ks.split(",")]:
        t0 = time.perf_counter()
        trees, nears, xs, off = [], [], [], 0
        for r in range(k):
            tr = xrl.Tree(ctx, m.verts, m.tris, leaf_max=a.leaf, part_rank=r if k > 1 else None,
                          part_world=k if k > 1 else None)
            trees.append(tr)
            nears.append(xrl.Near(tr))
            xs.append(xl[:, off:off + tr.n_local].contiguous())
            off += tr.n_local
        setup = time.perf_counter() - t0
        ys = [torch.empty_like(v) for v in xs]
        for _ in range(2):
            xrl.mvm_vranks(trees, nears, xs, ys)
        rank_ms, exch_ms = [], []
        for _ in range(a.reps):
            _, rms, ems = xrl.mvm_vranks(trees, nears, xs, ys, timing=True)
            rank_ms.append(rms)
            exch_ms.append(ems)
        # per-phase device times (event spans per phase, summed over the ranks, per rank on average)
        ctx.timing_reset()
        ctx.timing_enable(True)
        xrl.mvm_vranks(trees, nears, xs, ys)
        torch.cuda.synchronize()
        ctx.timing_enable(False)
        phases = {kk: vv[0] / k for kk, vv in ctx.timing().items()}
        rank_med = np.median(np.array(rank_ms), axis=0)
        info = [xrl.exchange_info(t, n) for t, n in zip(trees, nears)]
        byts = [32 * (i["halo_send"] + i["halo_recv"]) + 3072 * (i["let_send"] + i["let_recv"]) +
                2 * 3072 * i["shared"] for i in info]
        # the halo overlaps the up pass (P2M + M2M read only the rank's own charges; xrl_mvm issues the halo on
        # its comm stream): only what exceeds the up pass is exposed; the all-reduce and the LET are not overlapped
        # NVLink 5 is full duplex (900 GB/s per direction): an exchange costs max(sent, received) / 900 GB/s
        halo_s = max(32 * max(i["halo_send"], i["halo_recv"]) for i in info) / (NVLINK_GBS * 1e9) + LAT_S
        up_s = 1e-3 * (phases.get("p2m", 0.0) + phases.get("m2m", 0.0) + phases.get("pack", 0.0))
        mu_s = max(3072 * max(i["let_send"], i["let_recv"]) + 2 * 3072 * i["shared"] for i in info) / (NVLINK_GBS * 1e9)
        comm_s = (max(0.0, halo_s - up_s) + mu_s + 2 * LAT_S) if k > 1 else 0.0
        t_k = float(rank_med.max()) + 1e3 * comm_s
        res["ks"][k] = {"rank_ms": rank_med.tolist(), "t_rank_max_ms": float(rank_med.max()),
                        "t_rank_mean_ms": float(rank_med.mean()),
                        "imbalance": float(rank_med.max() / rank_med.mean()),
                        "n_local": [t.n_local for t in trees], "exchange": info, "bytes_per_rank": byts,
                        "t_comm_ms": 1e3 * comm_s, "exchange_copy_ms_on_one_gpu": float(np.median(exch_ms)),
                        "t_projected_ms": t_k, "setup_s": round(setup, 2), "phases_ms_per_rank": phases}
        print(json.dumps({k: res["ks"][k]}), flush=True)
        del ys, xs, nears, trees
        torch.cuda.empty_cache()
    t1 = res["ks"].get(1, {}).get("t_projected_ms")
    for k, v in res["ks"].items():
        if t1:
            v["speedup_vs_k1"] = t1 / v["t_projected_ms"]
        v["speedup_vs_forked_1gpu"] = t_fork / v["t_projected_ms"]
        v["projected_mpanels_s"] = m.n / (v["t_projected_ms"] * 1e-3) / 1e6
    js = json.dumps(res, indent=1)
    print(js)
    if a.out:
        open(a.out, "w").write(js + "\n")


if __name__ == "__main__":
    main()
