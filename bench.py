#!/usr/bin/env python
"""Benchmark of the XRL hot path: FMM MVM throughput (Mpanels/s, one MVM =
3 complex components = 6 real right-hand sides through one tree pass).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl xrl|reference] [--config 4]

Workload (BASELINE.json): config 4 (package-on-package-like stack, ~1.9M
panels, highly non-uniform density) at N = 1; configs 1-3 are parity cases
(tests/).  A "step" is one xrl_mvm over one synthetic input triple already
resident in HBM.  L2 is flushed (256 MiB write) between timed steps, each
step timed with CUDA events on the library's stream.  Under torchrun the MVM
is sharded: every rank owns a work-balanced Morton range of
the panels, the owned slices of x are gathered with NCCL inside xrl_mvm, and
each rank computes its slice of y (strong scaling: the same problem on N
GPUs); the slowest rank's device time counts.

--impl reference runs the FP64 oracle (oracle/) on the host cores over a
bounded sample of target rows of the same workload (the reference arm of this
tier; rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG_NAMES = {1: "cfg1_bar_2100", 2: "cfg2_coils", 3: "cfg3_bga16", 4: "cfg4_pop_2M", 5: "cfg5_bga64"}
METRIC = "FMM MVM Mpanels/s (3 complex comps)"


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.samples = []
        self._stop = threading.Event()
        self._th = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for nm, v in zip(names, s[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def host_cpu():
    """lscpu model / sockets / cores / threads of the host the oracle runs on."""
    info = {}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            k = k.strip()
            if k in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core", "CPU(s)"):
                info[k] = v.strip()
    except Exception:
        pass
    return info


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_oracle_run(mesh, x, n_rows, seed=7):
    """Time the oracle on a seeded sample of target rows (all host cores)."""
    import numpy as np

    import oracle
    g = oracle.Geometry(mesh.verts, mesh.tris)
    rows = np.random.default_rng(seed).choice(mesh.n, size=n_rows, replace=False)
    t0 = time.perf_counter()
    oracle.mvm_rows(g, x, rows)
    dt = time.perf_counter() - t0
    return dt, oracle.num_threads()


def cpu_baseline(mesh, x, budget_s=12.0):
    """Oracle direct sum on a bounded row sample; value = target rows / s / 1e6
    (the same unit as the GPU metric: panels of y produced per second)."""
    import numpy as np
    rows0 = 64
    dt0, cores = cpu_oracle_run(mesh, x, rows0, seed=11)
    rows = int(min(mesh.n, max(rows0, rows0 * budget_s / max(dt0, 1e-3))))
    dt, cores = cpu_oracle_run(mesh, x, rows)
    return {"value": rows / dt / 1e6, "unit": "Mpanels/s", "cores": cores, "kind": "oracle",
            "sample": f"{rows} seeded target rows x all {mesh.n} sources, FP64 direct sum (O(N^2) per MVM, "
                      f"not an FMM), {dt:.2f} s wall; full MVM extrapolated {dt * mesh.n / rows:.0f} s",
            "host": host_cpu()}


def parallelism_name(world):
    return f"morton-range shards x{world} (halo + LET exchanges over NCCL)" if world > 1 else "single GPU"


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from inputs import meshes
    mesh = meshes.make_config(args.config)
    x = meshes.make_x(args.config, mesh.n)
    # bounded sample per step so that warmup + steps stay within a few minutes
    import numpy as np
    _, cores = cpu_oracle_run(mesh, x, 16, seed=3)
    dt16, _ = cpu_oracle_run(mesh, x, 64, seed=5)
    per_step_rows = int(max(64, 64 * 8.0 / max(dt16, 1e-3)))
    for w in range(args.warmup):
        cpu_oracle_run(mesh, x, min(per_step_rows, 256), seed=100 + w)
    times = []
    for s in range(args.steps):
        dt, cores = cpu_oracle_run(mesh, x, per_step_rows, seed=200 + s)
        times.append(dt)
    tot = sum(times)
    value = per_step_rows * args.steps / tot / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Mpanels/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": CFG_NAMES[args.config], "n_panels": mesh.n, "p": 10, "leaf_max": args.leaf,
                   "eta": 1.5, "parallelism": parallelism_name(world)},
        "cpu_baseline": {"value": value, "unit": "Mpanels/s", "cores": cores, "kind": "oracle",
                         "sample": f"{per_step_rows} seeded target rows per step x all {mesh.n} sources (FP64 direct sum)"
                                   ", host threads (OpenMP), rank 0 only",
                         "host": host_cpu()},
        "e2e": {"value": value, "unit": "Mpanels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _tc_subtiles(tree) -> int:
    """Number of tcgen05 MMA groups (one per <= 16-pair tile) the M2L issues."""
    return int(tree.info()["n_m2l_subtiles"])


def traffic_from_profiles(kernel: str, key: str):
    """DRAM read+write bytes per launch of `kernel` from a committed ncu
    capture of the same workload/leaf (profiles/traffic.json), else None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(p)).get(key, {}).get(kernel)
    except Exception:
        return None


def gmres_iteration_time(xrl, tree, near, args, freq=1e9):
    """BASELINE config 4 also asks for the GMRES iteration time: loop-space
    operator at 1 GHz (sigma 5.8e7, zeta 10 um), block diag-of-P
    preconditioner, one random complex RHS (seed 1404), a fixed number of
    restarted-GMRES iterations timed with CUDA events (operator + preconditioner
    + CGS2 orthogonalisation per iteration)."""
    import numpy as np
    import torch
    t0 = time.perf_counter()
    topo = xrl.Topology(tree, [])
    op = xrl.Operator(tree, near, topo, freq, sigma=5.8e7, zeta=10e-6)
    pc = xrl.Precond(op, 64)
    setup = time.perf_counter() - t0
    nl = topo.n_loops
    rng = np.random.default_rng(1404)
    b = torch.from_numpy((rng.random((1, nl)) - 0.5 + 1j * (rng.random((1, nl)) - 0.5)).astype(np.complex64)).cuda()
    xrl.gmres(op, pc, b, max_iters=2, tol=1e-30)  # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, rep = xrl.gmres(op, pc, b, max_iters=args.gmres_iters, restart=50, tol=1e-30)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    solve = None
    if args.gmres_solve > 0:  # optional: the solve to the paper's tolerance (1e-4 above 1 MHz)
        e0.record()
        _, rep2 = xrl.gmres(op, pc, b, max_iters=args.gmres_solve)
        e1.record()
        torch.cuda.synchronize()
        solve = {"iters": int(rep2["iters"][0]), "ms": e0.elapsed_time(e1), "true_rre": float(rep2["true_rre"][0]),
                 "converged": bool(rep2["converged"][0])}
    info = topo.info()
    return {"ms_per_iter": ms / max(int(rep["iters"][0]), 1), "iters": int(rep["iters"][0]), "freq_hz": freq,
            "solve_to_tol": solve,
            "n_loops": nl, "vertex_loops": info["n_vertex_loops"], "fundamental_loops": info["n_fundamental_loops"],
            "preconditioned_rre_after": float(rep["rre"][0]), "setup_s": round(setup, 2),
            "note": "iteration = loop operator (sparse maps + FMM MVM) + block preconditioner + CGS2; the average "
                    "over one call, which also applies the operator for its initial and true residual (2 of the "
                    "iteration count's applies)"}


def leaf64_line(xrl, mesh, x_user, ctx, dev, flush, args):
    """the same workload at the BASELINE leaf size 64 (the headline uses the tuned leaf):
    K MVMs timed with CUDA events, L2 flushed between them."""
    import torch
    t0 = time.perf_counter()
    tree = xrl.Tree(ctx, mesh.verts, mesh.tris, leaf_max=64)
    near = xrl.Near(tree, eta=1.5)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    xd = tree.to_library_order(torch.from_numpy(x_user).to(dev))
    y = torch.empty_like(xd)
    for _ in range(3):
        xrl.mvm(tree, near, xd, y)
    torch.cuda.synchronize()
    ts = []
    for _ in range(max(args.steps, 20)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.zero_()
        e0.record(ctx.stream)
        xrl.mvm(tree, near, xd, y)
        e1.record(ctx.stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sum(ts) / len(ts)
    info = tree.info()
    out = {"leaf_max": 64, "value": mesh.n / (ms * 1e-3) / 1e6, "unit": "Mpanels/s", "ms_per_step": ms,
           "ms_median": statistics.median(ts), "steps": len(ts), "setup_s": round(setup, 3),
           "leaves": info["n_leaves"], "m2l_translations": info["n_v_pairs"], "p2p_pairs": info["n_p2p"]}
    del near, tree
    return out


def multi_gpu_projection(xrl, mesh, ctx, x_lib, ms_1gpu, args, k=8):
    """Projected k-GPU time of the sharded MVM from k virtual ranks on this GPU (tools/vrank_projection.py
    has the full sweep): each rank's phase groups timed alone on the GPU with the production
    schedule through xrl_mvm_vranks (the same plans, exchanges and kernels as the NCCL path), plus the
    exchange volume over NVLink 5 (900 GB/s per direction) and 15 us latency per exchange (3 exchanges)."""
    import numpy as np
    import torch
    trees, nears, xs, off = [], [], [], 0
    for r in range(k):
        tr = xrl.Tree(ctx, mesh.verts, mesh.tris, leaf_max=args.leaf, part_rank=r, part_world=k)
        trees.append(tr)
        nears.append(xrl.Near(tr))
        xs.append(x_lib[:, off:off + tr.n_local].contiguous())
        off += tr.n_local
    ys = [torch.empty_like(v) for v in xs]
    for _ in range(2):
        xrl.mvm_vranks(trees, nears, xs, ys)
    runs = [xrl.mvm_vranks(trees, nears, xs, ys, timing=True)[1] for _ in range(5)]
    rank_ms = np.median(np.array(runs), axis=0)
    ctx.timing_reset()
    ctx.timing_enable(True)
    xrl.mvm_vranks(trees, nears, xs, ys)
    torch.cuda.synchronize()
    ctx.timing_enable(False)
    ph = {kk: vv[0] / k for kk, vv in ctx.timing().items()}
    info = [xrl.exchange_info(t, n) for t, n in zip(trees, nears)]
    byts = [32 * (i["halo_send"] + i["halo_recv"]) + 3072 * (i["let_send"] + i["let_recv"]) + 2 * 3072 * i["shared"]
            for i in info]
    # the halo overlaps the up pass (comm stream); the all-reduce and the LET are on the critical path.  NVLink 5
    # is 900 GB/s per direction: a rank's sends and receives of one exchange proceed concurrently, so an
    # exchange costs max(sent, received) bytes / 900 GB/s; the shared-box all-reduce moves 2x its bytes each way
    halo_ms = 1e3 * (max(32 * max(i["halo_send"], i["halo_recv"]) for i in info) / 900e9 + 15e-6)
    up_ms = ph.get("pack", 0.0) + ph.get("p2m", 0.0) + ph.get("m2m", 0.0)
    mu_ms = 1e3 * max(3072 * max(i["let_send"], i["let_recv"]) + 2 * 3072 * i["shared"] for i in info) / 900e9
    comm_ms = max(0.0, halo_ms - up_ms) + mu_ms + 1e3 * 2 * 15e-6
    t_k = float(rank_ms.max()) + comm_ms
    out = {"k": k, "projected_ms": t_k, "rank_ms": [round(float(v), 4) for v in rank_ms], "comm_ms": comm_ms,
           "max_rank_bytes": int(max(byts)), "speedup_vs_1gpu": ms_1gpu / t_k,
           "projected_value": mesh.n / (t_k * 1e-3) / 1e6, "unit": "Mpanels/s",
           "halo_ms": halo_ms, "up_pass_ms": up_ms,
           "how": "virtual ranks on one GPU (xrl_mvm_vranks): max over ranks of each rank's MVM alone + the exposed "
                  "exchange time over NVLink 5 (900 GB/s per direction: max(sent, received) per exchange, 15 us "
                  "each; the halo overlaps the up pass); "
                  "a projection, not a multi-GPU measurement"}
    del ys, xs, nears, trees
    torch.cuda.empty_cache()
    return out


def run_xrl(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from inputs import meshes
    from paper_2409_12375_b200 import xrl

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    mesh = meshes.make_config(args.config)
    x_user = meshes.make_x(args.config, mesh.n)
    t0 = time.perf_counter()
    ctx = xrl.distributed_context(local) if world > 1 else xrl.Context(local)
    torch.cuda.synchronize()
    context_s = time.perf_counter() - t0  # once per process: CUDA init, FP64 operator tables
    t0 = time.perf_counter()
    tree = xrl.Tree(ctx, mesh.verts, mesh.tris, leaf_max=args.leaf)
    torch.cuda.synchronize()
    tree_s = time.perf_counter() - t0  # per mesh: root placement search, octree, lists, plans
    near = xrl.Near(tree, eta=1.5)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0  # per mesh: tree + near-field assembly
    info = tree.info()
    n = mesh.n

    x_lib = tree.to_library_order(torch.from_numpy(x_user).to(dev))
    xd = x_lib[:, tree.offset:tree.offset + tree.n_local].contiguous()  # this rank's slice
    y = torch.empty_like(xd)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = ctx.stream

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3)):
        xrl.mvm(tree, near, xd, y)
    barrier()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    ctx.timing_reset()
    ctx.timing_enable(True)
    launches0 = ctx.launch_count()
    with ClockSampler(local) as clk:
        barrier()
        for s in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            ev[s][0].record(stream)
            xrl.mvm(tree, near, xd, y)
            ev[s][1].record(stream)
        barrier()
    launches = ctx.launch_count() - launches0
    ctx.timing_enable(False)
    phases = ctx.timing()

    # SURVEY §8(d) protocol beside the contract's K-step total: the median of >= 20 calls spanning >= 1 s
    # (each call timed alone with CUDA events, L2 flushed in between)
    per_call = [a.elapsed_time(b) for a, b in ev]
    med_calls = list(per_call)
    while len(med_calls) < 20 or sum(med_calls) < 1000.0:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.zero_()
        e0.record(stream)
        xrl.mvm(tree, near, xd, y)
        e1.record(stream)
        e1.synchronize()
        med_calls.append(e0.elapsed_time(e1))
    med_ms = statistics.median(med_calls)

    # isolated kernel times: the same MVM with every kernel serialised on one stream (not the
    # headline; explains it).  Kernels run alone, so per-kernel rooflines are not diluted by sharing.
    ctx.set_sched(ctx.SCHED_SERIAL)
    for _ in range(2):
        xrl.mvm(tree, near, xd, y)
    barrier()
    ctx.timing_reset()
    ctx.timing_enable(True)
    iso_steps = max(3, min(args.steps, 10))
    for s in range(iso_steps):
        flush.zero_()
        xrl.mvm(tree, near, xd, y)
    barrier()
    ctx.timing_enable(False)
    phases_iso = ctx.timing()
    ctx.set_sched(ctx.SCHED_FORK)
    ms = sum(a.elapsed_time(b) for a, b in ev)
    t_dev = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t_dev, op=dist.ReduceOp.MAX)
    ms_max = float(t_dev.item())
    ms_per_step = ms_max / args.steps
    value = n / (ms_per_step * 1e-3) / 1e6  # whole job: all N panels per MVM

    # e2e through the public host API: pinned host buffers, H2D + reorder + MVM + reorder + D2H
    if world > 1:  # host slices in library order (xrl_mvm_host on a multi-rank context)
        xh = xd.cpu().pin_memory()
    else:
        xh = torch.from_numpy(x_user).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    xh_np, yh_np = xh.numpy(), yh.numpy()
    for _ in range(2):
        xrl.mvm_host(tree, near, xh_np, yh_np)
    barrier()
    e2e_times = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        xrl.mvm_host(tree, near, xh_np, yh_np)  # blocking
        e2e_times.append(time.perf_counter() - t1)
    te = torch.tensor([sum(e2e_times) / len(e2e_times)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_single = n / float(te.item()) / 1e6
    # pipelined end-to-end over all steps (xrl_mvm_host_batch): step k+1's H2D and step k-1's D2H overlap
    # step k's MVM; two pinned input and two pinned output buffers alternate (every step still copies its
    # input in and its result out)
    xh2, yh2 = xh.clone().pin_memory(), torch.empty_like(yh).pin_memory()
    xs = [xh_np, xh2.numpy()]
    ys = [yh_np, yh2.numpy()]
    xrl.mvm_host_batch(tree, near, [xs[k % 2] for k in range(3)], [ys[k % 2] for k in range(3)])
    barrier()
    t1 = time.perf_counter()
    xrl.mvm_host_batch(tree, near, [xs[k % 2] for k in range(args.steps)], [ys[k % 2] for k in range(args.steps)])
    tb = torch.tensor([(time.perf_counter() - t1) / args.steps], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tb, op=dist.ReduceOp.MAX)
    e2e_value = n / float(tb.item()) / 1e6

    # roofline of the dominant kernel (+ the other hot kernels for reference)
    peaks = _peaks()
    clocks = clk.summary()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    fp32_peak = nsm * 128 * 2 * sm_max * 1e6 / 1e12  # TFLOP/s, SIMT FFMA (derivation: DESIGN.md)
    hbm_peak = float(peaks.get("hbm_gbs", 6551.4))
    nc = 121
    nnz = near.nnz()
    tkey = f"{CFG_NAMES[args.config]}_leaf{args.leaf}"

    def per_launch_ms(ph, src=None):
        ms_, cnt = (src or phases)[ph]
        return ms_ / max(cnt, 1)

    def rate(ph, work, src=None):  # work units per launch / launch duration
        return work / (per_launch_ms(ph, src) * 1e-3)

    roofs = {}
    if phases["m2l"][1]:
        # the M2L runs 3xFP16 (kind::f16: per 21-pair tile 8 K-steps x 3 MMAs of M128 N128 K16) unless
        # XRL_M2L_TF32=1 selects 3xTF32 (kind::tf32: 16 K-steps x 3 MMAs of M128 N128 K8); both issue
        # 2*128*128*128*3 flops per tile
        h16 = os.environ.get("XRL_M2L_TF32", "0") != "1"
        n_sub = _tc_subtiles(tree)
        issued = n_sub * 3 * 2.0 * 128 * 128 * 128
        bf16_peak = float(peaks.get("bf16_tflops", 1656.1))
        tc_peak = bf16_peak if h16 else bf16_peak * 0.5  # f16 dense = bf16 dense; tf32 nominal 1.1/2.25 of it
        ceil3 = tc_peak / 3.0  # three MMAs per FP32-accurate product
        alg_w = 2.0 * nc * nc * 6 * info["n_v_pairs"]
        ai = rate("m2l", alg_w, phases_iso) / 1e12
        a = rate("m2l", alg_w) / 1e12
        issued_i = rate("m2l", issued, phases_iso) / 1e12
        kind = "3xFP16 kind::f16, 24 MMAs M128 N128 K16" if h16 else "3xTF32 kind::tf32, 48 MMAs M128 N128 K8"
        roofs["m2l"] = {"kernel": "k_m2l_tc", "bound": "tensor", "achieved": ai, "peak": tc_peak, "unit": "TFLOP/s",
                        "frac": ai / tc_peak, "traffic": traffic_from_profiles("k_m2l_tc", tkey),
                        "ms": per_launch_ms("m2l", phases_iso),
                        ("frac_of_3xf16_ceiling" if h16 else "frac_of_3xtf32_ceiling"): ai / ceil3,
                        "frac_of_fp32_simt_peak": ai / fp32_peak,
                        "in_step": {"achieved": a, "frac": a / tc_peak, "ms": per_launch_ms("m2l")},
                        "issued": {"achieved": issued_i, "frac": issued_i / tc_peak,
                                   "what": f"{n_sub} tiles x ({kind}) per launch"},
                        "algorithmic": f"{2 * nc * nc * 6} flops (121 x 121 operator x 6 RHS, dense) x "
                                       f"{info['n_v_pairs']} V-list translations per launch",
                        "peak_source": ("f16 dense = bf16_tflops (MEASURED_PEAKS.json)" if h16 else
                                        "tf32 dense = bf16_tflops (MEASURED_PEAKS.json) x 0.5 (nominal 1.1/2.25 PF)")
                                       + "; 3x ceiling = that / 3"}
    if phases["p2p"][1]:
        w = 20.0 * info["n_p2p"]
        a, ai = rate("p2p", w) / 1e12, rate("p2p", w, phases_iso) / 1e12
        roofs["p2p"] = {"kernel": "k_p2p", "bound": "alu", "achieved": ai, "peak": fp32_peak, "unit": "TFLOP/s",
                        "frac": ai / fp32_peak, "traffic": traffic_from_profiles("k_p2p", tkey),
                        "ms": per_launch_ms("p2p", phases_iso),
                        "in_step": {"achieved": a, "frac": a / fp32_peak, "ms": per_launch_ms("p2p")},
                        "algorithmic": f"20 flops x {info['n_p2p']} ordered panel pairs per launch (every P2P pair "
                                       f"of the MVM: 3 sub + 1 mul + 2 fma for r^2, rsqrt counted as 1, 6 fma x q/r + "
                                       f"... = 20)",
                        "note": "achieved/frac: the k_p2p launch of the isolated pass (serial schedule, fusion off: "
                                "it does every pair), CUDA events on its stream inside bench.py.  in_step: the "
                                "standalone launch inside the timed MVMs, where part of the leaf tasks run in "
                                "k_m2l_tc's three spare warps concurrently, so its per-launch rate undercounts",
                        "peak_source": f"{nsm} SMs x 128 FP32 lanes x 2 flops x {sm_max:.0f} MHz (sm_max_mhz, MEASURED_PEAKS.json)"}
    if phases["near"][1]:
        ni = near.info()
        nl_ = tree.n_local
        # SURVEY §8(d)'s per-unit figure for the near SpMV: 8 B per nnz (FP32 value + int32 column) + 8 B per row
        # (row pointer) + 24 B per row (x, read once) + 48 B per row (y read-modify-write).  The row-group format
        # streams its own bytes (18 B per union-column slot + 16 B per segment), reported beside it.
        # the CSR holds every row; on a partitioned tree the owned rows' share is taken pro rata
        nnz_loc = ni["nnz"] if nl_ == tree.n else int(ni["nnz"] * nl_ / tree.n)
        byts = 8.0 * nnz_loc + 80.0 * nl_
        fmt = 18.0 * ni["n_entries"] + 16.0 * ni["n_segments"] + 72.0 * nl_
        a, ai = rate("near", byts) / 1e9, rate("near", byts, phases_iso) / 1e9
        roofs["near"] = {"kernel": "k_near_rg", "bound": "hbm", "achieved": ai, "peak": hbm_peak, "unit": "GB/s",
                         "frac": ai / hbm_peak, "traffic": traffic_from_profiles("k_near_rg", tkey),
                         "ms": per_launch_ms("near", phases_iso),
                         "in_step": {"achieved": a, "frac": a / hbm_peak, "ms": per_launch_ms("near")},
                         "algorithmic": f"SURVEY 8(d): 8 B x {nnz_loc} nnz of the owned rows + 80 B x {nl_} rows "
                                        f"(8 B row pointer, 24 B x read once, 48 B y read-modify-write) per launch",
                         "format_bytes": fmt,
                         "format_frac": rate("near", fmt, phases_iso) / 1e9 / hbm_peak,
                         "format": f"row groups of 4 rows: 18 B x {ni['n_entries']} union-column slots (float4 of the "
                                   f"4 rows' values + u16 column offset) + 16 B x {ni['n_segments']} segments + "
                                   f"24 B x / 48 B y per row",
                         "peak_source": "hbm_gbs, MEASURED_PEAKS.json"}
    # dominant kernel: largest isolated time (the work that bounds the step)
    dom = max(roofs, key=lambda k: phases_iso[k][0]) if roofs else max(phases, key=lambda k: phases[k][0])
    roof = dict(roofs.get(dom) or {"kernel": "k_" + dom})
    roof["share_of_step"] = phases[dom][0] / args.steps / ms_per_step if ms_per_step else None
    roof["share_of_isolated_sum"] = phases_iso[dom][0] / sum(v[0] for v in phases_iso.values())
    roof["others"] = {k: {kk: v[kk] for kk in ("kernel", "bound", "achieved", "peak", "unit", "frac", "traffic", "ms",
                                               "in_step", "issued", "frac_of_3xtf32_ceiling",
                                               "frac_of_fp32_simt_peak", "algorithmic", "format", "format_bytes",
                                               "format_frac", "frac_of_3xf16_ceiling", "note") if kk in v}
                      for k, v in roofs.items() if k != dom}

    line = {
        "metric": METRIC, "value": value, "unit": "Mpanels/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": CFG_NAMES[args.config], "n_panels": n, "p": 10, "leaf_max": args.leaf, "eta": 1.5,
                   "parallelism": parallelism_name(world),
                   "n_local": tree.n_local,
                   "l2": "flushed (256 MiB write) between timed steps",
                   "boxes": info["n_boxes"], "leaves": info["n_leaves"], "levels": info["n_levels"],
                   "m2l_translations": info["n_v_pairs"], "p2p_pairs": info["n_p2p"],
                   "x_pairs": info["n_x_pairs"], "w_pairs": info["n_w_pairs"], "near_nnz": nnz,
                   "setup_s": round(setup_s, 3), "tree_s": round(tree_s, 3), "context_s": round(context_s, 3)},
        "e2e": {"value": e2e_value, "unit": "Mpanels/s", "h2d_bytes_per_step": int(xh.numel() * 8),
                "d2h_bytes_per_step": int(yh.numel() * 8),
                "api": "xrl_mvm_host_batch over the timed steps (copies double-buffered against the MVMs)",
                "l2": "not flushed inside the batch; each step streams > 1.5 GB (near CSR + copies), above L2",
                "unpipelined_value": e2e_single,
                "unpipelined_api": "one blocking xrl_mvm_host call per step (L2 flushed between calls)"},
        "gpu_launches": launches,
        "clocks": clocks,
        "roofline": roof,
        "timing": {"ms_per_step_total_over_k": ms_per_step,
                   "ms_median": med_ms, "calls_in_median": len(med_calls),
                   "median_span_ms": sum(med_calls),
                   "value_from_median": n / (med_ms * 1e-3) / 1e6,
                   "note": "value = K steps total (contract); the SURVEY 8(d) median of >= 20 calls spanning >= 1 s "
                           "is beside it (rank-local on N > 1)"},
        "phases_ms_per_step": {k: v[0] / args.steps for k, v in phases.items()},
        "phases_isolated_ms": {k: v[0] / iso_steps for k, v in phases_iso.items()},
        "sched": "FMM chain on a high-priority stream; P2P then near SpMV on a low-priority side stream",
    }
    if world == 1 and args.gmres_iters > 0:
        line["gmres"] = gmres_iteration_time(xrl, tree, near, args)
    if world == 1 and not args.no_leaf64 and args.leaf != 64:
        line["leaf64"] = leaf64_line(xrl, mesh, x_user, ctx, dev, flush, args)
    if world == 1 and args.project > 1:
        line["multi_gpu_projection"] = multi_gpu_projection(xrl, mesh, ctx, x_lib, ms_per_step, args, args.project)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(mesh, x_user)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["xrl", "reference"], default="xrl")
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--leaf", type=int, default=384)  # tuned for config 4
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-leaf64", action="store_true", help="skip the leaf-64 line (N=1)")
    ap.add_argument("--project", type=int, default=8, help="virtual-rank projection to this many GPUs (N=1; 0 = off)")
    ap.add_argument("--gmres-iters", type=int, default=40, help="GMRES iteration-time probe (N=1); 0 = off")
    ap.add_argument("--gmres-solve", type=int, default=0, help="also solve to tolerance with this iteration cap")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    return run_xrl(args)


if __name__ == "__main__":
    sys.exit(main())
