"""Table IV analogue: setup time and GMRES iterations of the diagonal-
of-P preconditioner (Eq. 10) against the traditional diagonal-of-L one, each as
block-Jacobi (64-loop blocks, GPU), as the whole Q factorised (host sparse LU, the paper's Pardiso
role) and as an incomplete LU(0) of the whole Q factorised on the GPU, plus no preconditioner, at the paper's Table IV tolerance 1e-6 (right preconditioning, restart 50).

    python tools/table4.py [--configs 1,2,4] [--freq 1e8] [--max-iters 1000] [--out file.json]

Right-hand sides: the unit port excitations where the config has ports (bar: 1, coils: 2), else one seeded
random loop vector (seed 1404, as bench.py's config-4 GMRES probe)."""
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

ZETA = {1: 100e-6, 2: 5e-6, 3: 20e-6, 4: 10e-6, 5: 20e-6}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,4")
    ap.add_argument("--freq", type=float, default=1e8)
    ap.add_argument("--tol", type=float, default=1e-6)
    ap.add_argument("--max-iters", type=int, default=1000)
    ap.add_argument("--out", default=None)
    ap.add_argument("--only-ilu", action="store_true")
    ap.add_argument("--only-exact", action="store_true")
    a = ap.parse_args()
    out = {"tol": a.tol, "freq_hz": a.freq, "restart": 50, "rows": []}
    for cfg in [int(c) for c in a.configs.split(",")]:
        m = meshes.make_config(cfg)
        ctx = xrl.Context(0)
        tree = xrl.Tree(ctx, m.verts, m.tris, leaf_max=64 if cfg <= 2 else 384)
        near = xrl.Near(tree)
        topo = xrl.Topology(tree, [(p, q) for _, p, q in m.ports])
        op = xrl.Operator(tree, near, topo, a.freq, sigma=5.8e7, zeta=ZETA[cfg])
        nl = topo.n_loops
        if m.ports:
            b = torch.zeros((len(m.ports), nl), dtype=torch.complex64, device="cuda")
            for p in range(len(m.ports)):
                topo.port_rhs(p, 1.0, out=b[p:p + 1])
            rhs = f"{len(m.ports)} unit port excitations"
        else:
            rng = np.random.default_rng(1404)
            b = torch.from_numpy((rng.random((1, nl)) - 0.5 + 1j * (rng.random((1, nl)) - 0.5)).astype(np.complex64)).cuda()
            rhs = "1 random loop vector (seed 1404)"
        for kind, exact in (("none", False), ("diag_p", False), ("diag_l", False), ("diag_p", True), ("diag_l", True),
                            ("diag_p", "ilu"), ("diag_l", "ilu")):
            if a.only_ilu and exact != "ilu":
                continue
            if a.only_exact and not (exact is True and kind == "diag_p"):
                continue
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            pc = None if kind == "none" else xrl.Precond(op, 64, exact=exact is True, kind=kind, ilu=exact == "ilu")
            torch.cuda.synchronize()
            setup = time.perf_counter() - t0
            t0 = time.perf_counter()
            x, rep = xrl.gmres(op, pc, b, tol=a.tol, max_iters=a.max_iters)
            torch.cuda.synchronize()
            solve = time.perf_counter() - t0
            row = {"config": cfg, "n_panels": m.n, "n_loops": nl, "rhs": rhs, "rre": [float(v) for v in rep["rre"]],
                   "preconditioner": kind + (" (ILU(0) on the GPU)" if exact == "ilu" else " (exact Q^-1)" if exact
                                             else " (block-Jacobi 64)" if kind != "none" else ""),
                   "setup_s": round(setup, 3), "iters": rep["iters"].tolist(), "converged": rep["converged"].tolist(),
                   "true_rre": [float(v) for v in rep["true_rre"]], "solve_s": round(solve, 3)}
            print(json.dumps(row), flush=True)
            out["rows"].append(row)
            del pc
        del op, topo, near, tree, ctx
        torch.cuda.empty_cache()
    if a.out:
        open(a.out, "w").write(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
