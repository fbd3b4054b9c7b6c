"""GMRES iteration counts: left / right block-Jacobi preconditioning vs none (coils, bar)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from inputs import meshes
from paper_2409_12375_b200 import xrl
from tests.gpu_helpers import cuda_setup
for name in ["coils", "bar"]:
    m = meshes.coils() if name == "coils" else meshes.bar()
    ctx, tree, near = cuda_setup(m)
    topo = xrl.Topology(tree, [(p, q) for _, p, q in m.ports])
    for f in ([1e6, 1e8, 1e10] if name == "coils" else [1e3, 1e6, 1e9]):
        kw = dict(sigma=5.8e7, zeta=5e-6) if name == "coils" else dict(sigma=5.8e7, zeta=1e-4)
        op = xrl.Operator(tree, near, topo, f, **kw)
        b = torch.zeros((len(m.ports), topo.n_loops), dtype=torch.complex64, device="cuda")
        for p in range(len(m.ports)):
            topo.port_rhs(p, 1.0, out=b[p:p + 1])
        for mode in ["none", "left64", "right64", "right32"]:
            pc = None if mode == "none" else xrl.Precond(op, int(mode[-2:]))
            t0 = time.time()
            x, rep = xrl.gmres(op, pc, b, max_iters=3000, right=mode.startswith("right"))
            torch.cuda.synchronize()
            print(f"{name} f={f:g} {mode:8s} iters={rep['iters']} rre={rep['rre']} true_rre={rep['true_rre']} t={time.time()-t0:.2f}s",
                  flush=True)
