"""Table IV analogue: GMRES iterations and times with the exact diag-of-P Q^-1
(xrl_precond_build_exact, host sparse LU) vs its block-Jacobi approximation (right preconditioning) vs
none, on the coil pair (config 2, 2 ports) and the DC-ish bar (config 1, 1 port)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from inputs import meshes  # noqa: E402
from paper_2409_12375_b200 import xrl  # noqa: E402
from tests.gpu_helpers import cuda_setup  # noqa: E402

for name in ["coils", "bar"]:
    m = meshes.coils() if name == "coils" else meshes.bar()
    ctx, tree, near = cuda_setup(m)
    topo = xrl.Topology(tree, [(p, q) for _, p, q in m.ports])
    print(f"{name}: panels {tree.info()['n']} loops {topo.n_loops}", flush=True)
    for f in ([1e6, 1e8, 1e10] if name == "coils" else [1e3, 1e6, 1e9]):
        kw = dict(sigma=5.8e7, zeta=5e-6) if name == "coils" else dict(sigma=5.8e7, zeta=1e-4)
        op = xrl.Operator(tree, near, topo, f, **kw)
        b = torch.zeros((len(m.ports), topo.n_loops), dtype=torch.complex64, device="cuda")
        for p in range(len(m.ports)):
            topo.port_rhs(p, 1.0, out=b[p:p + 1])
        for mode in ["none", "block64", "exact"]:
            t0 = time.time()
            pc = None if mode == "none" else xrl.Precond(op, 64, exact=(mode == "exact"))
            torch.cuda.synchronize()
            t1 = time.time()
            x, rep = xrl.gmres(op, pc, b, max_iters=3000)
            torch.cuda.synchronize()
            t2 = time.time()
            z = np.linalg.inv(topo.port_currents(x).T)
            print(f"{name} f={f:g} {mode:8s} iters={rep['iters']} true_rre={rep['true_rre']} "
                  f"setup={t1 - t0:.2f}s solve={t2 - t1:.2f}s Z00={z[0, 0]:.6g}", flush=True)
