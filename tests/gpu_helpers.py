"""Shared helpers for the -m gpu tests: build the CUDA path for a mesh and run
the oracle on the same seeded inputs."""
import numpy as np

import oracle
from inputs import meshes


def cuda_setup(mesh, leaf_max=64, eta=oracle.ETA, galerkin=False):
    import torch
    from paper_2409_12375_b200 import build, xrl
    build.build()
    ctx = xrl.Context(0)
    tree = xrl.Tree(ctx, mesh.verts, mesh.tris, leaf_max=leaf_max)
    near = xrl.Near(tree, eta=eta, galerkin=galerkin)
    return ctx, tree, near


def run_mvm(tree, near, x_user: np.ndarray, flags=0):
    """x_user complex64 [nvec][n] in mesh order -> y complex64 [nvec][n] in mesh order (device path)."""
    import torch
    from paper_2409_12375_b200 import xrl
    xd = torch.from_numpy(x_user).cuda()
    xl = tree.to_library_order(xd)
    yl = xrl.mvm(tree, near, xl, flags=flags)
    y = tree.from_library_order(yl)
    torch.cuda.synchronize()
    return y.cpu().numpy()


def oracle_rows(mesh, x, rows=None, nthreads=0, galerkin=False):
    g = oracle.Geometry(mesh.verts, mesh.tris, galerkin=galerkin)
    return oracle.mvm_rows(g, x, rows, nthreads=nthreads)
