"""Build libxrl.so in-tree for sm_100a (nvcc, no JIT, no torch extension).

    python -m paper_2409_12375_b200.build [--force] [-v]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libxrl.so")
ROOT = os.path.dirname(HERE)

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fopenmp",
                  "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]
SOURCES = ["abi.cu", "tree.cu", "near.cu", "fmm.cu", "solver.cu", "comm.cu", "operators.cpp", "topology.cpp",
           "extract.cpp", "precond_exact.cu", "exchange.cu"]


def _nccl_dirs():
    """NCCL bundled with torch (the version torch.distributed loads), else the system one."""
    try:
        import nvidia.nccl as nn
        base = nn.__path__[0]
        if os.path.exists(os.path.join(base, "include", "nccl.h")):
            return os.path.join(base, "include"), os.path.join(base, "lib")
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


NCCL_INC, NCCL_LIB = _nccl_dirs()
CUFLAGS = CUFLAGS + ["-I" + NCCL_INC]
# tuning experiments only (e.g. "-DXRL_P2P_TPT=6"): extra flags for every translation unit
CUFLAGS = CUFLAGS + os.environ.get("XRL_EXTRA_NVCC", "").split()
HEADERS = ["xrl_internal.h", "harmonics.h", "operators.h", "tcgen05.h"]


def _stale(obj, src):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src] + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "xrl.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile(src, force, verbose):
    path = os.path.join(CSRC, src)
    obj = os.path.join(BUILD, src + ".o")
    if not force and not _stale(obj, path):
        return obj, ""
    cmd = [NVCC] + CUFLAGS + ["-c", path, "-o", obj]
    if verbose and src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        res = list(ex.map(lambda s: _compile(s, force, verbose), SOURCES))
    objs = [o for o, _ in res]
    if verbose:
        for o, log in res:
            if log:
                print(f"--- {os.path.basename(o)}\n{log}")
    if force or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-Xcompiler", "-fopenmp", "-o", LIB + ".tmp"] + objs + [
            "-lcudart", "-ldl", "-L" + NCCL_LIB, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + NCCL_LIB]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
