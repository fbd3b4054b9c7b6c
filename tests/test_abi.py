"""CPU checks of the C-ABI boundary: the library loads, exports every symbol
include/xrl.h declares, and refuses to run without a GPU (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "xrl.h")


@pytest.fixture(scope="module")
def libxrl():
    from paper_2409_12375_b200 import build, xrl
    build.build()
    return xrl.lib()


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(xrl_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(libxrl):
    syms = declared_symbols()
    assert len(syms) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", libxrl._name], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(xrl_[a-z0-9_]+)\b", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    for s in syms:
        getattr(libxrl, s)


def test_binding_names_match_header():
    from paper_2409_12375_b200 import xrl
    assert sorted(xrl.EXPORTS) == [s for s in declared_symbols() if s in xrl.EXPORTS]
    assert set(xrl.EXPORTS) <= set(declared_symbols())


def test_sm100a_only_cubin(libxrl):
    out = subprocess.run(["cuobjdump", "--list-elf", libxrl._name], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_no_gpu_fails_loudly(libxrl):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    st = libxrl.xrl_ctx_create(0, None, 0, 1, None, ctypes.byref(h))
    assert st == -7  # XRL_ECUDA
    assert b"no CUDA device" in libxrl.xrl_last_error() or b"CUDA" in libxrl.xrl_last_error()


def test_argument_errors_are_synchronous(libxrl):
    # null handles are rejected before touching the device
    assert libxrl.xrl_mvm(None, None, None, None, 3, 0) == -1
    assert libxrl.xrl_tree_info(None, None) == -1
    assert libxrl.xrl_near_assemble(None, None, None) == -1
    assert libxrl.xrl_timing_count() == 9
