"""B200-native hot path of XRL (arXiv 2409.12375): FMM-accelerated panel MVM,
near-field correction and preconditioner behind a C-ABI (include/xrl.h).

The CUDA library libxrl.so is built in-tree by `paper_2409_12375_b200.build`;
`xrl` is the ctypes binding.  There is no CPU fallback.
"""
from . import xrl  # noqa: F401

__all__ = ["xrl"]
