"""paper_1410_0562_b200 -- B200-native set-bwte (arXiv 1410.0562) per-block insertion step.

The compute path is libsetbwte.so (hand-written sm_100a CUDA, C-ABI in
include/setbwte.h); ``SetBWTE`` is its ctypes binding.  Nothing here falls back
to the CPU.
"""
from .binding import EXPORTS, SetBWTE, SetBWTEError, load_library  # noqa: F401

__all__ = ["SetBWTE", "SetBWTEError", "load_library", "EXPORTS"]
