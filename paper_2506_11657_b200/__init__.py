"""B200-native hot path of arxiv 2506.11657 (time-uniform shared-pole
rational approximation of the TEM forward problem).

The product is libtem_b200.so (sm_100a CUDA kernels behind the C ABI in
include/tem_b200.h); this package is its thin Python binding.  It never
imports the CPU oracle and has no CPU fallback.
"""
from .solver import RationalTable, TemForward  # noqa: F401

__all__ = ["RationalTable", "TemForward"]
