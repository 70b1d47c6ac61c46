"""B200-native engine for the Concur / kvadmit simulator hot path.

The product is the in-tree native library `libkvgpu.so` (sm_100a CUDA kernels
behind the C ABI in include/kvgpu.h). This package is the Python mirror of the
reference interface over that ABI; it never computes simulations itself.
"""
from . import abi, config  # noqa: F401

__all__ = ["abi", "config", "engine"]
