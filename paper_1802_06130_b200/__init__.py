"""B200-native (sm_100a) inference hot path of multiscale BLADE denoising (arxiv 1802.06130).

The compute lives in `libblade_ms.so` (hand-written CUDA kernels behind the C ABI of
`include/blade_ms.h`); `blade_ms.BladeMS` is a thin ctypes binding over it.
"""
from .blade_ms import BladeError, BladeMS, lib, library_path  # noqa: F401

__all__ = ["BladeMS", "BladeError", "lib", "library_path"]
