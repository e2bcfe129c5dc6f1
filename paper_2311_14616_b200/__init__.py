"""B200-native mixed-precision iterative refinement (arXiv 2311.14616 hot path).

The product is ``libmpir_gpu.so`` (hand-written sm_100a CUDA kernels + the
C++ host handle and refinement loop) behind the C-ABI ``include/mpir_gpu.h``.
``paper_2311_14616_b200.mpir`` mirrors the reference's Python module;
``paper_2311_14616_b200.kernels`` exposes the kernel-level entry points.
"""
from . import _lib  # noqa: F401
from ._lib import build, lib  # noqa: F401

__all__ = ["build", "lib", "mpir", "kernels"]
