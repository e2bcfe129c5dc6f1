"""B200-native mixed-precision iterative refinement (arXiv 2311.14616 hot path).

The product is ``libmpir_gpu.so`` (hand-written sm_100a CUDA kernels + the
C++ host handle and refinement loop) behind the C-ABI ``include/mpir_gpu.h``.
``paper_2311_14616_b200.mpir`` mirrors the reference's Python module;
``paper_2311_14616_b200.kernels`` exposes the kernel-level entry points.
"""
import os as _os

# The LU runs its critical chain, bulk update, copy stream and late-column
# stream concurrently; with the default 8 hardware work queues, streams share
# queues and a stream waiting on a host-to-device chunk can hold up the
# critical chain. Effective only if set before the process creates its CUDA
# context (importing this package before the first CUDA call does that).
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from . import _lib  # noqa: F401,E402
from ._lib import build, lib  # noqa: F401,E402

__all__ = ["build", "lib", "mpir", "kernels"]
