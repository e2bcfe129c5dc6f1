"""Kernel-level entry points of libmpir_gpu.so on torch CUDA tensors.

Thin wrappers used by the parity tests and the bench: each one forwards the
tensors' device pointers and the current torch stream to the C-ABI
(include/mpir_gpu.h) and raises the reference exception type on failure.
Column-major matrices are passed as C-contiguous tensors holding A^T.
"""
from __future__ import annotations

import ctypes as C

from . import _lib as L
from ._lib import B16, B32, B64  # noqa: F401

_TORCH_PREC = {}


def _prec(t) -> int:
    import torch
    if not _TORCH_PREC:
        _TORCH_PREC.update({torch.float64: B64, torch.float32: B32, torch.float16: B16,
                            torch.int16: B16})
    return _TORCH_PREC[t.dtype]


def _stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def demote(src, dst) -> bool:
    """demote_matrix_into (matrix.hpp:74-85); returns the underflow flag."""
    err, uf = L.mpirg_error(), C.c_int(0)
    st = L.lib().mpirg_demote(_prec(src), _prec(dst), src.numel(), src.data_ptr(),
                              dst.data_ptr(), C.byref(uf), _stream(), C.byref(err))
    L.check(st, err)
    return bool(uf.value)


def one_norm(a_cm, rows: int, cols: int) -> float:
    """matrix_one_norm (mp_structures.hpp:22-36) of a column-major rows x cols matrix."""
    err, out = L.mpirg_error(), C.c_double(0.0)
    st = L.lib().mpirg_one_norm(_prec(a_cm), rows, cols, a_cm.data_ptr(), C.byref(out),
                                _stream(), C.byref(err))
    L.check(st, err)
    return out.value


def lu_factor(a_cm, ipiv, n: int, lu_mode: int = L.LU_EXACT, nb: int = 0) -> None:
    """lu_factor / lu_factor_half (dense_lu.hpp:151-171), in place."""
    err = L.mpirg_error()
    st = L.lib().mpirg_lu_factor(_prec(a_cm), n, a_cm.data_ptr(), ipiv.data_ptr(), lu_mode, nb,
                                 _stream(), C.byref(err))
    L.check(st, err)


def solve_mps(packed_cm, ipiv, x, tf: int | None = None) -> None:
    """solve_mps_into<TS,TF> (dense_lu.hpp:175-182), in place on x."""
    err = L.mpirg_error()
    st = L.lib().mpirg_solve_mps(_prec(x), _prec(packed_cm) if tf is None else tf, x.numel(),
                                 packed_cm.data_ptr(), ipiv.data_ptr(), x.data_ptr(), _stream(),
                                 C.byref(err))
    L.check(st, err)


def solve_lps(packed_cm, ipiv, r, scratch, tf: int | None = None) -> bool:
    """solve_lps_into<TW,TF> (dense_lu.hpp:204-232), in place on r; returns underflow."""
    err, uf = L.mpirg_error(), C.c_int(0)
    st = L.lib().mpirg_solve_lps(_prec(r), _prec(packed_cm) if tf is None else tf, r.numel(),
                                 packed_cm.data_ptr(), ipiv.data_ptr(), r.data_ptr(),
                                 scratch.data_ptr(), C.byref(uf), _stream(), C.byref(err))
    L.check(st, err)
    return bool(uf.value)


def residual(a_cm, x, b, r) -> None:
    """detail::residual_into<TW,TR> (ir_engine.hpp:115-139)."""
    err = L.mpirg_error()
    st = L.lib().mpirg_residual(_prec(a_cm), _prec(r), r.numel(), a_cm.data_ptr(), x.data_ptr(),
                                b.data_ptr(), r.data_ptr(), _stream(), C.byref(err))
    L.check(st, err)
