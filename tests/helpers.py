"""Shared helpers for the parity tests (numpy <-> column-major device buffers)."""
from __future__ import annotations

import ctypes as C

import numpy as np

B64, B32, B16 = 0, 1, 2
NP = {B64: np.float64, B32: np.float32, B16: np.uint16}


def gen_lib():
    import paper_2311_14616_b200 as p
    return p.lib()


def greens(n: int, alpha: float) -> np.ndarray:
    """A = I - alpha G as an (n, n) Fortran-order float64 array."""
    out = np.empty((n, n), dtype=np.float64, order="F")
    gen_lib().mpirg_gen_greens_operator(n, float(alpha), out.ctypes.data)
    return out


def normal_matrix(n: int, seed: int) -> np.ndarray:
    out = np.empty((n, n), dtype=np.float64, order="F")
    gen_lib().mpirg_gen_normal_matrix(n, n, seed, out.ctypes.data)
    return out


def uniform_matrix(n: int, seed: int, lo=-1.0, hi=1.0) -> np.ndarray:
    out = np.empty((n, n), dtype=np.float64, order="F")
    gen_lib().mpirg_gen_uniform_matrix(n, n, seed, lo, hi, out.ctypes.data)
    return out


def diag_dominant(n: int, seed: int, shift: float) -> np.ndarray:
    out = np.empty((n, n), dtype=np.float64, order="F")
    gen_lib().mpirg_gen_diag_dominant(n, seed, shift, out.ctypes.data)
    return out


def normal_vector(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    gen_lib().mpirg_gen_normal_matrix(n, 1, seed, out.ctypes.data)
    return out


def uniform_vector(n: int, seed: int, lo=-1.0, hi=1.0) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    gen_lib().mpirg_gen_uniform_matrix(n, 1, seed, lo, hi, out.ctypes.data)
    return out


def to_dev(a: np.ndarray):
    """Host array (matrix: any order) -> torch CUDA tensor holding column-major storage."""
    import torch
    if a.ndim == 2:
        buf = np.ascontiguousarray(np.asfortranarray(a).T)
    else:
        buf = np.ascontiguousarray(a)
    if buf.dtype == np.uint16:
        return torch.from_numpy(buf.view(np.int16)).cuda()
    return torch.from_numpy(buf).cuda()


def from_dev(t, shape=None, dtype=None) -> np.ndarray:
    """torch CUDA tensor (column-major storage) -> numpy (Fortran order for matrices)."""
    h = t.cpu().numpy()
    if h.dtype == np.int16:
        h = h.view(np.uint16)
    if dtype is not None:
        h = h.view(dtype)
    if h.ndim == 2:
        return np.asfortranarray(h.T)
    return h


def bits(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(np.asfortranarray(a).T) if a.ndim == 2 else np.ascontiguousarray(a)
    return a.view({8: np.uint64, 4: np.uint32, 2: np.uint16}[a.dtype.itemsize])


def same_bits(a: np.ndarray, b: np.ndarray, nan_equal=True) -> bool:
    """Bitwise equality, with every NaN equal to every NaN when nan_equal."""
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    if a.dtype == np.uint16:
        ha, hb = bits(a), bits(b)
        if nan_equal:
            na = ((ha & 0x7C00) == 0x7C00) & ((ha & 0x3FF) != 0)
            nb = ((hb & 0x7C00) == 0x7C00) & ((hb & 0x3FF) != 0)
            return bool(np.array_equal(na, nb) and np.array_equal(ha[~na], hb[~nb]))
        return bool(np.array_equal(ha, hb))
    ba, bb = bits(a), bits(b)
    if nan_equal:
        na, nb = np.isnan(np.asarray(a).ravel(order="F")), np.isnan(np.asarray(b).ravel(order="F"))
        return bool(np.array_equal(na, nb) and np.array_equal(ba.ravel()[~na], bb.ravel()[~nb]))
    return bool(np.array_equal(ba, bb))


def demote_host(a64: np.ndarray, to: int) -> np.ndarray:
    import oracle
    st, out, _, _ = oracle.restatement().demote(np.asfortranarray(a64), to)
    assert st == 0
    return out
