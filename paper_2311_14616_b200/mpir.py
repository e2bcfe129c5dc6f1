"""Python mirror of the reference's ``mpir`` module over the B200 C-ABI.

Same names, keyword arguments, return dictionaries and exception types as the
reference pybind11 module (proj/python/bindings.cpp:126-290,
proj/python/mpir/__init__.py), so a reference user switches by changing the
import. Everything numeric runs on the GPU through libmpir_gpu.so:

* ``Factorization`` -> AnyFactorization (proj/src/runtime.cpp:67-134): float64
  input rounded once into the working precision (on the device, with the
  reference's overflow check), then MPFactorization<TW,TF,TR> on the device.
* ``Factorization.solve`` -> ir_solve_report (ir_engine.hpp:291-297).
* ``solve`` -> factor once and refine (bindings.cpp:221-240).

``krylov="gmres"`` / ``krylov="bicgstab"`` attach the reference's Krylov
workspace: ``solve`` is then krylov_ir_solve_report (krylov_ir.hpp:297-318)
with GMRES / BiCGSTAB corrections on the device, bitwise equal to the
reference, and the report carries ``khist``. ``direct_solve`` is not built
(SURVEY.md section 8(f)); it raises instead of silently running on the CPU.
"""
from __future__ import annotations

import ctypes as C
import math
import time

import numpy as np

from . import _lib as L
from ._lib import (B16, B32, B64, DimensionMismatch, Error, InvalidConfig,  # noqa: F401
                   InvalidParameter, InvalidSize, NonFiniteResult, NotConverged,
                   OverflowDetected, SingularPivot)

__version__ = "0.1.0"

_PARSE = {"b64": B64, "B64": B64, "double": B64, "f64": B64,
          "b32": B32, "B32": B32, "single": B32, "f32": B32,
          "b16": B16, "B16": B16, "half": B16, "f16": B16}
NAMES = {B64: "b64", B32: "b32", B16: "b16"}
NP_DTYPE = {B64: np.float64, B32: np.float32, B16: np.uint16}


def parse_precision(s: str) -> int:
    """precision.hpp:82-91."""
    if s not in _PARSE:
        raise InvalidParameter(f"unknown precision '{s}'")
    return _PARSE[s]


def machine_eps(precision: str) -> float:
    return L.lib().mpirg_machine_eps(parse_precision(precision))


def unit_roundoff(precision: str) -> float:
    return L.lib().mpirg_unit_roundoff(parse_precision(precision))


def resolve_config(tw: int, tf: int | None = None, tr: int | None = None,
                   on_the_fly: bool | None = None) -> L.mpirg_config:
    """resolve_config (mp_structures.hpp:44-59)."""
    cfg = L.mpirg_config()
    err = L.mpirg_error()
    st = L.lib().mpirg_resolve_config(tw, -1 if tf is None else tf, -1 if tr is None else tr,
                                      -1 if on_the_fly is None else int(on_the_fly),
                                      C.byref(cfg), C.byref(err))
    L.check(st, err)
    return cfg


def update_parms(cr=None, ce=None, rmax=None, litmax=None) -> L.mpirg_term_params:
    """update_parms (ir_engine.hpp:49-64)."""
    tp = L.mpirg_term_params()
    err = L.mpirg_error()
    nan = float("nan")
    if litmax is not None and litmax < 1:
        raise InvalidParameter("litmax must be at least 1")
    # NaN means "not given" at the C-ABI; an explicit NaN must fail validation
    # like the reference's TermParams::validate (ir_engine.hpp:40-45).
    for nm, v in (("cr", cr), ("ce", ce)):
        if v is not None and not (v == v):
            raise InvalidParameter(f"{nm} must be positive and finite")
    if rmax is not None and not (rmax == rmax):
        raise InvalidParameter("rmax must lie in (0, 1]")
    st = L.lib().mpirg_update_parms(nan if cr is None else float(cr),
                                    nan if ce is None else float(ce),
                                    nan if rmax is None else float(rmax),
                                    0 if litmax is None else int(litmax), C.byref(tp),
                                    C.byref(err))
    L.check(st, err)
    return tp


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise L.CudaError("no CUDA device available (the B200 path has no CPU fallback)")
    return torch


def _to_device_working(arr64: np.ndarray, tw: int):
    """Round float64 host data once into TW on the device (runtime.cpp:23-28,56-63)."""
    torch = _torch()
    src = torch.from_numpy(np.ascontiguousarray(arr64, dtype=np.float64)).cuda()
    if tw == B64:
        return src
    dst = torch.empty(src.shape, dtype=torch.float32, device=src.device)
    err = L.mpirg_error()
    st = L.lib().mpirg_demote(B64, B32, src.numel(), src.data_ptr(), dst.data_ptr(), None,
                              C.c_void_p(torch.cuda.current_stream().cuda_stream), C.byref(err))
    L.check(st, err)
    return dst


def _colmajor(a) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise DimensionMismatch("matrix must be two-dimensional")
    return np.ascontiguousarray(a.T)  # C-contiguous transpose == column-major storage


class Factorization:
    """A matrix bound to its low precision LU factors on the GPU
    (AnyFactorization, runtime.hpp:34-68)."""

    def __init__(self, a, *, working="double", factor=None, residual=None, on_the_fly=None,
                 resid_term=True, krylov=None, basissize=10, lu_mode="exact", nb=0,
                 device=None):
        kind = {None: 0, "none": 0, "gmres": 1, "bicgstab": 2}.get(
            krylov if krylov is None else str(krylov).lower(), -1)
        if kind < 0:
            raise InvalidParameter("unknown Krylov kind (gmres, bicgstab or none)")
        if kind and int(basissize) < 1:
            raise InvalidParameter("Krylov basis budget must be at least 1")
        cfg = resolve_config(parse_precision(working),
                             None if factor is None else parse_precision(factor),
                             None if residual is None else parse_precision(residual),
                             on_the_fly)
        cfg.resid_term = int(bool(resid_term))
        cfg.lu_mode = {"exact": L.LU_EXACT, "tc": L.LU_TC}[lu_mode]
        cfg.nb = int(nb)
        cfg.device = -1 if device is None else int(device)
        acm = _colmajor(a)
        if acm.shape[0] != acm.shape[1]:
            raise DimensionMismatch("matrix must be square")
        self._n = acm.shape[0]
        self._cfg = cfg
        dev = _to_device_working(acm, cfg.tw)
        self._h = C.c_void_p()
        err = L.mpirg_error()
        st = L.lib().mpirg_factorization_create(C.byref(self._h), self._n, C.byref(cfg),
                                                dev.data_ptr(), 1, C.byref(err))
        L.check(st, err)
        L.lib().mpirg_factorization_config(self._h, C.byref(self._cfg))
        self._krylov = kind
        if kind:
            L.check(L.lib().mpirg_factorization_enable_krylov(self._h, kind, int(basissize),
                                                              C.byref(err)), err)

    @classmethod
    def _allocate(cls, n: int, cfg) -> "Factorization":
        """A handle with buffers but no factorization yet (the distributed LU
        of config 5a fills it: mpirg_factorization_cast / _set_factored)."""
        self = cls.__new__(cls)
        self._n = n
        self._cfg = cfg
        self._krylov = 0
        self._h = C.c_void_p()
        err = L.mpirg_error()
        st = L.lib().mpirg_factorization_create(C.byref(self._h), n, C.byref(cfg), None, 1,
                                                C.byref(err))
        L.check(st, err)
        L.lib().mpirg_factorization_config(self._h, C.byref(self._cfg))
        return self

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            L.lib().mpirg_factorization_destroy(h)
            self._h = None

    # -- properties (bindings.cpp:153-172) ---------------------------------
    n = property(lambda self: self._n)
    working = property(lambda self: NAMES[self._cfg.tw])
    factor = property(lambda self: NAMES[self._cfg.tf])
    residual = property(lambda self: NAMES[self._cfg.tr])
    on_the_fly = property(lambda self: bool(self._cfg.on_the_fly))
    resid_term = property(lambda self: bool(self._cfg.resid_term))

    @property
    def a_norm1(self) -> float:
        return L.lib().mpirg_factorization_a_norm1(self._h)

    @property
    def demotion_underflowed(self) -> bool:
        return bool(L.lib().mpirg_factorization_demotion_underflowed(self._h))

    @property
    def matrix_bytes(self) -> int:
        return L.lib().mpirg_factorization_matrix_bytes(self._h)

    @property
    def last_factor_ms(self) -> float:
        return L.lib().mpirg_factorization_last_factor_ms(self._h)

    def ipiv(self) -> np.ndarray:
        out = np.zeros(self._n, dtype=np.int32)
        L.lib().mpirg_factorization_get_ipiv(self._h, out.ctypes.data)
        return out

    def pivots(self) -> np.ndarray:
        out = np.zeros(self._n, dtype=np.int32)
        L.lib().mpirg_factorization_get_pivots(self._h, out.ctypes.data)
        return out

    def packed_lu(self) -> np.ndarray:
        """Factor storage as an (n, n) array in the factor precision (binary16 as uint16 bits)."""
        out = np.zeros((self._n, self._n), dtype=NP_DTYPE[self._cfg.tf])
        L.lib().mpirg_factorization_get_packed_lu(self._h, out.ctypes.data)
        return out.T  # stored column-major

    def a_high(self) -> np.ndarray:
        out = np.zeros((self._n, self._n), dtype=NP_DTYPE[self._cfg.tw])
        L.lib().mpirg_factorization_get_a_high(self._h, out.ctypes.data)
        return out.T

    # -- solve ---------------------------------------------------------------
    def solve(self, b, *, cr=None, ce=None, rmax=None, litmax=None) -> dict:
        """Refine to working precision (bindings.cpp:174-189): returns
        {'x', 'rhist', 'dhist', 'khist', 'reason', 'seconds'}."""
        tp = update_parms(cr, ce, rmax, litmax)
        b = np.asarray(b, dtype=np.float64).reshape(-1)
        if b.size != self._n:
            raise DimensionMismatch("right-hand side length does not match the matrix")
        bdev = _to_device_working(b, self._cfg.tw)
        return self._solve_device(bdev, tp)

    def _solve_device(self, bdev, tp) -> dict:
        torch = _torch()
        sol = torch.empty(self._n, dtype=bdev.dtype, device=bdev.device)
        cap = tp.litmax + 1
        rh = (C.c_double * cap)()
        dh = (C.c_double * cap)()
        rep = L.mpirg_report(sol.data_ptr(), 1, rh, dh, cap, 0, 0, 0, 0.0)
        err = L.mpirg_error()
        t0 = time.perf_counter()
        st = L.lib().mpirg_ir_solve(self._h, bdev.data_ptr(), 1, C.byref(tp), C.byref(rep),
                                    C.byref(err))
        sec = time.perf_counter() - t0
        rhist = [rh[i] for i in range(rep.rhist_len)]
        dhist = [dh[i] for i in range(rep.dhist_len)]
        L.check(st, err, rhist=rhist, dhist=dhist)
        khist, breakdown = [], False
        if getattr(self, "_krylov", 0):
            kh = (C.c_int * cap)()
            klen, brk = C.c_int(0), C.c_int(0)
            L.lib().mpirg_factorization_last_khist(self._h, kh, cap, C.byref(klen), C.byref(brk))
            khist, breakdown = [kh[i] for i in range(min(klen.value, cap))], bool(brk.value)
        return {"x": sol.double().cpu().numpy(), "rhist": rhist, "dhist": dhist, "khist": khist,
                "breakdown": breakdown,
                "reason": L.REASONS[rep.reason], "seconds": sec, "device_ms": rep.solve_ms}

    def solve_many(self, bs, **kw) -> list:
        """Several right-hand sides against the one factorization: the columns of a
        2-D ``bs`` (or an iterable of vectors), one ir_solve_report each on the
        handle's reused buffers -- each report equals the single ``solve`` of its
        column bit for bit. (The reference has no multi-right-hand-side entry
        point: bindings.cpp:38 takes a 1-D b; its users loop exactly like this,
        test_mp_structures.cpp:141-196.)"""
        arr = np.asarray(bs, dtype=np.float64) if not isinstance(bs, (list, tuple)) else None
        cols = ([arr[:, j] for j in range(arr.shape[1])] if arr is not None and arr.ndim == 2
                else [arr] if arr is not None else list(bs))
        return [self.solve(np.ascontiguousarray(c), **kw) for c in cols]

    def refactor(self, a) -> None:
        """Refactor a new matrix of the same size in place (runtime.cpp:122-134)."""
        acm = _colmajor(a)
        if acm.shape != (self._n, self._n):
            raise DimensionMismatch("refactor matrix has a different shape")
        dev = _to_device_working(acm, self._cfg.tw)
        err = L.mpirg_error()
        st = L.lib().mpirg_factorization_refactor(self._h, dev.data_ptr(), 1, C.byref(err))
        L.check(st, err)

    def residual_tr(self, x, b) -> np.ndarray:
        """residual_tr (ir_engine.hpp:277-287): b - A x in the residual precision."""
        torch = _torch()
        xd = _to_device_working(np.asarray(x, dtype=np.float64), self._cfg.tw)
        bd = _to_device_working(np.asarray(b, dtype=np.float64), self._cfg.tw)
        r = torch.empty(self._n, dtype=torch.float64 if self._cfg.tr == B64 else torch.float32,
                        device=xd.device)
        err = L.mpirg_error()
        st = L.lib().mpirg_residual_tr(self._h, xd.data_ptr(), bd.data_ptr(), r.data_ptr(), 1,
                                       C.byref(err))
        L.check(st, err)
        return r.double().cpu().numpy()

    def direct_solve(self, b, *, method="gmres", maxiters=100, tol=1e-10):
        raise InvalidParameter("Krylov direct solves are not part of the B200 IR hot path")


def solve(a, b, *, working="double", factor=None, residual=None, on_the_fly=None,
          resid_term=True, krylov=None, basissize=10, cr=None, ce=None, rmax=None,
          litmax=None, **kw) -> dict:
    """Factor once and refine (bindings.cpp:221-240)."""
    tp = update_parms(cr, ce, rmax, litmax)  # validate before any allocation
    f = Factorization(a, working=working, factor=factor, residual=residual,
                      on_the_fly=on_the_fly, resid_term=resid_term, krylov=krylov,
                      basissize=basissize, **kw)
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    if b.size != f.n:
        raise DimensionMismatch("right-hand side length does not match the matrix")
    return f._solve_device(_to_device_working(b, f._cfg.tw), tp)


def batch_solve(a, b, *, working="double", factor=None, residual=None, on_the_fly=None,
                resid_term=True, cr=None, ce=None, rmax=None, litmax=None, device=None,
                devices=None, raise_on_error=True) -> list[dict]:
    """Config 5b: ``count`` independent systems, each exactly one
    MPFactorization + ir_solve_report (concurrent solves use
    separate objects). ``a``: (count, n, n) float64 (row-major matrices) or a
    CUDA tensor of TW holding count column-major n*n blocks; ``b``: (count, n).
    The systems run concurrently on the device (mpirg_batch_ir_solve).
    ``devices=[d0, d1, ...]`` (host arrays only) shards the batch one
    contiguous slice per listed GPU with no collective -- the slices run from
    one host thread each and the reports come back in system order."""
    torch = _torch()
    if devices is not None and len(devices) > 1:
        if isinstance(a, torch.Tensor):
            raise InvalidParameter("devices=[...] takes host arrays (each slice is copied to "
                                   "its own GPU)")
        from concurrent.futures import ThreadPoolExecutor

        from .dist import batch_slice
        a = np.asarray(a, dtype=np.float64)
        b = np.asarray(b, dtype=np.float64)
        count = a.shape[0]
        kw = dict(working=working, factor=factor, residual=residual, on_the_fly=on_the_fly,
                  resid_term=resid_term, cr=cr, ce=ce, rmax=rmax, litmax=litmax,
                  raise_on_error=raise_on_error)

        def one(i):
            lo, hi = batch_slice(count, len(devices), i)
            if hi <= lo:
                return []
            with torch.cuda.device(int(devices[i])):
                return batch_solve(a[lo:hi], b[lo:hi], device=int(devices[i]), **kw)
        with ThreadPoolExecutor(len(devices)) as ex:
            parts = list(ex.map(one, range(len(devices))))
        return [rep for part in parts for rep in part]
    if devices is not None and len(devices) == 1:
        device = devices[0]
    tp = update_parms(cr, ce, rmax, litmax)
    cfg = resolve_config(parse_precision(working),
                         None if factor is None else parse_precision(factor),
                         None if residual is None else parse_precision(residual), on_the_fly)
    cfg.resid_term = int(bool(resid_term))
    cfg.device = -1 if device is None else int(device)
    if isinstance(a, torch.Tensor):
        adev, bdev = a, b
        count = b.shape[0]
        n = b.shape[1]
    else:
        a = np.asarray(a, dtype=np.float64)
        if a.ndim != 3 or a.shape[1] != a.shape[2]:
            raise DimensionMismatch("batch matrices must be (count, n, n)")
        count, n = a.shape[0], a.shape[1]
        adev = _to_device_working(np.ascontiguousarray(np.transpose(a, (0, 2, 1))), cfg.tw)
        bdev = _to_device_working(np.asarray(b, dtype=np.float64).reshape(count, n), cfg.tw)
    sol = torch.empty((count, n), dtype=bdev.dtype, device=bdev.device)
    cap = tp.litmax + 1
    rh = np.zeros((count, cap))
    dh = np.zeros((count, cap))
    rlen = np.zeros(count, dtype=np.int32)
    reason = np.zeros(count, dtype=np.int32)
    status = np.zeros(count, dtype=np.int32)
    ms = C.c_double(0.0)
    err = L.mpirg_error()
    torch.cuda.current_stream().synchronize()
    st = L.lib().mpirg_batch_ir_solve(count, n, C.byref(cfg), adev.data_ptr(), bdev.data_ptr(),
                                      1, C.byref(tp), sol.data_ptr(), rh.ctypes.data,
                                      dh.ctypes.data, cap, rlen.ctypes.data,
                                      reason.ctypes.data, status.ctypes.data, C.byref(ms),
                                      C.byref(err))
    if st != 0 and raise_on_error:
        L.check(st, err)
    x = sol.double().cpu().numpy()
    out = []
    for i in range(count):
        k = int(rlen[i])
        out.append({"x": x[i], "rhist": list(rh[i, :k]), "dhist": list(dh[i, :max(k - 1, 0)]),
                    "khist": [], "status": int(status[i]),
                    "reason": L.REASONS[int(reason[i])] if status[i] == 0 else None})
    batch_solve.last_device_ms = ms.value
    return out


# ---- problem generators (greens.cpp; inputs, not the timed path) ----------
def build_operator(n: int, alpha: float) -> np.ndarray:
    """I - alpha*G (greens.cpp:48-59), bitwise the reference's."""
    if n < 3:
        raise InvalidSize("operator needs at least three grid points")
    out = np.empty((n, n), dtype=np.float64)  # column-major fill -> transpose view
    L.lib().mpirg_gen_greens_operator(n, float(alpha), out.ctypes.data)
    return out.T


def greens_matrix(n: int) -> np.ndarray:
    """G with trapezoid weights folded into the columns (greens.cpp:16-43).
    Elementwise products only, so numpy reproduces the reference bits."""
    if n < 3:
        raise InvalidSize("operator needs at least three grid points")
    h = 1.0 / (n - 1)
    x = np.arange(n, dtype=np.float64) * h
    x[n - 1] = 1.0
    w = np.full(n, h)
    w[0] = w[n - 1] = 0.5 * h
    xi, xj = x[:, None], x[None, :]
    g = np.where(xi > xj, xj * (1.0 - xi), xi * (1.0 - xj))
    return g * w[None, :]


def greens_problem(n: int, alpha: float, rhs: str = "manufactured") -> dict:
    """build_problem<double> (greens.hpp:52-69)."""
    a = build_operator(n, alpha)
    x = np.ones(n)
    if rhs == "manufactured":
        b = np.empty(n)
        acm = np.ascontiguousarray(a.T)
        L.lib().mpirg_gen_matvec_compensated_f64(n, acm.ctypes.data, x.ctypes.data,
                                                 b.ctypes.data)
        return {"a": a, "b": b, "x_exact": x}
    if rhs == "integral":
        b = np.empty(n)
        L.lib().mpirg_gen_integral_rhs(n, float(alpha), b.ctypes.data)
        return {"a": a, "b": b, "x_exact": x}
    raise InvalidParameter("rhs kind must be 'manufactured' or 'integral'")


__all__ = ["DimensionMismatch", "Factorization", "InvalidConfig", "InvalidParameter",
           "NonFiniteResult", "NotConverged", "OverflowDetected", "SingularPivot",
           "__version__", "batch_solve", "build_operator", "greens_matrix", "greens_problem",
           "machine_eps", "solve", "unit_roundoff", "resolve_config", "update_parms"]
