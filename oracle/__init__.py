"""Parity checkers for the IR hot path -- TEST INFRASTRUCTURE ONLY.

Two CPU implementations with one numpy-facing interface:

* ``restatement()`` -- ``oracle/mpir_oracle.c`` (prefix ``orc_``), a plain-C
  restatement of the reference algorithm, built into ``oracle/build/``.
* ``reference()`` -- the unmodified reference headers compiled in place from
  ``/root/reference/proj`` (``oracle/ref_driver.cpp``, prefix ``ref_``), built
  into ``oracle/_ref/``. Absent on a box where it was never built.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
``--impl reference`` legs may import this package. The product path
(``paper_2311_14616_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libmpir_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmpir_ref.so")
REF_SRC = "/root/reference/proj"

B64, B32, B16 = 0, 1, 2
DTYPES = {B64: np.float64, B32: np.float32, B16: np.uint16}
STATUS = {0: "ok", 1: "OverflowDetected", 2: "SingularPivot", 3: "NonFiniteResult",
          4: "DimensionMismatch", 5: "InvalidConfig", 6: "InvalidParameter", 7: "Error"}
REASONS = ["SmallResidual", "SmallBackwardError", "ResidualStagnation",
           "CorrectionStagnation", "IterationLimit"]

_P = C.c_void_p
_I = C.c_int
_D = C.c_double
_IP = C.POINTER(C.c_int)
_DP = C.POINTER(C.c_double)


def build(ref: bool | None = None) -> None:
    """Compile the restatement (and the reference shim when its sources exist)."""
    targets = ["oracle"]
    if ref or (ref is None and os.path.isdir(os.path.join(REF_SRC, "include", "mpir"))):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _ptr(a):
    return a.ctypes.data_as(_P) if a is not None else None


def fmat(a, dtype=None):
    """Column-major (Fortran-order) view/copy, the storage of mpir::Matrix."""
    return np.asfortranarray(a if dtype is None else np.asarray(a).astype(dtype, copy=False))


class CpuImpl:
    """numpy wrapper over one of the two checker libraries."""

    def __init__(self, path: str, prefix: str):
        self.path = path
        self.prefix = prefix
        self.lib = C.CDLL(path)
        f = self._fn
        f("demote", _I, [_I, _I, C.c_size_t, _P, _P, _IP, _DP])
        f("one_norm", _D, [_I, _I, _I, _P])
        f("lu", _I, [_I, _I, _P, _IP, _IP, _IP])
        f("solve_mps", _I, [_I, _I, _I, _P, _IP, _P])
        f("solve_lps", _I, [_I, _I, _I, _P, _IP, _P, _P, _IP])
        f("residual", _I, [_I, _I, _I, _P, _P, _P, _P])
        if prefix == "orc_":
            f("ir", _I, [_I, _I, _I, _I, _I, _I, _P, _P, _D, _D, _D, _I, _P, _DP, _DP, _IP,
                         _IP, _IP, _P, _DP, _IP, _IP, _DP])
            f("f2h", C.c_uint16, [C.c_float])
            f("d2h", C.c_uint16, [C.c_double])
            f("h2f", C.c_float, [C.c_uint16])
            f("dlu_panel", _I, [_I, _I, _P, _I, _I, _IP, _IP, _IP, _IP])
            f("dlu_update", _I, [_I, _I, _P, _I, _I, _IP, _I, _I, _I, _I, _I, _I, _I, _IP])
        else:
            f("ir", _I, [_I, _I, _I, _I, _I, _I, _P, _P, _D, _D, _D, _I, _P, _DP, _DP, _IP,
                         _IP, _IP, _P, _DP, _IP, _IP, _DP, _DP, _DP])
            if hasattr(self.lib, "ref_krylov_ir"):
                f("krylov_ir", _I, [_I, _I, _I, _I, _I, _I, _I, _P, _P, _D, _D, _D, _I, _P, _DP,
                                    _DP, _IP, _IP, _IP, _IP])
            f("build_operator", None, [_I, _D, _DP])
            f("integral_rhs", None, [_I, _D, _DP])
            f("matvec_compensated_f64", None, [_I, _DP, _DP, _DP])
            f("half_from_double", C.c_uint16, [C.c_double])
            f("half_from_float", C.c_uint16, [C.c_float])
            f("half_to_float", C.c_float, [C.c_uint16])

    def _fn(self, name, res, args):
        fn = getattr(self.lib, self.prefix + name)
        fn.restype = res
        fn.argtypes = args
        setattr(self, "_" + name, fn)

    # -- kernels -----------------------------------------------------------
    def demote(self, src: np.ndarray, to: int):
        """Elementwise demotion in column-major storage order (matrices: order='F')."""
        frm = {np.dtype(np.float64): B64, np.dtype(np.float32): B32,
               np.dtype(np.uint16): B16}[src.dtype]
        src = fmat(src)
        dst = np.empty(src.shape, dtype=DTYPES[to], order="F")
        uf = C.c_int(0)
        bad = C.c_double(0.0)
        st = self._demote(frm, to, src.size, _ptr(src), _ptr(dst), C.byref(uf), C.byref(bad))
        return st, dst, bool(uf.value), bad.value

    def one_norm(self, a: np.ndarray, prec: int) -> float:
        rows, cols = a.shape
        return self._one_norm(prec, rows, cols, _ptr(fmat(a, DTYPES[prec])))

    def lu(self, a: np.ndarray, prec: int):
        """In-place LU of a copy of the (n, n) matrix a (any order; stored column-major)."""
        n = a.shape[0]
        a = np.array(a, dtype=DTYPES[prec], order="F", copy=True)
        ipiv = np.zeros(n, dtype=np.int32)
        perm = np.zeros(n, dtype=np.int32)
        sc = C.c_int(-1)
        st = self._lu(prec, n, _ptr(a), ipiv.ctypes.data_as(_IP), perm.ctypes.data_as(_IP),
                      C.byref(sc))
        return st, a, ipiv, perm, sc.value

    # -- blocked steps of the distributed LU (restatement only) ---------------
    def dlu_panel(self, prec, a_ptr, n, k0, jb, ipiv: np.ndarray, singular: list):
        """Panel step on a rank's n*n buffer at a_ptr; returns the (dst, src) moves."""
        moves = np.zeros(2 * 2 * jb, dtype=np.int32)
        nm = C.c_int(0)
        sc = C.c_int(singular[0])
        st = self._dlu_panel(prec, n, C.c_void_p(a_ptr), k0, jb, ipiv.ctypes.data_as(_IP),
                             moves.ctypes.data_as(_IP), C.byref(nm), C.byref(sc))
        assert st == 0
        singular[0] = sc.value
        return moves[: 2 * nm.value].reshape(-1, 2).copy()

    def dlu_update(self, prec, a_ptr, n, k0, jb, moves: np.ndarray, G, r, sh, cb, ce, left,
                   perm: np.ndarray | None):
        mv = np.ascontiguousarray(moves, dtype=np.int32).reshape(-1)
        st = self._dlu_update(prec, n, C.c_void_p(a_ptr), k0, jb, mv.ctypes.data_as(_IP),
                              mv.size // 2, G, r, sh, cb, ce, left,
                              None if perm is None else perm.ctypes.data_as(_IP))
        assert st == 0

    def solve_mps(self, ts, tf, packed, ipiv, x):
        x = np.array(x, dtype=DTYPES[ts], copy=True)
        st = self._solve_mps(ts, tf, x.size, _ptr(fmat(packed, DTYPES[tf])),
                             np.ascontiguousarray(ipiv, dtype=np.int32).ctypes.data_as(_IP),
                             _ptr(x))
        return st, x

    def solve_lps(self, tw, tf, packed, ipiv, r):
        r = np.array(r, dtype=DTYPES[tw], copy=True)
        scr = np.zeros(r.size, dtype=DTYPES[tf])
        uf = C.c_int(0)
        st = self._solve_lps(tw, tf, r.size, _ptr(fmat(packed, DTYPES[tf])),
                             np.ascontiguousarray(ipiv, dtype=np.int32).ctypes.data_as(_IP),
                             _ptr(r), _ptr(scr), C.byref(uf))
        return st, r, bool(uf.value)

    def residual(self, tw, tr, a, x, b):
        n = b.size
        r = np.zeros(n, dtype=DTYPES[tr])
        self._residual(tw, tr, n, _ptr(fmat(a, DTYPES[tw])),
                       _ptr(np.ascontiguousarray(x, dtype=DTYPES[tr])),
                       _ptr(np.ascontiguousarray(b, dtype=DTYPES[tw])), _ptr(r))
        return r

    def ir(self, tw, tf, tr, a, b, on_the_fly=-1, resid_term=True, cr=1.0, ce=1.0,
           rmax=0.5, litmax=10, want_packed=False):
        """MPFactorization<TW,TF,TR>(a) + ir_solve_report(f, b, tp)."""
        n = b.size
        a = fmat(a, DTYPES[tw])
        b = np.ascontiguousarray(b, dtype=DTYPES[tw])
        sol = np.zeros(n, dtype=DTYPES[tw])
        cap = max(litmax, 1) + 1
        rhist = np.zeros(cap)
        dhist = np.zeros(cap)
        rlen, reason, uf, sc = C.c_int(0), C.c_int(-1), C.c_int(0), C.c_int(-1)
        ipiv = np.zeros(n, dtype=np.int32)
        packed = np.zeros((n, n), dtype=DTYPES[tf], order="F") if want_packed else None
        anorm, bad = C.c_double(0.0), C.c_double(0.0)
        args = [tw, tf, tr, on_the_fly, int(resid_term), n, _ptr(a), _ptr(b), cr, ce, rmax,
                litmax, _ptr(sol), rhist.ctypes.data_as(_DP), dhist.ctypes.data_as(_DP),
                C.byref(rlen), C.byref(reason), ipiv.ctypes.data_as(_IP), _ptr(packed),
                C.byref(anorm), C.byref(uf), C.byref(sc), C.byref(bad)]
        tfac, tsol = C.c_double(0.0), C.c_double(0.0)
        if self.prefix == "ref_":
            args += [C.byref(tfac), C.byref(tsol)]
        st = self._ir(*args)
        k = rlen.value
        return {
            "status": STATUS.get(st, str(st)), "x": sol, "rhist": rhist[:k].copy(),
            "dhist": dhist[:max(k - 1, 0)].copy(),
            "reason": REASONS[reason.value] if st == 0 else None, "ipiv": ipiv,
            "packed": packed, "a_norm1": anorm.value, "underflow": bool(uf.value),
            "singular_col": sc.value, "bad_value": bad.value,
            "t_factor": tfac.value, "t_solve": tsol.value,
        }


    def krylov_ir(self, tw, tf, tr, a, b, kind="gmres", basissize=10, resid_term=True, cr=1.0,
                  ce=1.0, rmax=0.5, litmax=10):
        """MPFactorization(a, opts, kind, basissize) + krylov_ir_solve_report
        (compiled reference only)."""
        n = b.size
        a = fmat(a, DTYPES[tw])
        b = np.ascontiguousarray(b, dtype=DTYPES[tw])
        sol = np.zeros(n, dtype=DTYPES[tw])
        cap = max(litmax, 1) + 1
        rhist, dhist = np.zeros(cap), np.zeros(cap)
        khist = np.zeros(cap, dtype=np.int32)
        rlen, reason, brk = C.c_int(0), C.c_int(-1), C.c_int(0)
        st = self._krylov_ir(tw, tf, tr, {"gmres": 1, "bicgstab": 2}[kind], basissize,
                             int(resid_term), n, _ptr(a), _ptr(b), cr, ce, rmax, litmax,
                             _ptr(sol), rhist.ctypes.data_as(_DP), dhist.ctypes.data_as(_DP),
                             khist.ctypes.data_as(_IP), C.byref(rlen), C.byref(reason),
                             C.byref(brk))
        k = rlen.value
        return {"status": STATUS.get(st, str(st)), "x": sol, "rhist": rhist[:k].copy(),
                "dhist": dhist[:max(k - 1, 0)].copy(), "khist": khist[:max(k - 1, 0)].copy(),
                "reason": REASONS[reason.value] if st == 0 else None,
                "breakdown": bool(brk.value)}


_cache: dict = {}


def restatement() -> CpuImpl:
    if "orc" not in _cache:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        _cache["orc"] = CpuImpl(ORACLE_SO, "orc_")
    return _cache["orc"]


def reference(path: str = REF_SO) -> CpuImpl | None:
    """The compiled reference, or None when it was never built here."""
    if path not in _cache:
        if not os.path.exists(path):
            if os.path.isdir(os.path.join(REF_SRC, "include", "mpir")):
                build(ref=True)
            else:
                return None
        _cache[path] = CpuImpl(path, "ref_")
    return _cache[path]
