"""ctypes binding of the C-ABI in include/mpir_gpu.h (libmpir_gpu.so).

The shared library is built in-tree (``paper_2311_14616_b200/libmpir_gpu.so``)
by ``__graft_entry__.build()`` / ``make -C paper_2311_14616_b200/csrc``. There
is no CPU fallback: when the library is missing this module raises, and when
no GPU is visible every compute call returns MPIRG_ERR_CUDA.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
# MPIRG_LIB selects an in-tree build variant (e.g. the instrumented panel build
# of tools/); default: the product library.
LIB_PATH = os.path.join(HERE, os.environ.get("MPIRG_LIB", "libmpir_gpu.so"))
HEADER = os.path.join(os.path.dirname(HERE), "include", "mpir_gpu.h")

B64, B32, B16 = 0, 1, 2
LU_EXACT, LU_TC = 0, 1
KERNEL_CLASSES = ["cast", "panel", "moves", "trsm", "gemm", "trsv_lower", "trsv_upper",
                  "residual", "vector"]
REASONS = ["SmallResidual", "SmallBackwardError", "ResidualStagnation",
           "CorrectionStagnation", "IterationLimit"]


class Error(RuntimeError):
    """mpir::Error (errors.hpp:14-18)."""


class OverflowDetected(OverflowError, Error):
    pass


class SingularPivot(ArithmeticError, Error):
    def __init__(self, msg, column=-1):
        super().__init__(msg)
        self.column = column


class NonFiniteResult(ArithmeticError, Error):
    def __init__(self, msg, rhist=(), dhist=(), khist=()):
        super().__init__(msg)
        self.rhist = list(rhist)
        self.dhist = list(dhist)
        self.khist = list(khist)


class DimensionMismatch(ValueError, Error):
    pass


class InvalidConfig(ValueError, Error):
    pass


class InvalidParameter(ValueError, Error):
    pass


class InvalidSize(ValueError, Error):
    pass


class NotConverged(Error):
    pass


class CudaError(Error):
    pass


STATUS_EXC = {1: OverflowDetected, 2: SingularPivot, 3: NonFiniteResult, 4: DimensionMismatch,
              5: InvalidConfig, 6: InvalidParameter, 7: InvalidSize, 8: CudaError, 9: CudaError}


class mpirg_error(C.Structure):
    _fields_ = [("status", C.c_int), ("column", C.c_int), ("value", C.c_double),
                ("message", C.c_char * 256)]


class mpirg_config(C.Structure):
    _fields_ = [("tw", C.c_int), ("tf", C.c_int), ("tr", C.c_int), ("on_the_fly", C.c_int),
                ("resid_term", C.c_int), ("lu_mode", C.c_int), ("nb", C.c_int),
                ("device", C.c_int)]


class mpirg_term_params(C.Structure):
    _fields_ = [("cr", C.c_double), ("ce", C.c_double), ("rmax", C.c_double),
                ("litmax", C.c_int)]


class mpirg_report(C.Structure):
    _fields_ = [("sol", C.c_void_p), ("sol_on_device", C.c_int),
                ("rhist", C.POINTER(C.c_double)), ("dhist", C.POINTER(C.c_double)),
                ("hist_capacity", C.c_int), ("rhist_len", C.c_int), ("dhist_len", C.c_int),
                ("reason", C.c_int), ("solve_ms", C.c_double)]


_P, _I, _D, _S = C.c_void_p, C.c_int, C.c_double, C.c_size_t
_E = C.POINTER(mpirg_error)
_H = C.c_void_p  # opaque mpirg_factorization*

PROTOTYPES = {
    "mpirg_abi_version": (_I, []),
    "mpirg_device_count": (_I, []),
    "mpirg_resolve_config": (_I, [_I, _I, _I, _I, C.POINTER(mpirg_config), _E]),
    "mpirg_update_parms": (_I, [_D, _D, _D, _I, C.POINTER(mpirg_term_params), _E]),
    "mpirg_machine_eps": (_D, [_I]),
    "mpirg_unit_roundoff": (_D, [_I]),
    "mpirg_factorization_create": (_I, [C.POINTER(_H), _I, C.POINTER(mpirg_config), _P, _I, _E]),
    "mpirg_factorization_refactor": (_I, [_H, _P, _I, _E]),
    "mpirg_factorization_destroy": (None, [_H]),
    "mpirg_factorization_n": (_I, [_H]),
    "mpirg_factorization_config": (_I, [_H, C.POINTER(mpirg_config)]),
    "mpirg_factorization_a_norm1": (_D, [_H]),
    "mpirg_factorization_demotion_underflowed": (_I, [_H]),
    "mpirg_factorization_matrix_bytes": (_S, [_H]),
    "mpirg_factorization_last_factor_ms": (_D, [_H]),
    "mpirg_factorization_get_ipiv": (_I, [_H, _P]),
    "mpirg_factorization_get_pivots": (_I, [_H, _P]),
    "mpirg_factorization_get_packed_lu": (_I, [_H, _P]),
    "mpirg_factorization_get_a_high": (_I, [_H, _P]),
    "mpirg_factorization_a_high_device": (_P, [_H]),
    "mpirg_factorization_packed_lu_device": (_P, [_H]),
    "mpirg_factorization_ipiv_device": (_P, [_H]),
    "mpirg_factorization_stream": (_P, [_H]),
    "mpirg_factorization_residual_buf_device": (_P, [_H]),
    "mpirg_factorization_sol_buf_device": (_P, [_H]),
    "mpirg_factorization_comp_buf_device": (_P, [_H]),
    "mpirg_factorization_low_buf_device": (_P, [_H]),
    "mpirg_factorization_work_buf_device": (_P, [_H]),
    "mpirg_ir_solve": (_I, [_H, _P, _I, C.POINTER(mpirg_term_params), C.POINTER(mpirg_report), _E]),
    "mpirg_residual_tr": (_I, [_H, _P, _P, _P, _I, _E]),
    "mpirg_factorization_enable_krylov": (_I, [_H, _I, _I, _E]),
    "mpirg_factorization_last_khist": (_I, [_H, C.POINTER(C.c_int), _I, C.POINTER(C.c_int),
                                            C.POINTER(C.c_int)]),
    "mpirg_demote": (_I, [_I, _I, _S, _P, _P, C.POINTER(C.c_int), _P, _E]),
    "mpirg_one_norm": (_I, [_I, _I, _I, _P, C.POINTER(C.c_double), _P, _E]),
    "mpirg_lu_factor": (_I, [_I, _I, _P, _P, _I, _I, _P, _E]),
    "mpirg_solve_mps": (_I, [_I, _I, _I, _P, _P, _P, _P, _E]),
    "mpirg_solve_lps": (_I, [_I, _I, _I, _P, _P, _P, _P, C.POINTER(C.c_int), _P, _E]),
    "mpirg_residual": (_I, [_I, _I, _I, _P, _P, _P, _P, _P, _E]),
    "mpirg_factorization_cast": (_I, [_H, _P, _I, _E]),
    "mpirg_factorization_buffers": (_I, [_H, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                         C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "mpirg_factorization_set_factored": (_I, [_H, _I, _E]),
    "mpirg_tc_update": (_I, [_I, _P, _I, _I, _I, _P, _E]),
    "mpirg_tc_gemm": (_I, [_I, _P, _I, _I, _I, _I, _I, _I, _P, _E]),
    "mpirg_dlu_create": (_I, [C.POINTER(_H), _I, _I, _I, _I, _I, _I, _I, _E]),
    "mpirg_dlu_destroy": (None, [_H]),
    "mpirg_dlu_nb": (_I, [_H]),
    "mpirg_dlu_npanels": (_I, [_H]),
    "mpirg_dlu_block_cols": (_I, [_H]),
    "mpirg_dlu_owner": (_I, [_H, _I]),
    "mpirg_dlu_msg_bytes": (_S, [_H, _I]),
    "mpirg_dlu_begin": (_I, [_H, _P, _P, _E]),
    "mpirg_dlu_panel": (_I, [_H, _P, _I, _P, _P, _E]),
    "mpirg_dlu_pack": (_I, [_H, _P, _I, _P, _P, _P, _E]),
    "mpirg_dlu_unpack": (_I, [_H, _P, _I, _P, _P, _P, _E]),
    "mpirg_dlu_update": (_I, [_H, _P, _I, _I, _P, _P, _E]),
    "mpirg_dlu_end": (_I, [_H, _P, C.POINTER(C.c_int), _E]),
    "mpirg_dlu_factor": (_I, [_H, _P, _P, _P, _P, _P, _P, C.POINTER(C.c_int), _E]),
    "mpirg_comm_unique_id": (_I, [_P, _E]),
    "mpirg_comm_create": (_I, [C.POINTER(_H), _I, _I, _P, _I, _E]),
    "mpirg_comm_destroy": (None, [_H]),
    "mpirg_comm_nranks": (_I, [_H]),
    "mpirg_comm_rank": (_I, [_H]),
    "mpirg_comm_version": (_I, []),
    "mpirg_comm_bcast": (_I, [_P, _P, _S, _I, _P]),
    "mpirg_comm_send": (_I, [_H, _P, _S, _I, _P]),
    "mpirg_comm_recv": (_I, [_H, _P, _S, _I, _P]),
    "mpirg_batch_ir_solve": (_I, [_I, _I, C.POINTER(mpirg_config), _P, _P, _I,
                                  C.POINTER(mpirg_term_params), _P, _P, _P, _I, _P, _P, _P,
                                  C.POINTER(C.c_double), _E]),
    "mpirg_profile_enable": (None, [_I]),
    "mpirg_profile_collect": (_I, [C.POINTER(C.c_double), C.POINTER(C.c_int), _I]),
    "mpirg_ffma_peak": (_I, [C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "mpirg_ubench_gemm_f32": (_I, [_I, _I, _I, _I, C.POINTER(C.c_double),
                                   C.POINTER(C.c_double)]),
    "mpirg_dfma_peak": (_I, [C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "mpirg_fma_latency": (_I, [_I, C.POINTER(C.c_double)]),
    "mpirg_check_fast_div": (_I, [C.c_int, C.c_ulonglong, C.c_longlong,
                                  C.POINTER(C.c_longlong), C.POINTER(C.c_double)]),
    "mpirg_gen_uniform_matrix": (None, [_I, _I, C.c_uint64, _D, _D, _P]),
    "mpirg_gen_normal_matrix": (None, [_I, _I, C.c_uint64, _P]),
    "mpirg_gen_diag_dominant": (None, [_I, C.c_uint64, _D, _P]),
    "mpirg_gen_greens_operator": (None, [_I, _D, _P]),
    "mpirg_gen_integral_rhs": (None, [_I, _D, _P]),
    "mpirg_gen_greens_operator_device": (_I, [_I, _D, _I, _I, _P, _S, _P]),
    "mpirg_gen_matvec_compensated_f64": (None, [_I, _P, _P, _P]),
}

# mpirg_bcast_fn: the distributed LU's broadcast hook
BCAST_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p)

_lib = None


def build() -> None:
    """Compile the CUDA extension in-tree for sm_100a."""
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "csrc"), "-j8"], check=True)


def lib() -> C.CDLL:
    """Load libmpir_gpu.so (fails loudly when it is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing; build it with __graft_entry__.build() or "
                "`make -C paper_2311_14616_b200/csrc` (the IR path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.mpirg_abi_version() != 1:
            raise ImportError("libmpir_gpu.so ABI version mismatch")
        _lib = L
    return _lib


def check(status: int, err: mpirg_error, **extra) -> None:
    """Raise the Python twin of the reference exception for a non-OK status."""
    if status == 0:
        return
    msg = err.message.decode(errors="replace")
    exc = STATUS_EXC.get(status, Error)
    if exc is SingularPivot:
        raise SingularPivot(msg, err.column)
    if exc is NonFiniteResult:
        raise NonFiniteResult(msg, extra.get("rhist", ()), extra.get("dhist", ()))
    e = exc(msg)
    if exc is OverflowDetected:
        e.value = err.value
    raise e
