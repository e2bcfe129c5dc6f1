"""The C-ABI boundary (CPU only): the library loads, exports exactly what
include/mpir_gpu.h declares, validates like the reference before any device
work, and has no CPU fallback."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

import paper_2311_14616_b200 as pkg
from paper_2311_14616_b200 import _lib as L
from paper_2311_14616_b200 import mpir

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "mpir_gpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mpirg_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = pkg.lib()
    syms = declared_symbols()
    assert len(syms) > 40
    for s in syms:
        assert hasattr(lib, s), s
    # and the Python binding covers all of them
    assert set(syms) <= set(L.PROTOTYPES)


def test_abi_version_and_no_gpu_here():
    lib = pkg.lib()
    assert lib.mpirg_abi_version() == 1
    assert lib.mpirg_device_count() >= 0


def test_library_is_sm100a():
    """The shipped library carries sm_100a SASS (no PTX-JIT or other-arch fallback)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", L.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_resolve_config_matches_reference():
    """test_mp_structures.cpp:17-48 (resolve_config defaults + validation)."""
    c = mpir.resolve_config(0)
    assert (c.tf, c.tr, c.on_the_fly) == (1, 0, 0)
    c = mpir.resolve_config(1)
    assert (c.tf, c.tr, c.on_the_fly) == (2, 1, 1)
    assert mpir.resolve_config(0, 2).on_the_fly == 1
    assert mpir.resolve_config(0, 0).on_the_fly == 1
    assert mpir.resolve_config(1, 1, None, False).on_the_fly == 1
    c = mpir.resolve_config(1, None, 0)
    assert (c.tf, c.tr, c.on_the_fly) == (2, 0, 1)
    assert mpir.resolve_config(0, 1, None, True).on_the_fly == 1
    for bad in [(2,), (1, 0), (0, None, 1)]:
        with pytest.raises(mpir.InvalidConfig):
            mpir.resolve_config(*bad)


def test_term_params_match_reference():
    """test_ir_engine.cpp:46-74."""
    t = mpir.update_parms()
    assert (t.cr, t.ce, t.rmax, t.litmax) == (1.0, 1.0, 0.5, 10)
    t = mpir.update_parms(2.0, 5.0, 0.25, 4)
    assert (t.cr, t.ce, t.rmax, t.litmax) == (2.0, 5.0, 0.25, 4)
    for kw in [dict(cr=0.0), dict(cr=-1.0), dict(ce=0.0), dict(rmax=0.0), dict(rmax=1.5),
               dict(litmax=0), dict(cr=math.nan)]:
        with pytest.raises(mpir.InvalidParameter):
            mpir.update_parms(**kw)
    mpir.update_parms(rmax=1.0, litmax=1)


def test_eps_constants():
    """tests/python/test_smoke.py::test_eps_constants."""
    assert mpir.machine_eps("double") == 2.0 ** -52
    assert mpir.machine_eps("single") == 2.0 ** -23
    assert mpir.machine_eps("half") == 2.0 ** -10
    assert mpir.unit_roundoff("double") == 2.0 ** -53
    with pytest.raises(mpir.InvalidParameter):
        mpir.machine_eps("b128")


def test_validation_precedes_device_work():
    """Shape/config/parameter errors surface as the reference's ValueError
    subclasses before any GPU call (test_smoke.py::test_validation_errors)."""
    a = np.eye(4)
    with pytest.raises(ValueError):
        mpir.solve(a[:, :-1], np.ones(4))
    with pytest.raises(ValueError):
        mpir.solve(a, np.ones(4), working="single", factor="double")
    with pytest.raises(ValueError):
        mpir.solve(a, np.ones(4), rmax=0.0)


def test_no_cpu_fallback():
    """Without a GPU the compute entry points fail loudly (MPIRG_ERR_CUDA)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = pkg.lib()
    cfg = L.mpirg_config(0, 1, 0, -1, 1, 0, 0, -1)
    h = C.c_void_p()
    err = L.mpirg_error()
    a = np.eye(8)
    st = lib.mpirg_factorization_create(C.byref(h), 8, C.byref(cfg), a.ctypes.data, 0,
                                        C.byref(err))
    assert st == 8 and not h  # MPIRG_ERR_CUDA, nothing computed
    assert b"no CUDA device" in err.message
    with pytest.raises(L.CudaError):
        mpir.solve(np.eye(8), np.ones(8), factor="single")


def test_generators_match_reference(ref):
    """The seeded Green's operator and compensated matvec are the reference's bits."""
    from paper_2311_14616_b200 import configs
    for n, alpha in [(64, 1.0), (257, 800.0)]:
        a = configs.greens(n, alpha)
        r = np.empty(n * n)
        ref._build_operator(n, alpha, r.ctypes.data_as(C.POINTER(C.c_double)))
        assert a.tobytes() == r.tobytes()
        x = np.linspace(-1, 1, n)
        y1 = np.empty(n)
        y2 = np.empty(n)
        pkg.lib().mpirg_gen_matvec_compensated_f64(n, a.ctypes.data, x.ctypes.data, y1.ctypes.data)
        ref._matvec_compensated_f64(n, a.ctypes.data_as(C.POINTER(C.c_double)),
                                    x.ctypes.data_as(C.POINTER(C.c_double)),
                                    y2.ctypes.data_as(C.POINTER(C.c_double)))
        assert y1.tobytes() == y2.tobytes()
    rhs = np.empty(100)
    ref._integral_rhs(100, 799.0, rhs.ctypes.data_as(C.POINTER(C.c_double)))
    mine = mpir.greens_problem(100, 799.0, "integral")["b"]
    assert mine.tobytes() == rhs.tobytes()


def test_greens_matrix_matches_reference_kernel():
    g = mpir.greens_matrix(9)
    a = mpir.build_operator(9, 1.0)
    off = ~np.eye(9, dtype=bool)
    assert np.array_equal(-g[off], a[off])
    assert np.all(g[0] == 0) and np.all(g[-1] == 0) and np.all(g[:, 0] == 0)
