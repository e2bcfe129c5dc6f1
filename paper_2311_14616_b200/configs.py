"""The BASELINE.json workloads as seeded inputs.

Inputs only -- not the timed path. Every matrix is generated on the host by
the shared C generators (libstdc++ std::mt19937_64 + <random>, column-major
fill, restating proj/tests/support/test_support.hpp:17-46 and
proj/src/greens.cpp:11-68), so the GPU path, the C oracle and the compiled
reference consume byte-identical inputs.

Each config returns a dict: a (column-major storage as an (n, n) C array of
A^T, float64), b (float64), the precision triple, solver options and the
termination parameters the reference is run with.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

B64, B32, B16 = 0, 1, 2

# n used by BASELINE.json for each config
FULL_N = {"cfg1": 4096, "cfg2a": 4096, "cfg2b": 4096, "cfg3": 8192, "cfg4": 16384,
          "cfg5a": 65536, "cfg5b": 1024}


_GEN = None


def _gen():
    """The seeded generators (csrc/problems.cpp) from their own small host
    library, libmpir_problems.so -- not the product library, so the bench's
    reference arm never maps libmpir_gpu.so."""
    global _GEN
    if _GEN is not None:
        return _GEN
    import os
    here = os.path.dirname(os.path.abspath(__file__))
    path = os.path.join(here, "libmpir_problems.so")
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing; build it with __graft_entry__.build() or "
                          "`make -C paper_2311_14616_b200/csrc`")
    lib = C.CDLL(path)
    for name, args in (("mpirg_gen_greens_operator", [C.c_int, C.c_double, C.c_void_p]),
                       ("mpirg_gen_normal_matrix", [C.c_int, C.c_int, C.c_uint64, C.c_void_p]),
                       ("mpirg_gen_uniform_matrix",
                        [C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_double, C.c_void_p]),
                       ("mpirg_gen_diag_dominant", [C.c_int, C.c_uint64, C.c_double, C.c_void_p]),
                       ("mpirg_gen_matvec_compensated_f64",
                        [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p])):
        fn = getattr(lib, name)
        fn.restype = None
        fn.argtypes = args
    _GEN = lib
    return lib


def greens(n: int, alpha: float, out: np.ndarray | None = None) -> np.ndarray:
    """A = I - alpha G, column-major storage (flat, n*n), optionally into `out`
    (e.g. a numpy view of pinned host memory for the n = 65536 config)."""
    a = np.empty(n * n, dtype=np.float64) if out is None else out
    assert a.dtype == np.float64 and a.size == n * n and a.flags.c_contiguous
    _gen().mpirg_gen_greens_operator(n, alpha, a.ctypes.data)
    return a


def normal_vector(n: int, seed: int) -> np.ndarray:
    v = np.empty(n, dtype=np.float64)
    _gen().mpirg_gen_normal_matrix(n, 1, seed, v.ctypes.data)
    return v


def config(name: str, n: int | None = None, out: np.ndarray | None = None) -> dict:
    """BASELINE.json configs[i] as the reference API call they map to (`out`:
    optional host buffer for cfg5a's 34 GB matrix)."""
    n = n or FULL_N[name]
    g = _gen()
    if name == "cfg1":
        return dict(name=name, n=n, a=greens(n, 1.0), b=np.ones(n), tw=B64, tf=B32, tr=B64,
                    on_the_fly=-1, resid_term=False, ce=10.0, litmax=10)
    if name == "cfg2a":
        return dict(name=name, n=n, a=greens(n, 800.0), b=normal_vector(n, 0), tw=B64, tf=B32,
                    tr=B64, on_the_fly=-1, resid_term=False, ce=10.0, litmax=20)
    if name == "cfg2b":
        # runtime.cpp:23-28: the facade rounds A and b into TW = fp32 once
        return dict(name=name, n=n, a=greens(n, 800.0), b=normal_vector(n, 0), tw=B32, tf=B32,
                    tr=B64, on_the_fly=-1, resid_term=False, ce=10.0, litmax=20)
    if name == "cfg3":
        return dict(name=name, n=n, a=greens(n, 1.0), b=np.ones(n), tw=B32, tf=B16, tr=B32,
                    on_the_fly=-1, resid_term=False, ce=10.0, litmax=10)
    if name == "cfg4":
        a = np.empty(n * n, dtype=np.float64)
        g.mpirg_gen_normal_matrix(n, n, 1, a.ctypes.data)
        xt = np.empty(n, dtype=np.float64)
        g.mpirg_gen_uniform_matrix(n, 1, 2, -1.0, 1.0, xt.ctypes.data)
        b = np.empty(n, dtype=np.float64)
        g.mpirg_gen_matvec_compensated_f64(n, a.ctypes.data, xt.ctypes.data, b.ctypes.data)
        return dict(name=name, n=n, a=a, b=b, x_true=xt, tw=B64, tf=B32, tr=B64, on_the_fly=-1,
                    resid_term=False, ce=10.0, litmax=10)
    if name == "cfg5a":
        return dict(name=name, n=n, a=greens(n, 1.0, out), b=np.ones(n), tw=B64, tf=B32, tr=B64,
                    on_the_fly=-1, resid_term=False, ce=10.0, litmax=10)
    raise KeyError(name)


def batch_system(n: int, index: int) -> np.ndarray:
    """Config 5b system `index`: uniform(-1,1) with seed = index, a_ii += n."""
    a = np.empty(n * n, dtype=np.float64)
    _gen().mpirg_gen_diag_dominant(n, index, float(n), a.ctypes.data)
    return a


def to_working(cfg: dict, oracle_impl) -> tuple[np.ndarray, np.ndarray]:
    """(A, b) rounded into TW the way the reference facade does (runtime.cpp:23-28)."""
    n = cfg["n"]
    a = cfg["a"].reshape(n, n).T  # (n, n) view of the column-major storage
    if cfg["tw"] == B64:
        return a, cfg["b"]
    st, aw, _, _ = oracle_impl.demote(np.asfortranarray(a), B32)
    assert st == 0
    st, bw, _, _ = oracle_impl.demote(cfg["b"], B32)
    assert st == 0
    return aw, bw
