"""Refactor from host memory with the copy overlapped with the LU.

mpirg_factorization_refactor(h, host_a, 0) streams the columns of A in chunks
and starts the binary32 LU before the last chunk has landed (late chunks catch
up from panel snapshots, lu.cu launch_lu_late). The result must be the one of
the copy-then-refactor path bit for bit: packed factors, pivots, ||A||_1, the
first-overflow report and the refined solution.
"""
import ctypes as C

import numpy as np
import pytest

from helpers import B32, demote_host, greens, normal_matrix, normal_vector, same_bits

pytestmark = pytest.mark.gpu


def mirror():
    from paper_2311_14616_b200 import mpir
    return mpir


def lib():
    import paper_2311_14616_b200 as p
    return p.lib()


def refactor_host(f, a, pinned, dtype=np.float64):
    """Refactor handle f from a host column-major array of the working
    precision (optionally pinned)."""
    import torch
    from paper_2311_14616_b200 import _lib as L
    buf = np.asfortranarray(a).astype(dtype).ravel(order="F")
    t = torch.from_numpy(buf)
    if pinned:
        t = t.pin_memory()
    err = L.mpirg_error()
    st = lib().mpirg_factorization_refactor(f._h, C.c_void_p(t.data_ptr()), 0, C.byref(err))
    L.check(st, err)


def state(f):
    return f.packed_lu().copy(), f.ipiv().copy(), f.a_norm1


@pytest.mark.parametrize("kind,n,p", [("greens", 1024, 800.0), ("randn", 1024, 3),
                                      ("greens", 2048, 800.0), ("randn", 2048, 7),
                                      ("greens", 4096, 800.0), ("randn", 3072, 1)])
@pytest.mark.parametrize("working", ["double", "single"])
def test_streamed_refactor_matches_device_refactor(kind, n, p, working, gpulib):
    m = mirror()
    a = greens(n, p) if kind == "greens" else normal_matrix(n, int(p))
    if working == "single":
        a = a.astype(np.float32).astype(np.float64)
    b = normal_vector(n, 0)
    f = m.Factorization(a, working=working, factor="single", resid_term=False)
    want = state(f)
    xw = f.solve(b, ce=10.0, litmax=20)
    f.refactor(2.0 * a)  # something else in between
    for pinned in (True, False):
        refactor_host(f, a, pinned, np.float64 if working == "double" else np.float32)
        got = state(f)
        assert same_bits(got[0], want[0])
        np.testing.assert_array_equal(got[1], want[1])
        assert got[2] == want[2]
        xg = f.solve(b, ce=10.0, litmax=20)
        assert xg["reason"] == xw["reason"] and xg["rhist"] == xw["rhist"]
        assert np.array_equal(xg["x"].view(np.uint64), xw["x"].view(np.uint64))


def test_streamed_refactor_matches_oracle(orc, gpulib):
    m = mirror()
    n = 1088 + 64  # not a multiple of the chunk width
    a = normal_matrix(n, 5)
    f = m.Factorization(np.eye(n), working="double", factor="single")
    refactor_host(f, a, True)
    st, want, ipiv_want, _, _ = orc.lu(demote_host(a, B32), B32)
    assert st == 0
    np.testing.assert_array_equal(f.ipiv(), ipiv_want)
    assert same_bits(f.packed_lu(), want)


def test_streamed_refactor_reports_first_overflow(gpulib):
    m = mirror()
    n = 2048
    a = greens(n, 1.0)
    a[7, 1500] = 1e39   # late chunk
    a[3, 1800] = -2e39  # later in storage order
    f = m.Factorization(greens(n, 1.0), working="double", factor="single")
    with pytest.raises(m.OverflowDetected) as e_host:
        refactor_host(f, a, True)
    with pytest.raises(m.OverflowDetected) as e_dev:
        f.refactor(a)
    assert str(e_host.value) == str(e_dev.value)
    assert str(e_host.value).startswith("value 9999999999999999")  # 1e39, not -2e39


def test_streamed_refactor_graph_replay_reads_current_host_data(gpulib):
    """From the same pinned host pointer the streamed refactor runs directly,
    then is captured into a CUDA graph, then replayed: every call must read the
    buffer's current contents and give the device path's bits."""
    import torch
    from paper_2311_14616_b200 import _lib as L
    m = mirror()
    n = 1536
    mats = [greens(n, 800.0), normal_matrix(n, 11), 0.5 * greens(n, 800.0), normal_matrix(n, 12)]
    f = m.Factorization(mats[0], working="double", factor="single", resid_term=False)
    buf = torch.empty(n * n, dtype=torch.float64).pin_memory()
    err = L.mpirg_error()
    for rep in range(2):
        for a in mats:
            f.refactor(a)
            want = state(f)
            buf.numpy()[:] = np.asfortranarray(a).ravel(order="F")
            st = lib().mpirg_factorization_refactor(f._h, C.c_void_p(buf.data_ptr()), 0,
                                                    C.byref(err))
            L.check(st, err)
            got = state(f)
            assert same_bits(got[0], want[0])
            np.testing.assert_array_equal(got[1], want[1])
            assert got[2] == want[2]


def test_streamed_graph_survives_scal_reallocation(gpulib):
    """A solve with litmax above anything seen so far reallocates the handle's
    scalar slots; the captured streamed-refactor graph had the old ||A||_1 slot
    baked in, so it must be dropped (the replay used to write freed memory and
    a_norm1 came back 0, changing the stopping test)."""
    import torch
    from paper_2311_14616_b200 import _lib as L
    m = mirror()
    n = 1024
    a = greens(n, 800.0)
    b = normal_vector(n, 0)
    f = m.Factorization(a, working="double", factor="single", resid_term=False)
    want_norm = f.a_norm1
    want = f.solve(b, ce=10.0, litmax=40)
    buf = torch.empty(n * n, dtype=torch.float64).pin_memory()
    buf.numpy()[:] = np.asfortranarray(a).ravel(order="F")
    err = L.mpirg_error()

    def refactor():
        st = lib().mpirg_factorization_refactor(f._h, C.c_void_p(buf.data_ptr()), 0, C.byref(err))
        L.check(st, err)

    f2 = m.Factorization(a, working="double", factor="single", resid_term=False)
    f = f2  # a fresh handle whose scalar slots still have the default capacity
    refactor()
    refactor()  # captured
    refactor()  # replayed
    got = f.solve(b, ce=10.0, litmax=40)  # litmax > 16: slots reallocated
    refactor()
    assert f.a_norm1 == want_norm
    again = f.solve(b, ce=10.0, litmax=40)
    for g in (got, again):
        assert g["reason"] == want["reason"] and g["rhist"] == want["rhist"]
        assert np.array_equal(g["x"].view(np.uint64), want["x"].view(np.uint64))
