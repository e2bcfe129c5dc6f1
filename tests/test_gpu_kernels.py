"""Kernel-level parity: each sm_100a kernel against the C oracle, bit for bit.

Every case runs the CUDA path through the C-ABI (libmpir_gpu.so) and the
CPU restatement (oracle/mpir_oracle.c) on the same seeded inputs.
"""
import numpy as np
import pytest

from helpers import (B16, B32, B64, NP, demote_host, diag_dominant, from_dev, greens,
                     normal_matrix, normal_vector, same_bits, to_dev, uniform_matrix,
                     uniform_vector)

pytestmark = pytest.mark.gpu


def K():
    from paper_2311_14616_b200 import kernels
    return kernels


# ---------------------------------------------------------------- K1 cast --
SPECIALS = np.array([0.0, -0.0, 1.0, -1.0, 65504.0, 65519.99, 1e-8, 2.0 ** -24, 2.0 ** -25,
                     -(2.0 ** -25), 1.5 * 2.0 ** -24, 1e-30, 1e-300, np.inf, -np.inf,
                     1.0 + 2.0 ** -11 + 2.0 ** -40, float.fromhex("0x1.0000002p0"), 3.4e38, 1e-45, 1e-39])


@pytest.mark.parametrize("to", [B32, B16])
def test_demote_matches_oracle(orc, to, gpulib):
    import torch
    rng = np.random.default_rng(7)
    vals = np.concatenate([rng.standard_normal(5000) * 10.0 ** rng.integers(-8, 5, 5000),
                           SPECIALS])
    if to == B16:
        vals = vals[np.abs(vals) <= 65504.0]
    else:
        vals = vals[np.abs(vals) <= 3.4e38]
    st, want, uf_want, _ = orc.demote(vals, to)
    assert st == 0
    src = to_dev(vals)
    dst = torch.empty(vals.size, dtype=torch.float32 if to == B32 else torch.int16, device="cuda")
    uf = K().demote(src, dst)
    got = from_dev(dst)
    assert same_bits(got, want)
    assert uf == uf_want


def test_demote_f32_to_f16_matches_oracle(orc, gpulib):
    import torch
    rng = np.random.default_rng(8)
    vals = (rng.standard_normal(4099) * 10.0 ** rng.integers(-8, 4, 4099)).astype(np.float32)
    vals = vals[np.abs(vals) <= 65504.0]
    vals = np.concatenate([vals, np.array([65504.0, 65503.99, 2.0 ** -25, 1e-8], np.float32)])
    st, want, uf_want, _ = orc.demote(vals, B16)
    assert st == 0
    dst = torch.empty(vals.size, dtype=torch.int16, device="cuda")
    uf = K().demote(to_dev(vals), dst)
    assert same_bits(from_dev(dst), want) and uf == uf_want


def test_demote_overflow_reports_first_offender(gpulib):
    import torch
    from paper_2311_14616_b200._lib import OverflowDetected
    vals = np.array([1.0, 2.0, 7e4, 1e6, -8e4], dtype=np.float64)
    dst = torch.empty(vals.size, dtype=torch.int16, device="cuda")
    with pytest.raises(OverflowDetected) as ei:
        K().demote(to_dev(vals), dst)
    assert ei.value.value == 7e4
    assert "exceeds the largest finite b16 value" in str(ei.value)
    big = np.array([0.0, 1e39], dtype=np.float64)
    with pytest.raises(OverflowDetected):
        K().demote(to_dev(big), torch.empty(2, dtype=torch.float32, device="cuda"))


@pytest.mark.parametrize("prec", [B64, B32])
@pytest.mark.parametrize("rows,cols", [(1, 1), (33, 65), (257, 100), (1000, 1000)])
def test_one_norm_matches_oracle(orc, prec, rows, cols, gpulib):
    rng = np.random.default_rng(rows * 7 + cols)
    a = np.asfortranarray(rng.standard_normal((rows, cols)) * 3.0).astype(NP[prec])
    want = orc.one_norm(a, prec)
    got = K().one_norm(to_dev(a), rows, cols)
    assert got == want


# ------------------------------------------------------------------ LU -----
def lu_cases():
    return [("greens", 64, 1.0), ("greens", 200, 800.0), ("greens", 257, 799.0),
            ("randn", 50, 1), ("randn", 301, 2), ("randn", 1000, 3), ("unif", 777, 4),
            ("greens", 1500, 800.0), ("randn", 2100, 5), ("randn", 1088, 6),
            ("greens", 2048, 800.0)]


def make_case(kind, n, p):
    if kind == "greens":
        return greens(n, p)
    if kind == "randn":
        return normal_matrix(n, p)
    return uniform_matrix(n, p)


@pytest.mark.parametrize("prec", [B32, B64, B16])
@pytest.mark.parametrize("kind,n,p", lu_cases())
def test_lu_bitwise(orc, prec, kind, n, p, gpulib):
    import torch
    if prec == B16 and n > 1100:
        pytest.skip("binary16 oracle LU is slow at this size")
    a64 = make_case(kind, n, p)
    a = demote_host(a64, prec) if prec != B64 else a64
    st, want, ipiv_want, _, _ = orc.lu(a, prec)
    assert st == 0
    d = to_dev(a)
    ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
    K().lu_factor(d, ipiv, n)
    got = from_dev(d, dtype=NP[prec] if prec == B16 else None)
    np.testing.assert_array_equal(ipiv.cpu().numpy(), ipiv_want)
    assert same_bits(got, want)


def _spec_case(kind, n):
    """Matrices aimed at the whole-panel speculation of the binary32 panel kernel
    (lu_spec.cuh): clean panels, uncertifiable quotients, isolated interchanges."""
    rng = np.random.default_rng(123)
    a = rng.uniform(-1.0, 1.0, (n, n))
    if kind == "neg_diag_zeros":
        # negative pivots and exact zeros of both signs: the zero-numerator rule
        # (signed zero of the product) must match 0 / pivot
        a[rng.random((n, n)) < 0.5] = 0.0
        a[rng.random((n, n)) < 0.1] = -0.0
        a[np.arange(n), np.arange(n)] = -(n * 1.0 + rng.uniform(0, 1, n))
    elif kind == "late_interchange":
        # diagonally dominant except single entries deep in a few panels
        a[np.arange(n), np.arange(n)] = n * 1.0
        for col, row in [(37, n - 3), (64 + 63, 64 + 64), (5 * 64 + 1, 5 * 64 + 2)]:
            if row < n and col < n:
                a[row, col] = 4.0 * n
    elif kind == "tiny_entries":
        # numerators below the certified range (|a| < 2^-60): the panel must fall
        # back to the exchange algorithm's div.rn and still match
        a[np.arange(n), np.arange(n)] = n * 1.0
        a[rng.random((n, n)) < 0.05] *= 1e-30
        a[np.arange(n), np.arange(n)] = n * 1.0
    elif kind == "huge_pivots":
        a[np.arange(n), np.arange(n)] = 1e25  # divisors above 2^61
    return np.asfortranarray(a)


@pytest.mark.parametrize("n", [300, 1000, 1500])
@pytest.mark.parametrize("kind", ["neg_diag_zeros", "late_interchange", "tiny_entries", "huge_pivots"])
def test_lu_speculation_edges(orc, kind, n, gpulib):
    import torch
    a = demote_host(_spec_case(kind, n), B32)
    st, want, ipiv_want, _, _ = orc.lu(a, B32)
    assert st == 0
    d = to_dev(a)
    ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
    K().lu_factor(d, ipiv, n)
    np.testing.assert_array_equal(ipiv.cpu().numpy(), ipiv_want)
    assert same_bits(from_dev(d), want)


@pytest.mark.parametrize("nb", [32, 64])
def test_lu_bitwise_any_panel_width(orc, nb, gpulib):
    import torch
    a = demote_host(normal_matrix(700, 11), B32)
    st, want, ipiv_want, _, _ = orc.lu(a, B32)
    d = to_dev(a)
    ipiv = torch.zeros(700, dtype=torch.int32, device="cuda")
    K().lu_factor(d, ipiv, 700, nb=nb)
    assert same_bits(from_dev(d), want)
    np.testing.assert_array_equal(ipiv.cpu().numpy(), ipiv_want)


@pytest.mark.parametrize("prec,n", [(B64, 200), (B32, 200), (B16, 200), (B64, 1500),
                                    (B32, 1500)])
@pytest.mark.parametrize("where", ["diag", "below", "inf"])
def test_lu_nonfinite_entries(orc, prec, n, where, gpulib):
    """dense_lu.hpp:65-78 with non-finite data: a NaN is never chosen as a
    pivot unless it sits at position k (then p = k and the column becomes NaN);
    Inf wins the search. Bitwise (any NaN equals any NaN) against the oracle,
    single-CTA (n=200) and cluster (n=1500) panels."""
    import torch
    a64 = normal_matrix(n, 40 + n)
    k = n // 3
    if where == "diag":
        a64[k, k] = np.nan
    elif where == "below":
        a64[k + 5, k] = np.nan
    else:
        a64[k + 3, k] = np.inf
    a = demote_host(a64, prec) if prec != B64 else a64
    st, want, ipiv_want, _, _ = orc.lu(a, prec)
    assert st == 0
    d = to_dev(a)
    ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
    K().lu_factor(d, ipiv, n)
    got = from_dev(d, dtype=NP[prec] if prec == B16 else None)
    np.testing.assert_array_equal(ipiv.cpu().numpy(), ipiv_want)
    assert same_bits(got, want)


def test_lu_singular_column(gpulib):
    """test_dense_lu.cpp:45-66: column 2 all zero -> SingularPivot(column=2)."""
    import torch
    from paper_2311_14616_b200._lib import SingularPivot
    s = np.zeros((3, 3), order="F")
    s[0, 0] = 1.0
    s[1, 1] = 2.0
    d = to_dev(s)
    with pytest.raises(SingularPivot) as ei:
        K().lu_factor(d, torch.zeros(3, dtype=torch.int32, device="cuda"), 3)
    assert ei.value.column == 2


def test_lu_antidiagonal_pivots(gpulib):
    """test_dense_lu.cpp:31-43."""
    import torch
    a = np.array([[0.0, 1.0], [1.0, 0.0]], order="F")
    d = to_dev(a)
    ipiv = torch.zeros(2, dtype=torch.int32, device="cuda")
    K().lu_factor(d, ipiv, 2)
    assert ipiv.cpu().tolist() == [1, 1]


# ---------------------------------------------------------------- TRSV -----
@pytest.mark.parametrize("ts,tf", [(B64, B32), (B32, B32), (B32, B16), (B64, B64), (B64, B16)])
@pytest.mark.parametrize("n", [1, 31, 100, 1025, 2113])
def test_solve_mps_bitwise(orc, ts, tf, n, gpulib):
    import torch
    a64 = normal_matrix(n, 100 + n) if n > 1 else np.ones((1, 1), order="F")
    af = demote_host(a64, tf) if tf != B64 else a64
    st, packed, ipiv, _, _ = orc.lu(af, tf)
    x64 = uniform_vector(n, 5)
    x = x64.astype(NP[ts])
    st, want = orc.solve_mps(ts, tf, packed, ipiv, x)
    xd = to_dev(x)
    K().solve_mps(to_dev(packed), torch.from_numpy(ipiv).cuda(), xd, tf=tf)
    got = from_dev(xd)
    assert same_bits(got, want)


@pytest.mark.parametrize("ts,tf", [(B64, B32), (B32, B32), (B32, B16)])
@pytest.mark.parametrize("kind", ["zeros", "tiny", "huge"])
def test_solve_mps_uncertified_operands(orc, ts, tf, kind, gpulib):
    """Right-hand sides whose back-substitution numerators fall outside the range
    where the one-fma division can be certified (exact zeros of both signs,
    magnitudes below 2^-60 / above 2^61): those slices take div.rn and the
    result is still the reference's bit for bit."""
    import torch
    n = 777
    a64 = greens(n, 800.0)
    af = demote_host(a64, tf) if tf != B64 else a64
    st, packed, ipiv, _, _ = orc.lu(af, tf)
    rng = np.random.default_rng(9)
    x64 = rng.uniform(-1.0, 1.0, n)
    if kind == "zeros":
        x64[rng.random(n) < 0.6] = 0.0
        x64[rng.random(n) < 0.1] = -0.0
        x64[n - 130:] = 0.0  # whole trailing blocks of zeros
    elif kind == "tiny":
        x64 *= 1e-25 if ts == B32 else 1e-160
    else:
        x64 *= 1e25 if ts == B32 else 1e160
    x = x64.astype(NP[ts])
    st, want = orc.solve_mps(ts, tf, packed, ipiv, x)
    xd = to_dev(x)
    K().solve_mps(to_dev(packed), torch.from_numpy(ipiv).cuda(), xd, tf=tf)
    assert same_bits(from_dev(xd), want)


@pytest.mark.parametrize("tw,tf", [(B64, B32), (B64, B16), (B32, B16)])
@pytest.mark.parametrize("n", [2, 64, 333, 1024])
def test_solve_lps_bitwise(orc, tw, tf, n, gpulib):
    import torch
    af = demote_host(diag_dominant(n, 9 + n, 2.0 * n), tf)
    st, packed, ipiv, _, _ = orc.lu(af, tf)
    r = (uniform_vector(n, 17) * 1e-3).astype(NP[tw])
    st, want, uf_want = orc.solve_lps(tw, tf, packed, ipiv, r)
    rd = to_dev(r)
    scratch = torch.zeros(n, dtype=torch.float32 if tf == B32 else torch.int16, device="cuda")
    uf = K().solve_lps(to_dev(packed), torch.from_numpy(ipiv).cuda(), rd, scratch, tf=tf)
    assert same_bits(from_dev(rd), want)
    assert uf == uf_want


def test_lps_flushes_below_half_subnormals(gpulib):
    """test_dense_lu.cpp:207-222."""
    import torch
    eye16 = np.asfortranarray(np.array([[0x3C00, 0], [0, 0x3C00]], dtype=np.uint16))
    ipiv = torch.tensor([0, 1], dtype=torch.int32, device="cuda")
    r = to_dev(np.array([2.0 ** 20, 2.0 ** -20]))
    uf = K().solve_lps(to_dev(eye16), ipiv, r, torch.zeros(2, dtype=torch.int16, device="cuda"),
                       tf=B16)
    assert r.cpu().tolist() == [2.0 ** 20, 0.0] and uf
    eye32 = np.eye(2, dtype=np.float32, order="F")
    r = to_dev(np.array([2.0 ** 20, 2.0 ** -20]))
    uf = K().solve_lps(to_dev(eye32), ipiv, r, torch.zeros(2, dtype=torch.float32, device="cuda"))
    assert r.cpu().tolist() == [2.0 ** 20, 2.0 ** -20] and not uf


def test_mps_zero_pivot_is_nonfinite(gpulib):
    """test_dense_lu.cpp:264-274."""
    import torch
    from paper_2311_14616_b200._lib import NonFiniteResult
    lu = np.zeros((2, 2), order="F")
    lu[1, 1] = 1.0
    with pytest.raises(NonFiniteResult):
        K().solve_mps(to_dev(lu), torch.tensor([0, 1], dtype=torch.int32, device="cuda"),
                      to_dev(np.array([1.0, 1.0])))


# ------------------------------------------------------------ residual -----
@pytest.mark.parametrize("tw,tr", [(B64, B64), (B32, B64), (B32, B32)])
@pytest.mark.parametrize("n", [1, 7, 64, 257, 1000, 1024])
def test_residual_bitwise(orc, tw, tr, n, gpulib):
    import torch
    a = (normal_matrix(n, 3 + n) * 2.0).astype(NP[tw], order="F")
    x = uniform_vector(n, 4).astype(NP[tr])
    b = normal_vector(n, 6).astype(NP[tw])
    want = orc.residual(tw, tr, a, x, b)
    r = torch.zeros(n, dtype=torch.float64 if tr == B64 else torch.float32, device="cuda")
    K().residual(to_dev(a), to_dev(x), to_dev(b), r)
    assert same_bits(r.cpu().numpy(), want)


# ------------------------------------------- reciprocal-based division --
@pytest.mark.parametrize("prec", [B64, B32])
def test_fast_division_matches_div_rn(prec, gpulib):
    """The back substitution divides by u_kk through a precomputed RN(1/u_kk)
    and two residual corrections (common.cuh div_rcp); it must equal the
    IEEE division bit for bit, specials and range fallbacks included."""
    import ctypes as C
    bad = C.c_longlong(-1)
    ex = (C.c_double * 2)()
    for seed in (1, 2, 3):
        rc = gpulib.mpirg_check_fast_div(prec, seed, 1 << 26, C.byref(bad), ex)
        assert rc == 0
        assert bad.value == 0, (prec, seed, bad.value, ex[0], ex[1])


@pytest.mark.parametrize("n,alpha,col0,ncols", [(257, 800.0, 0, 257), (1000, 1.0, 0, 1000),
                                                (1024, 1.0, 512, 300), (3, 2.5, 0, 3)])
def test_device_greens_generator_bitwise(gpulib, n, alpha, col0, ncols):
    """mpirg_gen_greens_operator_device against the host generator (itself
    pinned to the reference's build_operator, tests/test_abi.py): every bit of
    every entry, a column window included."""
    import torch
    from helpers import greens
    want = greens(n, alpha)  # (n, n) Fortran order
    out = torch.zeros(ncols * n, dtype=torch.float64, device="cuda")
    st = gpulib.mpirg_gen_greens_operator_device(n, alpha, col0, ncols, out.data_ptr(), n, None)
    torch.cuda.synchronize()
    assert st == 0
    got = out.cpu().numpy().reshape(ncols, n).T
    assert np.array_equal(got.view(np.uint64), np.ascontiguousarray(
        want[:, col0:col0 + ncols]).view(np.uint64))
