"""K5b: the tcgen05 tensor-core trailing update for binary16 factors (lu_mode TC).

Not bit-compatible with the reference by design (one fp32-accumulated
rounding per panel step instead of two roundings per term), so:
* kernel level: the TC update against an fp64-accumulated torch reference of
  the same operation, fp16(fp32(C) - L21 U12): within 1 binary16 ulp
  everywhere and exact on >= 99% of the tile (fp32 accumulation order is the
  tensor core's); untouched regions stay bit-identical;
* solve level (config 3 shape): the refined solution within BASELINE's
  tolerance 10*eps32*||x||_inf of the exact (reference-bitwise) path, and within
  the (looser) bound SURVEY.md 8(d) derives from the stopping rule,
  2*kappa*ce*eps32*(||b|| + ||A||_1 ||x||)/||x||.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ulp16(x):
    x = np.abs(x.astype(np.float32))
    e = np.floor(np.log2(np.maximum(x, 2.0 ** -14)))
    return 2.0 ** (e - 10)


@pytest.mark.parametrize("n,k0,cb,ce", [(640, 64, 128, 640), (1024, 320, 384, 1000),
                                        (512, 0, 64, 512)])
def test_tc_update_kernel(gpulib, n, k0, cb, ce):
    import torch

    from paper_2311_14616_b200 import _lib as L
    g = torch.Generator().manual_seed(n + k0)
    a = (torch.randn(n, n, generator=g) * 0.5).half()  # a[col, row]: column-major storage
    dev = a.clone().cuda()
    err = L.mpirg_error()
    st = L.lib().mpirg_tc_update(n, dev.data_ptr(), k0, cb, ce, None, C.byref(err))
    L.check(st, err)
    torch.cuda.synchronize()
    got = dev.cpu()
    c0 = k0 + 64
    L21 = a[k0:k0 + 64, c0:].double()       # [k, rows]
    U12 = a[cb:ce, k0:k0 + 64].double()      # [cols, k]
    prod = (U12 @ L21)                        # [cols, rows]
    want = (a[cb:ce, c0:].float() - prod.float()).half()
    tile = got[cb:ce, c0:]
    diff = (tile.float() - want.float()).abs().numpy()
    mag = np.maximum(np.abs(want.float().numpy()), np.abs(tile.float().numpy()))
    # one binary16 ulp of the result + the fp32 accumulation error of the 64
    # products (matters only under heavy cancellation, in the fp16 subnormals)
    absum = (a[cb:ce, c0:].double().abs() + a[cb:ce, k0:k0 + 64].double().abs()
             @ a[k0:k0 + 64, c0:].double().abs()).numpy()
    assert np.all(diff <= _ulp16(mag) + 64 * 2.0 ** -24 * absum)
    assert (diff == 0).mean() >= 0.99
    untouched = got.clone()
    untouched[cb:ce, c0:] = a[cb:ce, c0:]
    assert torch.equal(untouched.view(torch.int16), a.view(torch.int16))


@pytest.mark.parametrize("n,r0,r1,cb,ce,k0,K", [
    (1024, 512, 1024, 512, 1024, 0, 512),      # 128 x 256 tiles, 8 stages of k
    (1024, 256, 700, 320, 1000, 64, 192),      # ragged rows and columns
    (2048, 1024, 2048, 1024, 1088, 0, 1024),   # 64-column tiles (narrow right half)
    (2048, 1024, 2048, 1024, 1152, 512, 512),  # 128-column tiles
    (2048, 64, 128, 128, 2048, 0, 64),         # short and wide (inside the U12 solve)
    (8192, 4096, 8192, 4096, 8192, 2048, 2048),  # 256 x 256 tiles (both accumulators)
])
def test_tc_gemm_general(gpulib, n, r0, r1, cb, ce, k0, K):
    """The persistent tcgen05 update at the shapes the recursive LU issues,
    against an fp64 product on the device: within one binary16 ulp of the
    rounded result plus the fp32 accumulation error; everything outside
    [r0:r1, cb:ce] untouched."""
    import torch

    from paper_2311_14616_b200 import _lib as L
    g = torch.Generator().manual_seed(n + K + r0)
    a = (torch.randn(n, n, generator=g) * (0.5 / max(1.0, (K / 64) ** 0.5))).half().cuda()
    dev = a.clone()  # a[col, row]: column-major storage
    err = L.mpirg_error()
    st = L.lib().mpirg_tc_gemm(n, dev.data_ptr(), r0, r1, cb, ce, k0, K, None, C.byref(err))
    L.check(st, err)
    torch.cuda.synchronize()
    Lm = a[k0:k0 + K, r0:r1].double()   # [k, rows]
    Um = a[cb:ce, k0:k0 + K].double()   # [cols, k]
    prod = Um @ Lm                      # [cols, rows]
    cold = a[cb:ce, r0:r1].double()
    want = (cold - prod).float().half()
    tile = dev[cb:ce, r0:r1]
    diff = (tile.double() - want.double()).abs().cpu().numpy()
    mag = np.maximum(want.float().abs().cpu().numpy(), tile.float().abs().cpu().numpy())
    absum = (cold.abs() + Um.abs() @ Lm.abs()).cpu().numpy()
    assert np.all(diff <= _ulp16(mag) + K * 2.0 ** -24 * absum)
    assert (diff == 0).mean() >= 0.98
    untouched = dev.clone()
    untouched[cb:ce, r0:r1] = a[cb:ce, r0:r1]
    assert torch.equal(untouched.view(torch.int16), a.view(torch.int16))


@pytest.mark.parametrize("kind,n", [("greens", 1024), ("randn", 1024), ("randn", 1984),
                                    ("randn", 1000)])
def test_tc_lu_backward_error(gpulib, kind, n):
    """The recursive tensor-core LU (binary32 panels, tcgen05 updates) as a
    factorization: ||P A - L U|| small against the binary16 unit roundoff, on a
    diagonally dominant and on pivot-heavy matrices (row moves crossing every
    level of the recursion), n not a power of two and not a multiple of 64."""
    import torch

    from helpers import greens, normal_matrix
    from paper_2311_14616_b200 import kernels
    a = greens(n, 1.0) if kind == "greens" else normal_matrix(n, 11) / np.sqrt(n)
    ah = torch.from_numpy(np.asfortranarray(a).T.copy()).half().cuda()  # [col, row]
    lu = ah.clone().reshape(-1)
    ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
    kernels.lu_factor(lu.view(torch.int16), ipiv, n, lu_mode=1)
    lu = lu.reshape(n, n).double().T  # (row, col)
    Lf = torch.tril(lu, -1) + torch.eye(n, dtype=torch.float64, device="cuda")
    Uf = torch.triu(lu)
    pa = ah.double().T.clone()
    for k, p in enumerate(ipiv.cpu().tolist()):
        if p != k:
            pa[[k, p]] = pa[[p, k]]
    resid = (pa - Lf @ Uf).abs().max().item()
    scale = (Lf.abs() @ Uf.abs()).max().item()
    assert resid <= 16 * 2.0 ** -11 * scale, (resid, scale)
    assert torch.all(Lf.abs() <= 1.0 + 2.0 ** -9)  # partial pivoting held


@pytest.mark.parametrize("n", [1024, pytest.param(8192, marks=pytest.mark.slow)])
def test_tc_mode_solution_within_stopping_rule_bound(gpulib, n):
    from helpers import greens

    from paper_2311_14616_b200 import mpir
    a = greens(n, 1.0)
    b = np.ones(n)
    kw = dict(working="single", factor="half", resid_term=False)
    exact = mpir.Factorization(a, **kw).solve(b, ce=10.0, litmax=10)
    ftc = mpir.Factorization(a, lu_mode="tc", **kw)
    tc = ftc.solve(b, ce=10.0, litmax=10)
    assert tc["reason"] == "SmallBackwardError"
    assert abs(len(tc["rhist"]) - len(exact["rhist"])) <= 1
    xe = exact["x"]
    kappa = 1.3  # kappa_inf(I - G)
    eps32 = 2.0 ** -23
    bound = 2 * kappa * 10.0 * eps32 * (1.0 + ftc.a_norm1 * np.max(np.abs(xe))) / np.max(
        np.abs(xe))
    rel = np.max(np.abs(tc["x"] - xe)) / np.max(np.abs(xe))
    assert rel <= bound, (rel, bound)
    # BASELINE.json's own tolerance for config 3, 10 eps32 ||x||_inf: met by the
    # recursive tensor-core LU at every size measured (profiles/r02*_tc_deviation:
    # 8.4e-7 at n = 1024, 2.1e-7 at n = 8192); the stopping rule admits up to
    # `bound`, so this is asserted where it was measured, not promised in general
    assert rel <= 10 * eps32, (rel, 10 * eps32)
