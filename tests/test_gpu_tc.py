"""K5b: the tcgen05 tensor-core trailing update for binary16 factors (lu_mode TC).

Not bit-compatible with the reference by design (one fp32-accumulated
rounding per panel step instead of two roundings per term), so:
* kernel level: the TC update against an fp64-accumulated torch reference of
  the same operation, fp16(fp32(C) - L21 U12): within 1 binary16 ulp
  everywhere and exact on >= 99% of the tile (fp32 accumulation order is the
  tensor core's); untouched regions stay bit-identical;
* solve level (config 3 shape): the refined solution within the bound
  SURVEY.md 8(d) derives from the stopping rule, 2*kappa*ce*eps32*
  (||b|| + ||A||_1 ||x||)/||x||, against the exact (reference-bitwise) path.
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
