"""GMRES-IR and BiCGSTAB-IR on the device (krylov_ir.hpp:62-254, 297-318)
against the compiled reference's krylov_ir_solve_report on the same inputs:
solution bits, residual / correction histories, inner iteration counts and the
stopping reason must all be equal.

The configurations are the reference's own use of Krylov corrections: factors
too coarse for plain refinement (binary16 factors of the ill-conditioned
I - 800 G, acceptance check 4/7) and the ordinary ones, where GMRES converges
in one or two inner iterations.
"""
import numpy as np
import pytest

from helpers import greens, normal_matrix, normal_vector

pytestmark = pytest.mark.gpu

NAMES = {0: "double", 1: "single", 2: "half"}


def _problem(kind, n):
    if kind == "greens800":
        return greens(n, 800.0), normal_vector(n, 0)
    if kind == "greens1":
        return greens(n, 1.0), np.ones(n)
    a = normal_matrix(n, 21) + np.sqrt(n) * np.eye(n)
    return a, normal_vector(n, 5)


@pytest.mark.parametrize("tw,tf,tr,kind,n,bs", [
    (0, 2, 0, "greens800", 256, 10),
    (0, 2, 0, "greens800", 1000, 10),
    (1, 2, 1, "greens800", 512, 10),
    (0, 1, 0, "greens800", 640, 6),
    (1, 2, 0, "greens1", 384, 4),
    (0, 2, 0, "randn", 512, 3),     # budget exhausted before the tolerance
    (0, 0, 0, "randn", 300, 5),
])
@pytest.mark.parametrize("solver", ["gmres", "bicgstab"])
def test_krylov_ir_bitwise_vs_compiled_reference(gpulib, ref, solver, tw, tf, tr, kind, n, bs):
    from paper_2311_14616_b200 import mpir
    if not hasattr(ref, "_krylov_ir"):
        pytest.skip("compiled reference built without the Krylov driver")
    a, b = _problem(kind, n)
    if tw == 1:  # the facade rounds the inputs once into TW (runtime.cpp:23-28)
        a = a.astype(np.float32).astype(np.float64)
        b = b.astype(np.float32).astype(np.float64)
    want = ref.krylov_ir(tw, tf, tr, a.astype(np.float32) if tw == 1 else a,
                         b.astype(np.float32) if tw == 1 else b, kind=solver, basissize=bs,
                         resid_term=False, ce=10.0, litmax=12)
    assert want["status"] == "ok"
    f = mpir.Factorization(a, working=NAMES[tw], factor=NAMES[tf], residual=NAMES[tr],
                           resid_term=False, krylov=solver, basissize=bs)
    got = f.solve(b, ce=10.0, litmax=12)
    assert got["khist"] == [int(k) for k in want["khist"]]
    assert got["reason"] == want["reason"]
    assert [v.hex() for v in got["rhist"]] == [float(v).hex() for v in want["rhist"]]
    assert [v.hex() for v in got["dhist"]] == [float(v).hex() for v in want["dhist"]]
    assert got["breakdown"] == want["breakdown"]
    xw = want["x"].astype(np.float64)
    assert np.array_equal(got["x"].view(np.uint64), xw.view(np.uint64))


def test_gmres_ir_rescues_half_precision_factors(gpulib):
    """Acceptance check 4's point: binary16 factors of I - 800 G do not refine to
    working precision with plain corrections, GMRES corrections do."""
    from paper_2311_14616_b200 import mpir
    n = 512
    a, b = _problem("greens800", n)
    kw = dict(working="double", factor="half", resid_term=False)
    plain = mpir.Factorization(a, **kw).solve(b, ce=10.0, litmax=20)
    gm = mpir.Factorization(a, krylov="gmres", basissize=10, **kw).solve(b, ce=10.0, litmax=20)
    x = np.linalg.solve(a, b)
    err_plain = np.max(np.abs(plain["x"] - x)) / np.max(np.abs(x))
    err_gm = np.max(np.abs(gm["x"] - x)) / np.max(np.abs(x))
    assert gm["reason"] == "SmallBackwardError" and err_gm < 1e-10
    assert err_gm < err_plain
    assert all(1 <= k <= 10 for k in gm["khist"]) and len(gm["khist"]) == len(gm["dhist"])


def test_krylov_argument_validation(gpulib):
    from paper_2311_14616_b200 import mpir
    a = greens(64, 1.0)
    with pytest.raises(mpir.InvalidParameter):
        mpir.Factorization(a, krylov="gmres", basissize=0)
    with pytest.raises(mpir.InvalidParameter):
        mpir.Factorization(a, krylov="bicgstab", basissize=0)
    with pytest.raises(mpir.InvalidParameter):
        mpir.Factorization(a, krylov="cg")
