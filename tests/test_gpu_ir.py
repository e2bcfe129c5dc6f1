"""End-to-end parity of the GPU refinement against the C oracle.

MPFactorization<TW,TF,TR> + ir_solve_report on the GPU (through the Python
mirror of the reference module and the C-ABI) versus the CPU restatement of
the same reference code on identical inputs: the solution, both histories,
the stop reason, the pivots and ||A||_1 must agree bit for bit.
"""
import numpy as np
import pytest

from helpers import (B16, B32, B64, NP, demote_host, diag_dominant, greens, normal_matrix,
                     normal_vector, same_bits)

pytestmark = pytest.mark.gpu

NAME = {B64: "double", B32: "single", B16: "half"}
COMBOS = [(B64, B64, B64), (B64, B32, B64), (B64, B16, B64), (B32, B32, B32),
          (B32, B16, B32), (B32, B32, B64), (B32, B16, B64)]


def mirror():
    from paper_2311_14616_b200 import mpir
    return mpir


def run_both(orc, a64, b64, tw, tf, tr, otf=None, resid_term=True, **tp):
    m = mirror()
    f = m.Factorization(a64, working=NAME[tw], factor=NAME[tf], residual=NAME[tr],
                        on_the_fly=otf, resid_term=resid_term)
    got = f.solve(b64, **tp)
    aw = a64 if tw == B64 else demote_host(a64, B32)
    bw = b64 if tw == B64 else demote_host(b64, B32)
    want = orc.ir(tw, tf, tr, aw, bw, on_the_fly=-1 if otf is None else int(otf),
                  resid_term=resid_term, cr=tp.get("cr", 1.0), ce=tp.get("ce", 1.0),
                  rmax=tp.get("rmax", 0.5), litmax=tp.get("litmax", 10))
    return f, got, want


def assert_same_report(got, want, tw):
    assert want["status"] == "ok"
    assert got["reason"] == want["reason"]
    np.testing.assert_array_equal(np.array(got["rhist"]), want["rhist"])
    np.testing.assert_array_equal(np.array(got["dhist"]), want["dhist"])
    x = got["x"].astype(NP[tw])
    assert same_bits(x, want["x"], nan_equal=False)


@pytest.mark.parametrize("tw,tf,tr", COMBOS)
@pytest.mark.parametrize("n,alpha", [(97, 1.0), (300, 800.0)])
def test_ir_all_combos_bitwise(orc, tw, tf, tr, n, alpha, gpulib):
    a = greens(n, alpha)
    b = normal_vector(n, 0)
    f, got, want = run_both(orc, a, b, tw, tf, tr, litmax=20)
    assert_same_report(got, want, tw)
    assert f.a_norm1 == want["a_norm1"]
    np.testing.assert_array_equal(f.ipiv(), want["ipiv"])


@pytest.mark.parametrize("otf", [False, True])
@pytest.mark.parametrize("resid_term", [False, True])
def test_ir_modes_bitwise(orc, otf, resid_term, gpulib):
    a = normal_matrix(400, 1)
    b = normal_vector(400, 2)
    _, got, want = run_both(orc, a, b, B64, B32, B64, otf=otf, resid_term=resid_term, ce=10.0,
                            litmax=10)
    assert_same_report(got, want, B64)


def test_ir_config1_small(orc, gpulib):
    """BASELINE config 1 shape (I - G, ones, ce=10, backward-error test) at n=1024."""
    a = greens(1024, 1.0)
    b = np.ones(1024)
    _, got, want = run_both(orc, a, b, B64, B32, B64, resid_term=False, ce=10.0, litmax=10)
    assert_same_report(got, want, B64)
    assert got["reason"] == "SmallBackwardError"


def test_ir_config2b_small(orc, gpulib):
    """BASELINE config 2b shape (fp32/fp32/fp64 promoted residual) at n=768."""
    a = greens(768, 800.0)
    b = normal_vector(768, 0)
    _, got, want = run_both(orc, a, b, B32, B32, B64, resid_term=False, ce=10.0, litmax=20)
    assert_same_report(got, want, B32)


def test_ir_pivot_heavy(orc, gpulib):
    """BASELINE config 4 shape (randn A, b = A x_true compensated) at n=1500."""
    from helpers import gen_lib, uniform_vector
    n = 1500
    a = normal_matrix(n, 1)
    xt = uniform_vector(n, 2)
    b = np.empty(n)
    gen_lib().mpirg_gen_matvec_compensated_f64(n, np.ascontiguousarray(a.T).ctypes.data,
                                               xt.ctypes.data, b.ctypes.data)
    _, got, want = run_both(orc, a, b, B64, B32, B64, resid_term=False, ce=10.0, litmax=10)
    assert_same_report(got, want, B64)
    assert np.max(np.abs(got["x"] - xt)) / np.max(np.abs(xt)) < 1e-10


def test_identity_converges_in_one_step(gpulib):
    """test_ir_engine.cpp:111-128."""
    m = mirror()
    f = m.Factorization(np.eye(5), working="double", factor="single", on_the_fly=True)
    b = np.array([1.0, -2.0, 3.0, -4.0, 5.0])
    rep = f.solve(b)
    assert rep["reason"] == "SmallResidual"
    assert rep["x"].tolist() == b.tolist()
    assert rep["rhist"] == [5.0, 0.0] and rep["dhist"] == [5.0]


def test_zero_rhs(gpulib):
    """test_ir_engine.cpp:130-137."""
    m = mirror()
    f = m.Factorization(np.eye(4), factor="single")
    rep = f.solve(np.zeros(4))
    assert rep["reason"] == "SmallResidual"
    assert rep["x"].tolist() == [0.0] * 4 and rep["rhist"] == [0.0, 0.0]


def test_nonfinite_carries_partial_history(gpulib):
    """test_ir_engine.cpp:244-262."""
    m = mirror()
    f = m.Factorization(np.array([[1e-38]]), factor="single")
    with pytest.raises(m.NonFiniteResult) as ei:
        f.solve(np.array([1e308]))
    assert ei.value.rhist == [1e308] and ei.value.dhist == []
    with pytest.raises(m.DimensionMismatch):
        f.solve(np.array([1.0, 2.0]))


def test_iteration_limit_and_refactor_reuse(orc, gpulib):
    """test_ir_engine.cpp:187-197 and test_mp_structures.cpp:141-196."""
    m = mirror()
    p = m.greens_problem(128, 799.0)
    f = m.Factorization(p["a"], working="double", factor="half")
    rep = f.solve(p["b"], rmax=1.0, litmax=4)
    assert rep["reason"] == "IterationLimit"
    assert len(rep["rhist"]) == 4 and len(rep["dhist"]) == 3
    f2 = m.Factorization(p["a"], factor="single")
    packed0 = f2.packed_lu().copy()
    x1 = f2.solve(p["b"])["x"]
    f2.refactor(2.0 * np.asarray(p["a"]))
    f2.refactor(p["a"])
    assert np.array_equal(f2.packed_lu(), packed0)
    assert np.array_equal(f2.solve(p["b"])["x"], x1)


def test_overflow_and_underflow_flags(gpulib):
    """test_mp_structures.cpp:198-213."""
    m = mirror()
    a = np.eye(4)
    a[2, 1] = 1e-30
    assert m.Factorization(a, factor="half").demotion_underflowed
    assert not m.Factorization(np.eye(4), factor="half").demotion_underflowed
    big = np.eye(4)
    big[1, 2] = 7e4
    with pytest.raises(m.OverflowDetected):
        m.Factorization(big, factor="half")
    m.Factorization(big, factor="single")
    with pytest.raises(m.DimensionMismatch):
        m.Factorization(np.zeros((3, 4)))


def test_singular_matrix(gpulib):
    m = mirror()
    s = np.zeros((3, 3))
    s[0, 0] = 1.0
    s[1, 1] = 2.0
    with pytest.raises(m.SingularPivot) as ei:
        m.Factorization(s, factor="single")
    assert ei.value.column == 2


def test_solve_many_equals_single_solves(gpulib):
    """Several right-hand sides on one handle: each report is the single solve's, bit for bit."""
    from paper_2311_14616_b200 import mpir
    n = 300
    a = greens(n, 800.0)
    rng = np.random.default_rng(4)
    bs = rng.standard_normal((n, 3))
    f = mpir.Factorization(a, working="double", factor="single", resid_term=False)
    many = f.solve_many(bs, ce=10.0, litmax=20)
    assert len(many) == 3
    for j, rep in enumerate(many):
        one = mpir.Factorization(a, working="double", factor="single", resid_term=False).solve(
            bs[:, j].copy(), ce=10.0, litmax=20)
        assert rep["reason"] == one["reason"] and rep["rhist"] == one["rhist"]
        assert np.array_equal(rep["x"].view(np.uint64), one["x"].view(np.uint64))
