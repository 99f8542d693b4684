"""GPU parity: fused gradient (K1) through the C ABI vs the CPU oracle.

Mirrors the reference's test_dual.cpp cases; tolerances are the reference's own
(1e-12 relative on sums and f, test_dual.cpp:87-119).
"""
import numpy as np
import pytest

import paper_2605_08793_b200 as rg

pytestmark = pytest.mark.gpu

RTOL = 1e-12


def to_problem(p):
    return rg.ProblemInstance(p["n"], p["m"], p["M"], p["a"], p["b"], p["eta"])


def check_against_oracle(solver, oracle, p, al, be, rtol=RTOL):
    solver.set_problem(to_problem(p))
    got = solver.fused_gradient(rg.DualPoint(al, be))
    ref = oracle.gradient(p, al, be)
    np.testing.assert_allclose(got.row_sums, ref["row"], rtol=rtol, atol=0)
    np.testing.assert_allclose(got.col_sums, ref["col"], rtol=rtol, atol=0)
    scale = max(1.0, abs(ref["f"]))
    assert abs(got.f - ref["f"]) <= rtol * scale * 10
    np.testing.assert_allclose(got.grad, ref["grad"], rtol=0, atol=rtol * max(ref["row"].max(), ref["col"].max()) * 4)
    assert abs(got.marginal_error - ref["marginal_error"]) <= 1e-11 * max(1.0, ref["marginal_error"])
    assert abs(got.duality_gap - ref["duality_gap"]) <= 1e-11 * max(1.0, abs(ref["duality_gap"]))
    assert abs(got.grad_norm2 - ref["grad_norm2"]) <= 1e-11 * max(1.0, ref["grad_norm2"])
    return got, ref


def test_two_by_two_hand_case(solver):
    # test_dual.cpp:72-85: zero cost, eta = 1, origin -> sums 2, grad 1.5, f 4 exactly
    p = rg.ProblemInstance(2, 2, np.zeros((2, 2)), np.full(2, 0.5), np.full(2, 0.5), 1.0)
    solver.set_problem(p)
    g = solver.fused_gradient(rg.DualPoint.zeros(2, 2))
    assert list(g.row_sums) == [2.0, 2.0] and list(g.col_sums) == [2.0, 2.0]
    assert list(g.grad) == [1.5, 1.5, 1.5] and g.f == 4.0


def test_clamp_matches_reference(solver):
    # test_dual.cpp:44-53: exponent 1e4 clamps to exp(+-700)
    p = rg.ProblemInstance(1, 2, np.zeros((1, 2)), np.ones(1), np.full(2, 0.5), 1e-4)
    solver.set_problem(p)
    T = solver.plan(rg.DualPoint(np.array([1.0]), np.zeros(2)))
    assert abs(T[0, 0] / np.exp(700.0) - 1.0) < 4e-16
    T = solver.plan(rg.DualPoint(np.array([-1.0]), np.zeros(2)))
    assert abs(T[0, 0] / np.exp(-700.0) - 1.0) < 4e-16


@pytest.mark.parametrize("shape", [(5, 7), (17, 33), (64, 64), (33, 128), (257, 19), (1, 1), (2, 513), (300, 257)])
def test_fused_gradient_matches_oracle(solver, oracle, shape):
    n, m = shape
    if m < 2 or n < 1:
        p = dict(n=n, m=m, M=np.zeros((n, m), order="F"), a=np.full(n, 1.0 / n), b=np.full(m, 1.0 / m), eta=1.0)
        al, be = np.full(n, 0.3), np.zeros(m)
    else:
        p = oracle.gen_problem("rand", n, m, 0.1, seed=300 + n)
        al, be = oracle.rand_dual(n, m, 0.2, 400 + m)
    check_against_oracle(solver, oracle, p, al, be)


def test_plan_matches_oracle_to_an_ulp(solver, oracle):
    p = oracle.gen_problem("rand", 40, 37, 0.05, seed=11)
    al, be = oracle.rand_dual(40, 37, 0.5, 12)
    solver.set_problem(to_problem(p))
    T = solver.plan(rg.DualPoint(al, be))
    Tref = oracle.plan(p, al, be)
    # the device multiplies by 1/eta where the reference divides (dual.h:64): the exponent t differs by
    # <= 1 ulp relative, so T differs by <= (|t| + 2) ulp (1 ulp for the exp itself)
    t = np.log(Tref)
    assert np.all(np.abs(T / Tref - 1.0) <= (np.abs(t) + 2.0) * 2.3e-16)


def test_row_major_and_column_major_uploads_agree(solver, oracle):
    p = oracle.gen_problem("rand", 70, 45, 0.1, seed=5)
    al, be = oracle.rand_dual(70, 45, 0.2, 6)
    solver.set_problem(rg.ProblemInstance(70, 45, np.asfortranarray(p["M"]), p["a"], p["b"], p["eta"]))
    g1 = solver.fused_gradient(rg.DualPoint(al, be))
    solver.set_problem(rg.ProblemInstance(70, 45, np.ascontiguousarray(p["M"]), p["a"], p["b"], p["eta"]))
    g2 = solver.fused_gradient(rg.DualPoint(al, be))
    assert g1.f == g2.f and np.array_equal(g1.grad, g2.grad)


def test_gauge_violation_is_a_validation_error(solver, oracle):
    p = oracle.gen_problem("rand", 6, 5, 0.1, seed=1)
    solver.set_problem(to_problem(p))
    x = rg.DualPoint(np.zeros(6), np.zeros(5))
    x.beta[4] = 1e-3
    with pytest.raises(rg.ValidationError, match="gauge violated"):
        solver.fused_gradient(x)
    with pytest.raises(rg.ValidationError, match="dimension mismatch"):
        solver.fused_gradient(rg.DualPoint(np.zeros(5), np.zeros(5)))


def test_small_eta_cold_start_is_finite(solver, oracle):
    # exponents down to -1000 and up: clamp + table exp stay finite and match
    p = oracle.gen_problem("synth2", 96, 80, 0.001)
    al, be = np.zeros(96), np.zeros(80)
    got, ref = check_against_oracle(solver, oracle, p, al, be, rtol=1e-11)
    assert np.isfinite(got.f)


def test_synth1_at_a_thousand(solver, oracle):
    # BASELINE config A: n = m = 1000 Gaussian clouds in R^2, eta = 0.01 (acceptance seed 7)
    p = oracle.gen_problem("synth1-iid", 1000, 1000, 0.01, d=2, seed=7)
    al, be = oracle.rand_dual(1000, 1000, 0.02, 77)
    check_against_oracle(solver, oracle, p, al, be, rtol=1e-11)


def test_deterministic(solver, oracle):
    p = oracle.gen_problem("rand", 500, 700, 0.05, seed=3)
    al, be = oracle.rand_dual(500, 700, 0.3, 4)
    solver.set_problem(to_problem(p))
    a = solver.fused_gradient(rg.DualPoint(al, be))
    b = solver.fused_gradient(rg.DualPoint(al, be))
    assert a.f == b.f and np.array_equal(a.grad, b.grad)
