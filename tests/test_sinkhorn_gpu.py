"""GPU parity: log-domain Sinkhorn kernels (K7/K8/K9) and run_sinkhorn vs the oracle.
Mirrors the reference's test_sinkhorn.cpp."""
import numpy as np
import pytest

import paper_2605_08793_b200 as rg

pytestmark = pytest.mark.gpu


def to_problem(p):
    return rg.ProblemInstance(p["n"], p["m"], p["M"], p["a"], p["b"], p["eta"])


@pytest.mark.parametrize("shape,eta", [((24, 17), 0.05), ((33, 300), 0.1), ((500, 37), 0.02), ((257, 513), 0.05)])
def test_optimal_alpha_beta_match_oracle(solver, oracle, shape, eta):
    n, m = shape
    p = oracle.gen_problem("rand", n, m, eta, seed=1001)
    al, be = oracle.rand_dual(n, m, 0.3, 1002)
    solver.set_problem(to_problem(p))
    a_dev = solver.optimal_alpha(rg.DualPoint(al, be))
    a_ref = oracle.optimal_alpha(p, al, be)
    np.testing.assert_allclose(a_dev, a_ref, rtol=0, atol=5e-14 * max(1.0, np.abs(a_ref).max()))
    b_dev = solver.optimal_beta(a_ref)
    b_ref = oracle.optimal_beta(p, a_ref)
    np.testing.assert_allclose(b_dev, b_ref, rtol=0, atol=5e-14 * max(1.0, np.abs(b_ref).max()))


def test_alpha_update_solves_row_block(solver, oracle):
    # test_sinkhorn.cpp:12-19
    p = oracle.gen_problem("rand", 24, 17, 0.05, seed=1001)
    al, be = oracle.rand_dual(24, 17, 0.3, 1002)
    solver.set_problem(to_problem(p))
    al2 = solver.optimal_alpha(rg.DualPoint(al, be))
    g = solver.fused_gradient(rg.DualPoint(al2, be))
    assert np.abs(g.row_sums - p["a"]).sum() <= 1e-12


def test_constant_cost_solved_in_one_step(solver):
    # test_sinkhorn.cpp:21-32
    p = rg.ProblemInstance(6, 9, np.ones((6, 9)), np.full(6, 1 / 6), np.full(9, 1 / 9), 0.5)
    solver.set_problem(p)
    x = solver.sinkhorn_step(rg.DualPoint.zeros(6, 9))
    assert solver.fused_gradient(x).marginal_error <= 1e-12


def test_step_matches_oracle_and_restores_gauge(solver, oracle):
    # test_sinkhorn.cpp:46-55
    p = oracle.gen_problem("rand", 60, 47, 0.05, seed=1301)
    al, be = oracle.rand_dual(60, 47, 0.4, 1302)
    solver.set_problem(to_problem(p))
    x = rg.DualPoint(al, be)
    ra, rb = al, be
    for _ in range(5):
        x = solver.sinkhorn_step(x)
        ra, rb = oracle.sinkhorn_step(p, ra, rb)
        assert x.beta[-1] == 0.0
        np.testing.assert_allclose(x.alpha, ra, rtol=0, atol=1e-12)
        np.testing.assert_allclose(x.beta, rb, rtol=0, atol=1e-12)


@pytest.mark.parametrize("eta", [1e-3, 1e-4])
def test_small_eta_cold_start_survives(solver, oracle, eta):
    # test_sinkhorn.cpp:57-71
    p = oracle.gen_problem("synth2", 32, 32, eta)
    solver.set_problem(to_problem(p))
    x = rg.DualPoint.zeros(32, 32)
    ra, rb = x.alpha, x.beta
    for _ in range(50):
        x = solver.sinkhorn_step(x)
        ra, rb = oracle.sinkhorn_step(p, ra, rb)
    assert np.isfinite(x.alpha).all() and np.isfinite(x.beta).all()
    err = solver.fused_gradient(x).marginal_error
    assert np.isfinite(err) and err < 2.0
    np.testing.assert_allclose(x.alpha, ra, rtol=0, atol=1e-9)


def test_run_sinkhorn_trace_matches_oracle(solver, oracle):
    # test_sinkhorn.cpp:73-86 + row-by-row agreement with the oracle
    p = oracle.gen_problem("synth2", 24, 24, 0.01)
    solver.set_problem(to_problem(p))
    cfg = rg.SinkhornConfig(max_iter=40, record_every=1)
    res = solver.run_sinkhorn(rg.DualPoint.zeros(24, 24), cfg)
    ref = oracle.run_sinkhorn(p, np.zeros(24), np.zeros(24), cfg._c())
    assert len(res.trace.rows) == 41 == len(ref["trace"])
    assert res.trace.algo == "sinkhorn" and res.trace.config_hash == rg.sinkhorn_config_hash(cfg)
    for got, want in zip(res.trace.rows, ref["trace"]):
        assert got.iter == want[0]
        assert abs(got.f - want[2]) <= 1e-12 * (1 + abs(want[2]))
        assert abs(got.marginal_error - want[3]) <= 1e-11
    for r in range(1, 41):
        prev = res.trace.rows[r - 1].f
        assert res.trace.rows[r].f <= prev + 1e-12 * (1 + abs(prev))
    np.testing.assert_allclose(res.x.alpha, ref["alpha"], atol=1e-11)


def test_tolerance_stops_early_and_record_cadence(solver, oracle):
    # test_sinkhorn.cpp:135-145
    p = oracle.gen_problem("synth2", 32, 32, 0.05)
    solver.set_problem(to_problem(p))
    cfg = rg.SinkhornConfig(max_iter=100000, tol=1e-6, record_every=100000)
    res = solver.run_sinkhorn(rg.DualPoint.zeros(32, 32), cfg)
    ref = oracle.run_sinkhorn(p, np.zeros(32), np.zeros(32), cfg._c())
    assert res.trace.rows[-1].iter < 100000 and res.trace.rows[-1].marginal_error <= 1e-6
    assert res.trace.rows[-1].iter == ref["trace"][-1][0]
    assert [r.iter for r in res.trace.rows] == [r[0] for r in ref["trace"]]


def test_config_validation(solver):
    with pytest.raises(rg.ValidationError):
        rg.SinkhornConfig(max_iter=0).validate()
    with pytest.raises(rg.ValidationError):
        rg.SinkhornConfig(tol=-1.0).validate()


def test_solver_sinkhorn_updates_match_exact_kernels_and_fall_back(solver, oracle):
    """Inside run_sinkhorn / run_splr the update takes the gradient-sweep form (alpha += eta (log a - log r)):
    same iterates as the log-sum-exp kernels to rounding; a start whose plan overflows the clamp range
    (sums outside [e^-600, e^600]) must take the exact path and still match the oracle."""
    p = oracle.gen_problem("rand", 70, 300, 0.01, seed=4242)
    solver.set_problem(to_problem(p))
    cfg = rg.SinkhornConfig(max_iter=12, tol=1e-300, record_every=1)
    for scale in (0.05, 9.0):  # 9.0 / eta = 900 > 700: clamped entries, row sums ~ e^700: fallback
        al, be = oracle.rand_dual(70, 300, scale, 99)
        res = solver.run_sinkhorn(rg.DualPoint(al, be), cfg)
        ref = oracle.run_sinkhorn(p, al, be, cfg._c())
        np.testing.assert_allclose(res.x.alpha, ref["alpha"], atol=1e-11)
        np.testing.assert_allclose(res.x.beta, ref["beta"], atol=1e-11)
        fs = [r.f for r in res.trace.rows]
        fr = [r[2] for r in ref["trace"]]
        assert len(fs) == len(fr)
        np.testing.assert_allclose(fs[1:], fr[1:], rtol=1e-10)
