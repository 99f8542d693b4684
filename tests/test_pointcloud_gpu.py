"""GPU parity: point-cloud problems (regot_b200_set_pointcloud).

The cost |x_i - y_j|^2 / max is formed on the device, either materialised in HBM or recomputed on the
fly by the sweep kernels' producer warps (BASELINE config E).  Bars: the device cost equals the host
generator's matrix (problems.problem_from_points, the draw-for-draw mirror of problem.h:103-138) BIT
FOR BIT; every result of the on-the-fly mode equals the materialised mode bit for bit; both agree
with the CPU oracle within the tolerances of the resident-matrix tests.
"""
import numpy as np
import pytest

import paper_2605_08793_b200 as rg
from paper_2605_08793_b200 import problems

pytestmark = pytest.mark.gpu


def clouds(kind, n, m, d, seed):
    if kind == "gmm":
        return problems.gen_gmm_points(n, m, d, seed)
    if kind == "uniform":
        return problems.gen_uniform_points(n, m, d, seed)
    rng = problems.Rng(seed)  # gen_synthetic1 "iid" clouds (problem.h:112-122)
    X = np.array([rng.normal() for _ in range(n * d)]).reshape(n, d)
    Y = np.array([rng.normal() for _ in range(m * d)]).reshape(m, d)
    return X, Y


def marginals(n, m):
    return np.full(n, 1.0 / n), np.full(m, 1.0 / m)


@pytest.mark.parametrize("kind,n,m,d", [("normal", 50, 70, 2), ("uniform", 257, 300, 3), ("gmm", 128, 129, 10),
                                        ("normal", 17, 1030, 1), ("uniform", 600, 33, 7)])
def test_device_cost_equals_host_generator_bitwise(solver, kind, n, m, d):
    X, Y = clouds(kind, n, m, d, 5)
    a, b = marginals(n, m)
    want = problems.problem_from_points(X, Y, 0.01).M
    assert want.max() == 1.0
    for fly in (False, True):
        solver.set_pointcloud(X, Y, a, b, 0.01, on_the_fly=fly)
        solver.validate_problem()
        got = solver.get_cost()
        assert np.array_equal(got, want), (fly, np.abs(got - want).max())


def test_synthetic1_problem_is_reproduced(solver):
    # the reference generator (problem.h:103-138, seed 7 = acceptance seed): same matrix from its clouds
    p = problems.gen_synthetic1(96, 80, "iid", 2, 7, 0.01)
    X, Y = clouds("normal", 96, 80, 2, 7)
    solver.set_pointcloud(X, Y, p.a, p.b, p.eta, on_the_fly=True)
    assert np.array_equal(solver.get_cost(), p.M)


@pytest.mark.parametrize("kind,n,m,d,eta", [("uniform", 300, 700, 3, 0.01), ("normal", 1000, 513, 2, 0.01),
                                            ("gmm", 333, 257, 10, 0.02)])
def test_on_the_fly_equals_materialised_bitwise(solver, kind, n, m, d, eta):
    X, Y = clouds(kind, n, m, d, 9)
    a, b = marginals(n, m)
    rng = np.random.default_rng(n + m)
    al = 0.05 * rng.normal(size=n)
    be = 0.05 * rng.normal(size=m)
    be[-1] = 0.0
    x = rg.DualPoint(al, be)
    out = {}
    for fly in (False, True):
        solver.set_pointcloud(X, Y, a, b, eta, on_the_fly=fly)
        g = solver.fused_gradient(x)
        sk = solver.sinkhorn_step(x)
        T = solver.plan(x)
        A = solver.assemble_topk(x, rg.topk_budget(rg.ProblemInstance(n, m, None, a, b, eta), 0.05), 0.5, g)
        colptr, rowidx, values, coords = A.export()
        res = solver.run_splr(rg.DualPoint.zeros(n, m), rg.SplrConfig(max_iter=25, tol=1e-9))
        out[fly] = (g.f, g.row_sums, g.col_sums, g.grad, sk.alpha, sk.beta, T, colptr, rowidx, values, coords,
                    res.x.alpha, res.x.beta, np.array([r.f for r in res.trace.rows]))
    for u, v in zip(out[False], out[True]):
        assert np.array_equal(np.asarray(u), np.asarray(v))


def test_on_the_fly_matches_oracle(solver, oracle):
    n, m, d, eta = 257, 300, 3, 0.01
    X, Y = clouds("uniform", n, m, d, 31)
    p = problems.problem_from_points(X, Y, eta)
    op = dict(n=n, m=m, M=np.asfortranarray(p.M), a=p.a, b=p.b, eta=eta)
    al, be = oracle.rand_dual(n, m, 0.05, 3)
    solver.set_pointcloud(X, Y, p.a, p.b, eta, on_the_fly=True)
    g = solver.fused_gradient(rg.DualPoint(al, be))
    ref = oracle.gradient(op, al, be)
    np.testing.assert_allclose(g.row_sums, ref["row"], rtol=1e-12)
    np.testing.assert_allclose(g.col_sums, ref["col"], rtol=1e-12)
    assert abs(g.f - ref["f"]) <= 1e-11 * max(1.0, abs(ref["f"]))
    sk = solver.sinkhorn_step(rg.DualPoint(al, be))
    ra, rb = oracle.sinkhorn_step(op, al, be)
    np.testing.assert_allclose(sk.alpha, ra, atol=1e-12)
    np.testing.assert_allclose(sk.beta, rb, atol=1e-12)
    # pattern bit-exact given identical T (the oracle selects on the device plan)
    T = solver.plan(rg.DualPoint(al, be))
    k = rg.topk_budget(p, 0.03)
    A = solver.assemble_topk(rg.DualPoint(al, be), k, 0.25, g)
    assert np.array_equal(A.export()[3], oracle.select_topk(T, k))


def test_config_e_shape_solves_to_tolerance(solver):
    # BASELINE config E at reduced size: uniform clouds in R^3, eta = 0.01, cost never materialised
    n = m = 2000
    X, Y = clouds("uniform", n, m, 3, 31)
    a, b = marginals(n, m)
    solver.set_pointcloud(X, Y, a, b, 0.01, on_the_fly=True)
    res = solver.run_splr(rg.DualPoint.zeros(n, m), rg.SplrConfig(tol=1e-8, max_iter=300))
    last = res.trace.rows[-1]
    assert last.marginal_error <= 1e-8
    g = solver.fused_gradient(res.x)
    assert g.marginal_error <= 1e-8


def test_degenerate_cloud_is_rejected(solver):
    X = np.ones((4, 2))
    Y = np.ones((5, 2))
    a, b = marginals(4, 5)
    with pytest.raises(rg.DegenerateCostError):
        solver.set_pointcloud(X, Y, a, b, 0.01)
    with pytest.raises(rg.ValidationError):
        solver.set_pointcloud(np.array([[np.nan, 0.0]] * 4), Y, a, b, 0.01)


def test_high_dimension_clouds(solver):
    # on the fly the panel of target points lives in shared memory: d <= 64; above that only the materialised mode
    n, m, eta = 130, 270, 0.05
    for d in (33, 64):
        X, Y = clouds("normal", n, m, d, d)
        a, b = marginals(n, m)
        want = problems.problem_from_points(X, Y, eta).M
        solver.set_pointcloud(X, Y, a, b, eta, on_the_fly=True)
        assert np.array_equal(solver.get_cost(), want)
        g1 = solver.fused_gradient(rg.DualPoint.zeros(n, m))
        solver.set_pointcloud(X, Y, a, b, eta, on_the_fly=False)
        g0 = solver.fused_gradient(rg.DualPoint.zeros(n, m))
        assert g0.f == g1.f and np.array_equal(g0.row_sums, g1.row_sums) and np.array_equal(g0.col_sums, g1.col_sums)
    X, Y = clouds("normal", n, m, 65, 1)
    with pytest.raises(rg.RegotError):
        solver.set_pointcloud(X, Y, *marginals(n, m), eta, on_the_fly=True)
    solver.set_pointcloud(X, Y, *marginals(n, m), eta, on_the_fly=False)
    assert np.array_equal(solver.get_cost(), problems.problem_from_points(X, Y, eta).M)
