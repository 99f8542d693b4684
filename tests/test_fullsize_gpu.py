"""GPU: the BASELINE.json configurations at FULL size, checked through size-independent properties
(the oracle cannot run these sizes in seconds): conservation of mass, exact scaling of the plan,
marginals reproduced by the Sinkhorn updates, the top-k pattern against a numpy selection on the
downloaded plan (bit-exact, ties included), value refresh == fresh assembly, the direction's
residual, on-the-fly == materialised, and a full solve to 1e-8.

  B  n = m = 10,000 image histograms (100 x 100 grids), eta = 0.001
  C  n = 20,000 x m = 5,000 synthetic II, eta = 0.0005
  D  n = m = 50,000 Gaussian mixtures in R^10, eta = 0.001 (20 GB block, materialised on the device)
  E  n = m = 100,000 uniform clouds in R^3, eta = 0.01, cost formed on the fly
"""
import math

import numpy as np
import pytest

import paper_2605_08793_b200 as rg
from paper_2605_08793_b200 import problems

pytestmark = pytest.mark.gpu


def image_clouds(side):
    """Config B as point clouds: pixel (r, c) -> (c, r) / (side - 1); |p - q|^2 / max == gen_image's cost."""
    s = 1.0 / float(side - 1)
    idx = np.arange(side * side)
    xs, ys = (idx % side).astype(np.float64) * s, (idx // side).astype(np.float64) * s
    return np.stack([xs, ys], axis=1)


def check_pass_properties(solver, n, m, eta, x):
    g = solver.fused_gradient(x)
    # conservation: row sums, column sums and the total are the same mass
    tot_r, tot_c = math.fsum(g.row_sums), math.fsum(g.col_sums)
    assert abs(tot_r - tot_c) <= 1e-11 * tot_r and abs(g.total_mass - tot_r) <= 1e-11 * tot_r
    # T(alpha + c, beta) = e^{c / eta} T(alpha, beta): every row sum scales by the same factor
    c = 0.25 * eta
    g2 = solver.fused_gradient(rg.DualPoint(x.alpha + c, x.beta))
    np.testing.assert_allclose(g2.row_sums, math.exp(c / eta) * g.row_sums, rtol=2e-11)
    np.testing.assert_allclose(g2.col_sums, math.exp(c / eta) * g.col_sums, rtol=2e-11)
    return g


def check_sinkhorn_properties(solver, a, b, x):
    # optimal_alpha: row sums of the new plan equal a; sinkhorn_step: column sums equal b (sinkhorn.h:44-115)
    al = solver.optimal_alpha(x)
    g = solver.fused_gradient(rg.DualPoint(al, x.beta))
    np.testing.assert_allclose(g.row_sums, a, rtol=1e-10)
    y = solver.sinkhorn_step(x)
    assert y.beta[-1] == 0.0
    g = solver.fused_gradient(y)
    np.testing.assert_allclose(g.col_sums, b, rtol=1e-10)
    return y


def check_against_oracle(solver, oracle, p, x):
    """One fused_gradient pass and one sinkhorn_step of the CPU oracle on the FULL matrix (a few seconds each)
    against the device: sums, objective, gradient and the Sinkhorn update at the same point."""
    op = dict(n=p.n, m=p.m, M=np.asfortranarray(p.M), a=p.a, b=p.b, eta=p.eta)
    g = solver.fused_gradient(x)
    ref = oracle.gradient(op, x.alpha, x.beta)
    np.testing.assert_allclose(g.row_sums, ref["row"], rtol=1e-11)
    np.testing.assert_allclose(g.col_sums, ref["col"], rtol=1e-11)
    assert abs(g.f - ref["f"]) <= 1e-11 * (1 + abs(ref["f"]))
    scale = max(np.abs(ref["row"]).max(), np.abs(ref["col"]).max())
    np.testing.assert_allclose(g.grad, ref["grad"], rtol=0, atol=1e-11 * scale)
    err = np.abs(ref["row"] - p.a).sum() + np.abs(ref["col"] - p.b).sum()
    assert abs(g.marginal_error - err) <= 1e-11 * (1 + err)
    y = solver.sinkhorn_step(x)
    ra, rb = oracle.sinkhorn_step(op, x.alpha, x.beta)
    np.testing.assert_allclose(y.alpha, ra, rtol=0, atol=1e-11)
    np.testing.assert_allclose(y.beta, rb, rtol=0, atol=1e-11)
    assert y.beta[-1] == 0.0 and rb[-1] == 0.0


def test_config_b_oracle_parity_full_matrix(solver, oracle):
    p = problems.gen_image(100, 0.001)
    solver.set_problem(p)
    x = rg.DualPoint.zeros(p.n, p.m)
    for _ in range(3):
        x = solver.sinkhorn_step(x)
    check_against_oracle(solver, oracle, p, x)


def test_config_c_oracle_parity_full_matrix(solver, oracle):
    p = problems.gen_synthetic2(20000, 5000, 0.0005)
    solver.set_problem(p)
    x = rg.DualPoint.zeros(p.n, p.m)
    for _ in range(2):
        x = solver.sinkhorn_step(x)
    check_against_oracle(solver, oracle, p, x)


def test_config_b_full_size(solver):
    side, eta = 100, 0.001
    p = problems.gen_image(side, eta)
    n, m = p.n, p.m
    solver.set_problem(p)
    solver.validate_problem()
    x = rg.DualPoint.zeros(n, m)
    for _ in range(3):
        x = solver.sinkhorn_step(x)
    g = check_pass_properties(solver, n, m, eta, x)
    check_sinkhorn_properties(solver, p.a, p.b, x)

    # the same problem from its point clouds, materialised and on the fly: same cost bits, same pass bits
    P = image_clouds(side)
    solver.set_pointcloud(P, P, p.a, p.b, eta, on_the_fly=True)
    gf = solver.fused_gradient(x)
    assert gf.f == g.f and np.array_equal(gf.row_sums, g.row_sums) and np.array_equal(gf.col_sums, g.col_sums)
    solver.set_problem(p)

    # top-k pattern == numpy selection on the downloaded plan, ties in row-major order (sparsity.h:44-91)
    T = solver.plan(x)
    k = rg.topk_budget(p, 0.01)
    A = solver.assemble_topk(x, k, 0.5, g)
    colptr, rowidx, values, coords = A.export()
    Tm = T[:, : m - 1]
    flat = Tm.ravel()
    kth = np.partition(flat, flat.size - k)[flat.size - k]
    sel = flat > kth
    ties = np.flatnonzero(flat == kth)
    sel[ties[: k - int(sel.sum())]] = True
    want = sel.reshape(n, m - 1)
    want[0, :] = True
    want[:, 0] = True
    got = np.zeros((n, m - 1), dtype=bool)
    got[coords[:, 0], coords[:, 1]] = True
    assert coords.shape[0] == int(want.sum()) and np.array_equal(got, want)

    # update_values == fresh assemble, bitwise (test_sparsity.cpp:172-197)
    y = solver.sinkhorn_step(x)
    gy = solver.fused_gradient(y)
    A.update_values(y, 0.25, gy)
    B = solver.assemble(y, rg.SparsityPattern(n, m - 1, coords), 0.25, gy)
    assert np.array_equal(A.export()[2], B.export()[2])

    # direction: residual of the Newton system through the mat-vec
    d, its = solver.compute_direction(B, gy.grad, cg_rtol=1e-10)
    r = B.matvec(d) + gy.grad
    assert its > 0 and np.linalg.norm(r) <= 1e-8 * np.linalg.norm(gy.grad) and gy.grad @ d < 0

    # full solve to tolerance; accepted steps never increase the objective
    res = solver.run_splr(rg.DualPoint.zeros(n, m), rg.SplrConfig(tol=1e-8))
    last = res.trace.rows[-1]
    assert last.marginal_error <= 1e-8 and last.iter < 200
    fs = [s.f_after for s in res.steps]
    assert all(f1 <= f0 + 1e-12 * (1 + abs(f0)) for f0, f1 in zip(fs, fs[1:]))
    chk = solver.fused_gradient(res.x)
    assert chk.marginal_error <= 1e-8 and abs(chk.f - last.f) <= 1e-12 * (1 + abs(last.f))


def test_config_c_full_size(solver):
    p = problems.gen_synthetic2(20000, 5000, 0.0005)
    solver.set_problem(p)
    x = rg.DualPoint.zeros(p.n, p.m)
    for _ in range(2):
        x = solver.sinkhorn_step(x)
    check_pass_properties(solver, p.n, p.m, p.eta, x)
    check_sinkhorn_properties(solver, p.a, p.b, x)


def test_config_d_full_size(solver):
    n = m = 50000
    X, Y = problems.gen_gmm_points(n, m, 10, 21)
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    solver.set_pointcloud(X, Y, a, b, 0.001)  # 20 GB cost block built on the device
    x = rg.DualPoint.zeros(n, m)
    for _ in range(2):
        x = solver.sinkhorn_step(x)
    check_pass_properties(solver, n, m, 0.001, x)
    check_sinkhorn_properties(solver, a, b, x)
    # free the block for the tests that follow
    solver.set_problem(problems.gen_synthetic2(8, 8, 0.1))


def test_config_e_full_size_on_the_fly(solver):
    n = m = 100000
    X, Y = problems.gen_uniform_points(n, m, 3, 31)
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    solver.set_pointcloud(X, Y, a, b, 0.01, on_the_fly=True)
    x = rg.DualPoint.zeros(n, m)
    x = solver.sinkhorn_step(x)
    check_pass_properties(solver, n, m, 0.01, x)
    check_sinkhorn_properties(solver, a, b, x)
    solver.set_problem(problems.gen_synthetic2(8, 8, 0.1))
