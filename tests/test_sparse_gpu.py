"""GPU parity: top-k sparsification (K2), assembly / value refresh (K3), mat-vec (K4),
PCG direction (K5) vs the oracle.  Mirrors test_sparsity.cpp and the direction
cases of test_splr.cpp."""
import numpy as np
import pytest

import paper_2605_08793_b200 as rg

pytestmark = pytest.mark.gpu


def to_problem(p):
    return rg.ProblemInstance(p["n"], p["m"], p["M"], p["a"], p["b"], p["eta"])


def test_worked_example(solver):
    # test_sparsity.cpp:74-85
    T = np.array([[3.0, 1, 9], [2, 2, 9], [0, 5, 9]])
    om = solver.select_topk(T, 2)
    assert om.coords.tolist() == [[0, 0], [0, 1], [1, 0], [2, 0], [2, 1]]


def test_ties_break_lexicographically(solver):
    # test_sparsity.cpp:87-99
    T = np.zeros((3, 4))
    T[0, 1] = T[1, 1] = T[1, 2] = T[2, 2] = 1.0
    c = solver.select_topk(T, 1).coords.tolist()
    assert [0, 1] in c and [1, 2] not in c and [2, 2] not in c


def test_saturation_and_minimum_set(solver):
    # test_sparsity.cpp:56-72
    rng = np.random.default_rng(0)
    T = np.abs(rng.normal(size=(5, 4)))
    om = solver.select_topk(T, 1000)
    assert len(om.coords) == 15 and om.contains_minimum_set()
    T = np.abs(rng.normal(size=(6, 5)))
    om = solver.select_topk(T, 0)
    assert len(om.coords) == 6 + 4 - 1 and om.contains_minimum_set()
    assert all(i == 0 or j == 0 for i, j in om.coords.tolist())


@pytest.mark.parametrize("seed", range(12))
def test_topk_pattern_bit_exact_with_injected_ties(solver, oracle, seed):
    # test_sparsity.cpp:101-122: the pattern must equal the oracle's exactly given identical T
    rng = np.random.default_rng(2024 + seed)
    n, m = int(2 + rng.random() * 62), int(2 + rng.random() * 62)
    T = np.where(rng.random((n, m)) < 0.3, 0.5, rng.random((n, m)))
    k = int(rng.random() * n * (m - 1))
    got = solver.select_topk(T, k).coords
    want = oracle.select_topk(T, k)
    assert got.shape == want.shape and np.array_equal(got, want)


@pytest.mark.parametrize("shape", [(300, 700), (1000, 257), (64, 2049)])
def test_topk_pattern_bit_exact_larger(solver, oracle, shape):
    n, m = shape
    rng = np.random.default_rng(n + m)
    # log-normal spread over many binades plus exact duplicates and zeros
    T = np.exp(rng.normal(size=(n, m)) * 8.0)
    T[rng.random((n, m)) < 0.05] = 0.0
    dup = rng.random((n, m)) < 0.1
    T[dup] = np.float64(2.0) ** rng.integers(-20, 5, size=dup.sum())
    for k in (1, n * (m - 1) // 100, n * (m - 1) // 3):
        got = solver.select_topk(np.asfortranarray(T), k).coords
        want = oracle.select_topk(T, k)
        assert np.array_equal(got, want)


def test_assemble_matches_oracle_csc_and_update_values_bitwise(solver, oracle):
    # test_sparsity.cpp:124-136, 172-197
    p = oracle.gen_problem("rand", 41, 29, 0.1, seed=3401)
    a0, b0 = oracle.rand_dual(41, 29, 0.2, 3402)
    a1, b1 = oracle.rand_dual(41, 29, 0.2, 3403)
    solver.set_problem(to_problem(p))
    T = oracle.plan(p, a0, b0)
    coords = oracle.select_topk(T, 120)
    om = rg.SparsityPattern(41, 28, coords, 120)
    x0, x1 = rg.DualPoint(a0, b0), rg.DualPoint(a1, b1)
    A = solver.assemble(x0, om, 0.5)
    R = oracle.assemble(p, a0, b0, coords, 0.5)
    cp, ri, va, co = A.export()
    rcp, rri, rva = R.export()
    assert np.array_equal(cp, rcp) and np.array_equal(ri, rri) and np.array_equal(co, coords)
    assert A.info()[3] == R.info()[3]  # pattern_id (FNV-1a over dim, colptr, rowidx)
    np.testing.assert_allclose(va, rva, rtol=2e-14)
    g0 = solver.fused_gradient(x0)
    diag = va[cp[:41]]
    assert np.array_equal(diag, g0.row_sums / p["eta"] + 0.5)  # diagonal == sums/eta + tau bitwise
    # update_values == fresh assemble, bitwise; idempotent
    A.update_values(x1, 0.25)
    fresh = solver.assemble(x1, om, 0.25)
    v1, v2 = A.export()[2], fresh.export()[2]
    assert np.array_equal(v1, v2)
    A.update_values(x1, 0.25)
    assert np.array_equal(A.export()[2], v1)


def test_assemble_topk_on_device_matches_dense_route(solver, oracle):
    p = oracle.gen_problem("rand", 200, 300, 0.02, seed=77)
    al, be = oracle.rand_dual(200, 300, 0.05, 78)
    solver.set_problem(to_problem(p))
    x = rg.DualPoint(al, be)
    k = rg.topk_budget(to_problem(p), 0.01)
    A = solver.assemble_topk(x, k, 0.1)
    # same T (device plan) through the dense parity entry point -> identical pattern
    T = solver.plan(x)
    want = solver.select_topk(T, k).coords
    assert np.array_equal(A.export()[3], want)
    # and against the oracle on the device's own T
    assert np.array_equal(want, oracle.select_topk(T, k))


def test_matvec_matches_oracle(solver, oracle):
    # test_sparsity.cpp:199-216
    p = oracle.gen_problem("rand", 80, 60, 0.1, seed=3501)
    al, be = oracle.rand_dual(80, 60, 0.2, 3502)
    solver.set_problem(to_problem(p))
    coords = oracle.select_topk(oracle.plan(p, al, be), 900)
    A = solver.assemble(rg.DualPoint(al, be), rg.SparsityPattern(80, 59, coords), 0.1)
    R = oracle.assemble(p, al, be, coords, 0.1)
    v = np.random.default_rng(3504).uniform(-1, 1, 139)
    y, yr = A.matvec(v), R.matvec(v)
    np.testing.assert_allclose(y, yr, rtol=0, atol=1e-13 * np.abs(yr).max() * 139)


def test_long_rows_and_columns_matvec(solver, oracle):
    # rows/columns longer than a warp's budget go through the CTA path (row 0 / column 0 of Omega*)
    n, m = 1500, 1400
    p = oracle.gen_problem("rand", n, m, 0.05, seed=9)
    al, be = oracle.rand_dual(n, m, 0.1, 10)
    solver.set_problem(to_problem(p))
    coords = oracle.select_topk(oracle.plan(p, al, be), 30000)
    A = solver.assemble(rg.DualPoint(al, be), rg.SparsityPattern(n, m - 1, coords), 0.01)
    R = oracle.assemble(p, al, be, coords, 0.01)
    v = np.random.default_rng(1).uniform(-1, 1, n + m - 1)
    y, yr = A.matvec(v), R.matvec(v)
    np.testing.assert_allclose(y, yr, rtol=0, atol=1e-12 * np.abs(yr).max())


def test_direction_matches_cholesky_oracle(solver, oracle):
    # test_splr.cpp:89-129: device PCG direction vs the reference's sparse-Cholesky route, <= 1e-8 relative
    p = oracle.gen_problem("rand", 50, 45, 0.1, seed=6700)
    a0, b0 = oracle.rand_dual(50, 45, 0.2, 6800)
    solver.set_problem(to_problem(p))
    coords = oracle.select_topk(oracle.plan(p, a0, b0), 300)
    x = rg.DualPoint(a0, b0)
    g = solver.fused_gradient(x)
    tau = min(1.0, g.grad_norm2)
    A = solver.assemble(x, rg.SparsityPattern(50, 44, coords), tau, g)
    R = oracle.assemble(p, a0, b0, coords, tau)
    d, its = solver.compute_direction(A, g.grad, cg_rtol=1e-13)
    dr, _ = R.compute_direction(oracle.gradient(p, a0, b0)["grad"])
    assert its > 0 and np.linalg.norm(d - dr) <= 1e-8 * np.linalg.norm(dr)
    assert g.grad @ d < 0
    # Woodbury branch with an active low-rank term
    rng = np.random.default_rng(5)
    s = 0.05 * rng.uniform(-1, 1, 94)
    u = R.matvec(s) + 0.3 * s  # y- with y's > 0
    v = R.matvec(s)
    xi, zeta = 1.0 / (u @ s), -1.0 / (v @ s)
    d2, _ = solver.compute_direction(A, g.grad, u, v, xi, zeta, cg_rtol=1e-13)
    dr2, _ = R.compute_direction(oracle.gradient(p, a0, b0)["grad"], u, v, xi, zeta)
    assert np.linalg.norm(d2 - dr2) <= 1e-8 * np.linalg.norm(dr2)
    # zero gradient -> zero direction (test_splr.cpp:131-140)
    d0, _ = solver.compute_direction(A, np.zeros(94))
    assert np.abs(d0).max() == 0.0


@pytest.fixture(scope="module")
def multikernel_solver():
    """A context that takes the kernel-by-kernel Schur PCG (the path of row-sharded runs and of problems
    whose iterated vector does not fit in shared memory) on one GPU."""
    import os

    os.environ["REGOT_B200_MULTIKERNEL_PCG"] = "1"
    try:
        s = rg.Solver(0)
    finally:
        del os.environ["REGOT_B200_MULTIKERNEL_PCG"]
    yield s
    s.close()


@pytest.fixture(scope="module", params=[(64, 1, "many narrow panels"), (0, 1, "one panel"), (64, 0, "pieces read from the CSR / CSC copy")])
def panel_solver(request):
    """The kernel-by-kernel Schur PCG with its half mat-vecs in PANEL form (k_spmv_panel: the gathered vector
    staged in shared memory panel by panel -- the path of config D / E and of large sharded runs), forced on
    for small problems; a 64-entry panel width gives several panels and blocks even at n = 300."""
    import os

    os.environ["REGOT_B200_MULTIKERNEL_PCG"] = "1"
    os.environ["REGOT_B200_PANEL_SPMV"] = "1"
    if request.param[0]:
        os.environ["REGOT_B200_PANEL_WIDTH"] = str(request.param[0])
    os.environ["REGOT_B200_PANEL_ELL"] = str(request.param[1])
    try:
        s = rg.Solver(0)
    finally:
        for k in ("REGOT_B200_MULTIKERNEL_PCG", "REGOT_B200_PANEL_SPMV", "REGOT_B200_PANEL_WIDTH", "REGOT_B200_PANEL_ELL"):
            os.environ.pop(k, None)
    yield s
    s.close()


@pytest.mark.parametrize("n,m,k", [(300, 257, 6000), (90, 700, 9000), (1500, 1400, 30000), (260, 2600, 14000)])
def test_panel_matvec_pcg_matches_oracle(panel_solver, oracle, n, m, k):
    # long first row / column (items of a chunk of their own; with one panel the 2599-entry row is cut into two items,
    # whose sums the consumers add), ragged panels, two right-hand sides
    p = oracle.gen_problem("rand", n, m, 0.1, seed=6701)
    a0, b0 = oracle.rand_dual(n, m, 0.2, 6801)
    coords = oracle.select_topk(oracle.plan(p, a0, b0), k)
    x = rg.DualPoint(a0, b0)
    dim = n + m - 1
    s = panel_solver
    s.set_problem(to_problem(p))
    g = s.fused_gradient(x)
    tau = min(1.0, g.grad_norm2)
    A = s.assemble(x, rg.SparsityPattern(n, m - 1, coords), tau, g)
    R = oracle.assemble(p, a0, b0, coords, tau)
    gref = oracle.gradient(p, a0, b0)["grad"]
    d, its = s.compute_direction(A, g.grad, cg_rtol=1e-13)
    dr, _ = R.compute_direction(gref)
    assert its > 0 and g.grad @ d < 0
    assert np.linalg.norm(d - dr) <= 1e-8 * np.linalg.norm(dr)
    # the residual through the (independent) full mat-vec kernel
    assert np.linalg.norm(A.matvec(d) + g.grad) <= 1e-9 * np.linalg.norm(g.grad)


def test_panel_path_solve_agrees_with_persistent_kernel(solver, panel_solver):
    from paper_2605_08793_b200 import problems

    p = problems.gen_synthetic1(300, 260, "iid", 2, 7, 0.01)
    cfg = rg.SplrConfig(max_iter=200, tol=1e-8)
    res = []
    for s in (solver, panel_solver):
        s.set_problem(p)
        res.append(s.run_splr(rg.DualPoint.zeros(p.n, p.m), cfg))
    a, b = res[0].trace.rows[-1], res[1].trace.rows[-1]
    assert a.marginal_error <= 1e-8 and b.marginal_error <= 1e-8
    for u, v in zip(res[0].steps[:15], res[1].steps[:15]):
        assert abs(u.f_after - v.f_after) <= 1e-11 * (1 + abs(u.f_after)) and abs(u.cg_iters - v.cg_iters) <= 1
    assert abs(a.f - b.f) <= 1e-9 * (1 + abs(a.f))
    # and it is deterministic: the deferred-piece lists are filled in arrival order, the sums are not
    again = panel_solver.run_splr(rg.DualPoint.zeros(p.n, p.m), cfg)
    assert [r.f for r in again.trace.rows] == [r.f for r in res[1].trace.rows]
    assert np.array_equal(again.x.alpha, res[1].x.alpha)


def test_multikernel_pcg_matches_oracle_and_persistent_kernel(solver, multikernel_solver, oracle):
    p = oracle.gen_problem("rand", 300, 257, 0.1, seed=6701)
    a0, b0 = oracle.rand_dual(300, 257, 0.2, 6801)
    coords = oracle.select_topk(oracle.plan(p, a0, b0), 6000)
    x = rg.DualPoint(a0, b0)
    dim = 300 + 257 - 1
    rng = np.random.default_rng(7)
    got = []
    for s in (solver, multikernel_solver):
        s.set_problem(to_problem(p))
        g = s.fused_gradient(x)
        tau = min(1.0, g.grad_norm2)
        A = s.assemble(x, rg.SparsityPattern(300, 256, coords), tau, g)
        d, its = s.compute_direction(A, g.grad, cg_rtol=1e-13)
        assert its > 0 and g.grad @ d < 0
        sv = 0.05 * rng.uniform(-1, 1, dim) if not got else sv
        R = oracle.assemble(p, a0, b0, coords, tau)
        u, v = R.matvec(sv) + 0.3 * sv, R.matvec(sv)
        xi, zeta = 1.0 / (u @ sv), -1.0 / (v @ sv)
        d2, _ = s.compute_direction(A, g.grad, u, v, xi, zeta, cg_rtol=1e-13)
        dr, _ = R.compute_direction(oracle.gradient(p, a0, b0)["grad"])
        dr2, _ = R.compute_direction(oracle.gradient(p, a0, b0)["grad"], u, v, xi, zeta)
        assert np.linalg.norm(d - dr) <= 1e-8 * np.linalg.norm(dr)
        assert np.linalg.norm(d2 - dr2) <= 1e-8 * np.linalg.norm(dr2)
        got.append((d, d2))
    assert np.linalg.norm(got[0][0] - got[1][0]) <= 1e-9 * np.linalg.norm(got[0][0])


def test_multikernel_pcg_solve_agrees_with_persistent_kernel(solver, multikernel_solver):
    from paper_2605_08793_b200 import problems

    p = problems.gen_synthetic2(96, 80, 0.01)
    cfg = rg.SplrConfig(max_iter=200, tol=1e-8)
    res = []
    for s in (solver, multikernel_solver):
        s.set_problem(p)
        res.append(s.run_splr(rg.DualPoint.zeros(p.n, p.m), cfg))
    a, b = res[0].trace.rows[-1], res[1].trace.rows[-1]
    assert a.marginal_error <= 1e-8 and b.marginal_error <= 1e-8
    # the same trajectory to rounding; the last few iterations sit on a plateau just above the tolerance,
    # so the crossing itself may move by a few iterations
    for u, v in zip(res[0].steps[:40], res[1].steps[:40]):
        assert abs(u.f_after - v.f_after) <= 1e-12 * (1 + abs(u.f_after))
        assert u.sinkhorn_selected == v.sinkhorn_selected and u.ls_evals == v.ls_evals
    assert abs(a.iter - b.iter) <= max(1, round(0.15 * a.iter))
    assert abs(a.f - b.f) <= 1e-9 * (1 + abs(a.f))


@pytest.mark.parametrize("n,m", [(11000, 300), (300, 11000)])
def test_persistent_pcg_with_one_phase_gathering_through_l2(solver, multikernel_solver, n, m):
    """One side longer than the shared-memory vector buffer (10,752 entries): that phase of the persistent kernel
    gathers through L2 instead.  Same trajectory as the kernel-by-kernel solve (config C's shape class)."""
    from paper_2605_08793_b200 import problems

    p = problems.gen_synthetic2(n, m, 0.01)
    cfg = rg.SplrConfig(max_iter=60, tol=1e-8)
    res = []
    for s in (solver, multikernel_solver):
        s.set_problem(p)
        res.append(s.run_splr(rg.DualPoint.zeros(p.n, p.m), cfg))
    assert len(res[0].steps) >= 10
    for u, v in zip(res[0].steps[:25], res[1].steps[:25]):
        assert abs(u.f_after - v.f_after) <= 1e-11 * (1 + abs(u.f_after)) and u.ls_evals == v.ls_evals
        assert abs(u.cg_iters - v.cg_iters) <= 1
    a, b = res[0].trace.rows[-1], res[1].trace.rows[-1]
    assert abs(a.iter - b.iter) <= max(1, round(0.15 * a.iter)) and abs(a.f - b.f) <= 1e-9 * (1 + abs(a.f))


def test_single_cluster_pcg_agrees_with_whole_grid_kernel(solver):
    """REGOT_B200_PCG_CLUSTER=16: the persistent kernel on one thread-block cluster with the hardware cluster
    barrier (an opt-in for small systems).  Same schedule code dealt over 16 CTAs instead of 148."""
    import os

    from paper_2605_08793_b200 import problems

    os.environ["REGOT_B200_PCG_CLUSTER"] = "16"
    try:
        clustered = rg.Solver(0)
    finally:
        del os.environ["REGOT_B200_PCG_CLUSTER"]
    try:
        p = problems.gen_synthetic1(300, 260, "iid", 2, 7, 0.01)
        cfg = rg.SplrConfig(max_iter=200, tol=1e-8)
        res = []
        for s in (solver, clustered):
            s.set_problem(p)
            res.append(s.run_splr(rg.DualPoint.zeros(p.n, p.m), cfg))
        a, b = res[0].trace.rows[-1], res[1].trace.rows[-1]
        assert a.marginal_error <= 1e-8 and b.marginal_error <= 1e-8
        for u, v in zip(res[0].steps[:15], res[1].steps[:15]):
            assert abs(u.f_after - v.f_after) <= 1e-11 * (1 + abs(u.f_after)) and u.cg_iters == v.cg_iters
        assert abs(a.iter - b.iter) <= max(1, round(0.15 * a.iter)) and abs(a.f - b.f) <= 1e-9 * (1 + abs(a.f))
    finally:
        clustered.close()


def test_foreign_and_invalid_inputs_rejected(solver, oracle):
    p = oracle.gen_problem("rand", 8, 6, 0.1, seed=3601)
    solver.set_problem(to_problem(p))
    x = rg.DualPoint.zeros(8, 6)
    with pytest.raises(rg.ValidationError):
        solver.assemble(x, rg.SparsityPattern(8, 5, np.array([[0, 0], [1, 1]], np.int32)), 0.1)  # Omega* missing
    with pytest.raises(rg.ValidationError):
        rg.select_topk(np.ones((3, 3)), -1)


@pytest.mark.parametrize("shift_binades", [0.0, 0.4, 3.0, -3.0, -0.6])
def test_topk_refresh_from_the_previous_threshold_bin_gives_the_same_pattern(oracle, shift_binades):
    """k2_topk.cu: a refresh starts its count sweep from the previous refresh's threshold bin (a binade of T) and runs the
    histogram sweep only when that guess is too high.  Same bin, threshold moved up (candidates: a superset) and threshold
    moved down (guess too high: the three-sweep path) must all give the pattern and values of a context without the
    guess, bit for bit, and that pattern is the oracle's."""
    import os

    n, m, k = 203, 157, 2500
    p = oracle.gen_problem("rand", n, m, 0.05, seed=811)
    a0, b0 = oracle.rand_dual(n, m, 0.1, 812)
    a1 = a0 + shift_binades * 0.05 * np.log(2.0) + 0.002 * np.cos(np.arange(n))  # T scaled by 2^shift, slightly reshuffled
    x0, x1 = rg.DualPoint(a0, b0), rg.DualPoint(a1, b0)

    def pattern_after(env, warm):
        old = os.environ.get("REGOT_B200_TOPK_GUESS")
        if env is not None:
            os.environ["REGOT_B200_TOPK_GUESS"] = env
        try:
            s = rg.Solver(0)
        finally:
            if env is not None:
                if old is None:
                    del os.environ["REGOT_B200_TOPK_GUESS"]
                else:
                    os.environ["REGOT_B200_TOPK_GUESS"] = old
        try:
            s.set_problem(to_problem(p))
            if warm:
                s.assemble_topk(x0, k, 0.1).free()  # leaves its threshold bin behind
            A = s.assemble_topk(x1, k, 0.1)
            return A.export_local()
        finally:
            s.close()

    guessed = pattern_after(None, True)
    plain = pattern_after("0", True)
    cold = pattern_after(None, False)
    for got in (guessed, cold):
        assert np.array_equal(got[0], plain[0]) and np.array_equal(got[1], plain[1])
    ref = oracle.select_topk(oracle.plan(p, a1, b0), k)
    assert np.array_equal(np.asarray(guessed[0]), np.asarray(ref))
