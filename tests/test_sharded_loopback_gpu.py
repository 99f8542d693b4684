"""The row-sharded device path (north_star item 5) executed for real on ONE GPU: R contexts -- one per rank,
each holding its row block -- driven from R threads of this process, with the product's NCCL function table
pointed at the loopback communicator of tests/fake_nccl (REGOT_B200_NCCL_LIB).  Every collective of the
sharded path runs: the allreduce of column sums and scalars (K1), max + rescale + sum of the column LSE (K8),
the u64 histogram allreduces and the tie-count exchange of the global top-k (K2), B't of the kernel-by-kernel
PCG (K4/K5), the zero-padded allgather of alpha, both communicators (main / side stream).

Bar: sharded == unsharded -- bitwise where the arithmetic is rank-local (row sums, alpha, the pattern),
<= 1e-12 where only the summation order over ranks differs, <= 1e-8 for the direction, same iteration
count and f <= 1e-9 for whole solves."""
import os
import threading

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
FAKE = os.path.join(HERE, "fake_nccl", "libfakenccl.so")
# must be in the environment before the library first resolves NCCL (it does so lazily, at the first comm_init)
os.environ.setdefault("REGOT_B200_NCCL_LIB", FAKE)

import paper_2605_08793_b200 as rg  # noqa: E402
from paper_2605_08793_b200 import problems  # noqa: E402

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]


def to_problem(p):
    return rg.ProblemInstance(p["n"], p["m"], p["M"], p["a"], p["b"], p["eta"])


def row_block(n, r, R):
    return (n * r) // R, (n * (r + 1)) // R - (n * r) // R


def run_ranks(R, p, fn, pointcloud=None):
    """fn(solver, rank) on R contexts of cuda:0, one thread each; returns the list of results."""
    assert os.path.exists(FAKE), "tests/fake_nccl/libfakenccl.so is missing: __graft_entry__.build() makes it"
    ids = rg.Solver.comm_unique_id()
    out, err = [None] * R, []

    def work(r):
        s = None
        try:
            s = rg.Solver(0)
            s.comm_init(r, R, ids)
            if pointcloud is not None:
                X, Y, a, b, eta, otf = pointcloud
                s.set_pointcloud(X, Y, a, b, eta, on_the_fly=otf, rows=row_block(X.shape[0], r, R))
            else:
                s.set_problem(p, rows=row_block(p.n, r, R))
            out[r] = fn(s, r)
        except BaseException as e:  # noqa: BLE001
            err.append((r, e))
        finally:
            if s is not None:
                s.close()

    th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=500)
    assert not any(t.is_alive() for t in th), "a rank is stuck"
    if err:
        raise err[0][1]
    return out


def merge_rows(parts, n, R):
    full = np.zeros(n)
    for r, v in enumerate(parts):
        b, c = row_block(n, r, R)
        full[b:b + c] = v[b:b + c]
    return full


@pytest.mark.parametrize("R", [2, 3, 4])
def test_sharded_gradient_and_sinkhorn_equal_unsharded(solver, oracle, R):
    n, m = 203, 157  # ragged in both directions; row blocks of unequal size
    p = to_problem(oracle.gen_problem("rand", n, m, 0.05, seed=510 + R))
    al, be = oracle.rand_dual(n, m, 0.1, 511)
    x = rg.DualPoint(al, be)
    solver.set_problem(p)
    g0 = solver.fused_gradient(x)
    s0 = solver.sinkhorn_step(x)
    b0 = solver.optimal_beta(al)
    a0 = solver.optimal_alpha(x)

    def fn(s, r):
        s.validate_problem()
        return s.fused_gradient(x), s.sinkhorn_step(x), s.optimal_beta(al), s.optimal_alpha(x)

    res = run_ranks(R, p, fn)
    rows = merge_rows([q[0].row_sums for q in res], n, R)
    assert np.array_equal(rows, g0.row_sums)  # row sums are rank-local: bitwise
    assert np.array_equal(merge_rows([q[3] for q in res], n, R), a0)
    for g, sk, ob, _ in res:
        np.testing.assert_allclose(g.col_sums, g0.col_sums, rtol=1e-12)
        assert abs(g.f - g0.f) <= 1e-12 * (1 + abs(g0.f))
        assert abs(g.marginal_error - g0.marginal_error) <= 1e-12 * (1 + g0.marginal_error)
        assert abs(g.duality_gap - g0.duality_gap) <= 1e-11 * (1 + abs(g0.duality_gap))
        assert abs(g.grad_norm2 - g0.grad_norm2) <= 1e-12 * (1 + g0.grad_norm2)
        np.testing.assert_allclose(g.grad[n:], g0.grad[n:], rtol=0, atol=1e-12 * np.abs(g0.col_sums).max())
        np.testing.assert_allclose(ob, b0, rtol=0, atol=1e-12)
        np.testing.assert_allclose(sk.beta, s0.beta, rtol=0, atol=1e-12)
        assert sk.beta[-1] == 0.0
    # every rank holds the same replicated beta-side results, bit for bit
    for q in res[1:]:
        assert np.array_equal(q[0].col_sums, res[0][0].col_sums) and q[0].f == res[0][0].f
        assert np.array_equal(q[1].beta, res[0][1].beta)
    al1 = merge_rows([q[1].alpha for q in res], n, R)
    np.testing.assert_allclose(al1, s0.alpha, rtol=0, atol=1e-12)


def _tie_problem(oracle, n, m, R):
    """Rows straddling every shard boundary are made identical (cost rows, alpha), so the plan has exact
    ties whose members live on different ranks (sparsity.h:69-75: ties are taken in row-major order)."""
    p = oracle.gen_problem("rand", n, m, 0.1, seed=99)
    al, be = oracle.rand_dual(n, m, 0.05, 98)
    M = np.array(p["M"])
    for r in range(1, R):
        b = (n * r) // R
        for i in (b - 2, b - 1, b + 1):
            M[i] = M[b]
            al[i] = al[b]
    p["M"] = M
    return to_problem(p), al, be


@pytest.mark.parametrize("R", [2, 3, 4])
def test_sharded_topk_pattern_bit_exact_with_ties_across_the_boundary(solver, oracle, R):
    n, m = 96, 70
    p, al, be = _tie_problem(oracle, n, m, R)
    x = rg.DualPoint(al, be)
    solver.set_problem(p)
    T = solver.plan(x)
    gr = solver.fused_gradient(x)
    # candidates in the reference's order (value desc, row-major index asc), last column excluded
    cand = T[:, :m - 1].ravel()
    order = np.lexsort((np.arange(cand.size), -cand))
    b = (n * 1) // R
    # position (in that order) of the tie group {b-2, b-1, b, b+1} x {column j}: cut inside it
    pos = {int(q): t for t, q in enumerate(order)}
    ks = set()
    for j in (3, 17, 40):
        first = pos[(b - 2) * (m - 1) + j]
        assert T[b - 2, j] == T[b - 1, j] == T[b, j] == T[b + 1, j]
        ks.update({first + 1, first + 2, first + 3})
    ks.update({0, 1, n * (m - 1) // 10, n * (m - 1)})
    for k in sorted(ks):
        want = oracle.select_topk(T, k)
        A0 = solver.assemble_topk(x, k, 0.1, gr)
        c0, v0 = A0.export_local()
        assert np.array_equal(c0, want)

        def fn(s, r):
            A = s.assemble_topk(x, k, 0.1, gr)
            return A.export_local()

        parts = run_ranks(R, p, fn)
        coords = np.concatenate([c for c, _ in parts])
        vals = np.concatenate([v for _, v in parts])
        assert np.array_equal(coords, want), f"k={k}"
        assert np.array_equal(vals, v0)  # same plan_entry definition on every rank
        for r, (c, _) in enumerate(parts):
            lo, cnt = row_block(n, r, R)
            assert c.shape[0] == 0 or (c[:, 0].min() >= lo and c[:, 0].max() < lo + cnt)


@pytest.mark.parametrize("R", [2, 3])
def test_sharded_matvec_and_direction(solver, oracle, R):
    n, m = 150, 130
    p = to_problem(oracle.gen_problem("rand", n, m, 0.05, seed=4100))
    al, be = oracle.rand_dual(n, m, 0.1, 4101)
    x = rg.DualPoint(al, be)
    solver.set_problem(p)
    gr = solver.fused_gradient(x)
    k = 3000
    A0 = solver.assemble_topk(x, k, 0.3, gr)
    rng = np.random.default_rng(5)
    dim = n + m - 1
    v = rng.uniform(-1, 1, dim)
    y0 = A0.matvec(v)
    g = gr.grad
    u = rng.normal(size=dim)
    w = A0.matvec(rng.normal(size=dim))
    d0, _ = solver.compute_direction(A0, g)
    d1, _ = solver.compute_direction(A0, g, u, w, xi=0.7, zeta=-0.4)

    def fn(s, r):
        A = s.assemble_topk(x, k, 0.3, gr)
        return A.matvec(v), s.compute_direction(A, g)[0], s.compute_direction(A, g, u, w, xi=0.7, zeta=-0.4)[0]

    res = run_ranks(R, p, fn)
    for idx, ref, tol in ((0, y0, 1e-12), (1, d0, 1e-8), (2, d1, 1e-8)):
        full = np.concatenate([merge_rows([q[idx][:n] for q in res], n, R), res[0][idx][n:]])
        np.testing.assert_allclose(full, ref, rtol=0, atol=tol * max(1.0, np.abs(ref).max()))
        for q in res[1:]:
            assert np.array_equal(q[idx][n:], res[0][idx][n:])  # replicated beta block: identical on every rank


@pytest.mark.parametrize("R,overlap", [(2, False), (2, True), (4, False)])
def test_sharded_run_splr_config_A(solver, R, overlap):
    """BASELINE config A (n = m = 1000, eta = 0.01), full solve: same iteration count, f within 1e-9."""
    p = problems.gen_synthetic1(1000, 1000, "iid", 2, 7, 0.01)
    cfg = rg.SplrConfig(tol=1e-8, overlap=overlap)
    x0 = rg.DualPoint.zeros(p.n, p.m)
    solver.set_problem(p)
    ref = solver.run_splr(x0, cfg)

    def fn(s, r):
        return s.run_splr(x0, cfg)

    res = run_ranks(R, p, fn)
    last0 = ref.trace.rows[-1]
    for q in res:
        last = q.trace.rows[-1]
        assert last.marginal_error <= 1e-8
        assert last.iter == last0.iter, (last.iter, last0.iter)
        assert abs(last.f - last0.f) <= 1e-9 * (1 + abs(last0.f))
        np.testing.assert_allclose(q.x.beta, ref.x.beta, rtol=0, atol=1e-7)
        np.testing.assert_allclose(q.x.alpha, ref.x.alpha, rtol=0, atol=1e-7)  # allgathered over the ranks
        for a, b in zip(q.trace.rows[:20], ref.trace.rows[:20]):
            assert abs(a.f - b.f) <= 1e-9 * (1 + abs(b.f))
    for q in res[1:]:  # ranks take identical decisions from identical (allreduced) scalars
        assert [s.ls_evals for s in q.steps] == [s.ls_evals for s in res[0].steps]
        assert [t.f for t in q.trace.rows] == [t.f for t in res[0].trace.rows]
        assert np.array_equal(q.x.beta, res[0].x.beta) and np.array_equal(q.x.alpha, res[0].x.alpha)


def test_sharded_pattern_reuse_takes_the_same_decisions_as_one_gpu():
    """Pattern reuse (regot_b200_set_pattern_reuse): the captured-mass share is allreduced, so every rank keeps or rebuilds
    the pattern at the same refreshes as the unsharded solve (shares differ in the last bits only)."""
    p = problems.gen_synthetic2(256, 192, 0.005)
    cfg = rg.SplrConfig(tol=1e-8)
    x0 = rg.DualPoint.zeros(p.n, p.m)
    one = rg.Solver(0)
    try:
        one.set_pattern_reuse(0.5, 3)
        one.set_problem(p)
        ref = one.run_splr(x0, cfg)
        counts0 = one.pattern_counts()
    finally:
        one.close()
    assert counts0[1] >= 1

    def fn(s, r):
        s.set_pattern_reuse(0.5, 3)
        q = s.run_splr(x0, cfg)
        return q, s.pattern_counts()

    res = run_ranks(2, p, fn)
    last0 = ref.trace.rows[-1]
    for q, counts in res:
        last = q.trace.rows[-1]
        assert last.marginal_error <= 1e-8
        assert counts == counts0, (counts, counts0)
        assert abs(last.iter - last0.iter) <= 2
        assert abs(last.f - last0.f) <= 1e-9 * (1 + abs(last0.f))
    assert [t.f for t in res[0][0].trace.rows] == [t.f for t in res[1][0].trace.rows]


def test_sharded_overlap_is_bitwise_identical_to_serial(oracle):
    """cfg.overlap moves the candidate chain to the side stream and the side communicator; results must not
    change (test_splr.cpp:270-305), also when sharded."""
    p = to_problem(oracle.gen_problem("synth2", 96, 80, 0.01))
    x0 = rg.DualPoint.zeros(p.n, p.m)
    runs = {}
    for overlap in (False, True):
        cfg = rg.SplrConfig(tol=1e-8, max_iter=60, overlap=overlap)
        runs[overlap] = run_ranks(2, p, lambda s, r: s.run_splr(x0, cfg))
    for r in range(2):
        a, b = runs[False][r], runs[True][r]
        assert [t.f for t in a.trace.rows] == [t.f for t in b.trace.rows]
        assert np.array_equal(a.x.alpha, b.x.alpha) and np.array_equal(a.x.beta, b.x.beta)


def test_sharded_run_sinkhorn_and_pointcloud(solver, oracle):
    # point-cloud rows: the cost maximum is allreduced; materialised and on-the-fly agree bitwise per rank
    rng = np.random.default_rng(8)
    n, m, d = 300, 260, 3
    X, Y = rng.random((n, d)), rng.random((m, d))
    a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    solver.set_pointcloud(X, Y, a, b, 0.05)
    cfg = rg.SinkhornConfig(max_iter=40, tol=1e-9)
    x0 = rg.DualPoint.zeros(n, m)
    ref = solver.run_sinkhorn(x0, cfg)
    M0 = solver.get_cost()
    for otf in (False, True):
        res = run_ranks(3, None, lambda s, r: (s.run_sinkhorn(x0, cfg), s.get_cost()), pointcloud=(X, Y, a, b, 0.05, otf))
        assert np.array_equal(np.concatenate([q[1] for q in res]), M0)  # global maximum on every rank
        for q, _ in res:
            assert q.trace.rows[-1].iter == ref.trace.rows[-1].iter
            np.testing.assert_allclose(q.x.beta, ref.x.beta, rtol=0, atol=1e-11)
            np.testing.assert_allclose(q.x.alpha, ref.x.alpha, rtol=0, atol=1e-11)
            assert abs(q.trace.rows[-1].marginal_error - ref.trace.rows[-1].marginal_error) <= 1e-11


def test_a_fast_update_flagged_on_one_rank_is_redone_by_all_of_them(solver):
    """The gradient-sweep form of a Sinkhorn update is exact only while every sum lies in [e^-600, e^600]; outside it the
    update is flagged and redone with the log-sum-exp kernels.  Row sums are rank-local, so the flag travels with the
    gradient pass's allreduce payload: here only the rows of the LAST rank are out of range at x0 = 0 (costs >= 0.75 at
    eta = 0.001), and every rank must still take the same kernels (a rank on its own would desynchronise the collectives)."""
    rng = np.random.default_rng(3)
    n, m = 192, 160
    M = rng.random((n, m))
    M[n // 2:, :] = 0.75 + 0.25 * M[n // 2:, :]
    p = rg.ProblemInstance(n, m, M, np.full(n, 1.0 / n), np.full(m, 1.0 / m), 0.001)
    x0 = rg.DualPoint.zeros(n, m)
    kcfg = rg.SinkhornConfig(max_iter=12, tol=1e-9)
    scfg = rg.SplrConfig(max_iter=12, tol=1e-8)
    solver.set_problem(p)
    ref_k = solver.run_sinkhorn(x0, kcfg)
    ref_s = solver.run_splr(x0, scfg)

    def fn(s, r):
        return s.run_sinkhorn(x0, kcfg), s.run_splr(x0, scfg)

    for qk, qs in run_ranks(2, p, fn):
        for q, ref in ((qk, ref_k), (qs, ref_s)):
            assert len(q.trace.rows) == len(ref.trace.rows)
            for u, v in zip(q.trace.rows, ref.trace.rows):
                assert abs(u.f - v.f) <= 1e-9 * (1 + abs(v.f)), (u.iter, u.f, v.f)
        np.testing.assert_allclose(qk.x.beta, ref_k.x.beta, rtol=0, atol=1e-9)
