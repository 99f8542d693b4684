"""GPU: the step-level interface -- SplrState / splr_init / splr_step (splr.h:82-97, 326-334, 348-478) over the
C ABI (regot_b200_splr_init / _splr_step / _splr_state_*).  Stepping by hand must reproduce run_splr bit for
bit, and the reference's own step-level test (spectrum sandwich at refresh, test_splr.cpp:349-378) is mirrored."""
import math
import threading

import numpy as np
import pytest

import paper_2605_08793_b200 as rg

pytestmark = pytest.mark.gpu


def to_problem(p):
    return rg.ProblemInstance(p["n"], p["m"], p["M"], p["a"], p["b"], p["eta"])


@pytest.mark.parametrize("overlap", [False, True])
def test_stepping_equals_run_splr_bitwise(solver, oracle, overlap):
    p = to_problem(oracle.gen_problem("synth2", 48, 40, 0.01))
    solver.set_problem(p)
    cfg = rg.SplrConfig(S=5, J=4, max_iter=23, tol=0.0, overlap=overlap)
    x0 = rg.DualPoint.zeros(48, 40)
    ref = solver.run_splr(x0, cfg)
    st = solver.splr_init(x0, cfg)
    assert st.iter == 0 and not st.has_prev and st.A is None
    assert st.cur.f == ref.trace.rows[0].f
    for k in range(23):
        # run_splr's loop (splr.h:509-531) by hand
        assert st.cur.marginal_error > cfg.tol
        rec = solver.splr_step(st, cfg)
        want = ref.steps[k]
        assert rec == want or (math.isnan(rec.f_cand_sinkhorn) and math.isnan(want.f_cand_sinkhorn)
                               and {**rec.__dict__, "f_cand_sinkhorn": 0} == {**want.__dict__, "f_cand_sinkhorn": 0})
        assert st.iter == k + 1 and st.has_prev
        cur = st.cur
        row = ref.trace.rows[k + 1]
        assert (cur.f, cur.marginal_error, cur.duality_gap) == (row.f, row.marginal_error, row.duality_gap)
    x = st.x
    assert np.array_equal(x.alpha, ref.x.alpha) and np.array_equal(x.beta, ref.x.beta)
    g = solver.fused_gradient(x)
    assert np.array_equal(st.cur.grad, g.grad) and np.array_equal(st.cur.row_sums, g.row_sums)
    st.free()
    with pytest.raises(rg.ValidationError):
        solver.splr_step(st, cfg)


def test_two_states_step_independently(solver, oracle):
    """States are values in the reference (splr_step takes and returns one): two of them on one context must not
    share anything but scratch."""
    p = to_problem(oracle.gen_problem("synth1-iid", 40, 36, 0.02, d=2, seed=3))
    solver.set_problem(p)
    cfg = rg.SplrConfig(S=3, J=2, max_iter=12, tol=0.0)
    ref = solver.run_splr(rg.DualPoint.zeros(40, 36), cfg)
    a = solver.splr_init(rg.DualPoint.zeros(40, 36), cfg)
    b = solver.splr_init(rg.DualPoint.zeros(40, 36), cfg)
    fa, fb = [], []
    for k in range(12):  # interleaved, b lags one step behind
        fa.append(solver.splr_step(a, cfg).f_after)
        if k:
            fb.append(solver.splr_step(b, cfg).f_after)
    fb.append(solver.splr_step(b, cfg).f_after)
    want = [s.f_after for s in ref.steps]
    assert fa == want and fb == want


def test_refresh_keeps_the_spectrum_sandwiched(solver, oracle):
    # test_splr.cpp:349-378: the freshly selected pattern must not widen the eigenvalue range of the dense
    # Hessian at the point it was built from
    n, m = 18, 14
    p = to_problem(oracle.gen_problem("rand", n, m, 0.05, seed=7401))
    solver.set_problem(p)
    cfg = rg.SplrConfig(S=4, J=2, max_iter=12, tol=0.0)
    st = solver.splr_init(rg.DualPoint.zeros(n, m), cfg)
    refreshes = 0
    for _ in range(12):
        refresh = st.iter % cfg.S == 0
        at = st.x  # the pattern is selected at this point
        rec = solver.splr_step(st, cfg)
        assert rec.refresh == refresh
        if not refresh:
            continue
        refreshes += 1
        coords = st.A.export()[3]
        HO = solver.assemble(at, rg.SparsityPattern(n, m - 1, coords), 0.0)
        colptr, rowidx, values, _ = HO.export()
        dim = n + m - 1
        D = np.zeros((dim, dim))
        for c in range(dim):
            D[rowidx[colptr[c]:colptr[c + 1]], c] = values[colptr[c]:colptr[c + 1]]
        assert np.array_equal(D, D.T)
        gr = solver.fused_gradient(at)
        T = solver.plan(at)
        H = np.zeros((dim, dim))  # hessian_dense (dual.h:191-207)
        H[np.arange(n), np.arange(n)] = gr.row_sums / p.eta
        H[n + np.arange(m - 1), n + np.arange(m - 1)] = gr.col_sums[:m - 1] / p.eta
        H[:n, n:] = T[:, :m - 1] / p.eta
        H[n:, :n] = H[:n, n:].T
        es, eh = np.linalg.eigvalsh(D), np.linalg.eigvalsh(H)
        slack = 1e-8 * eh[-1]
        assert eh[0] <= es[0] + slack and es[-1] <= eh[-1] + slack and es[0] > 0.0
    assert refreshes == 3


def test_state_is_the_resume_seam(solver, oracle):
    """Checkpoint / resume: x and iter of a state at a refresh boundary restart the solve on the
    same trajectory up to the quasi-Newton memory (the restarted state has no previous iterate)."""
    p = to_problem(oracle.gen_problem("synth2", 64, 64, 0.01))
    solver.set_problem(p)
    cfg = rg.SplrConfig(tol=1e-8, max_iter=200)
    st = solver.splr_init(rg.DualPoint.zeros(64, 64), cfg)
    for _ in range(20):
        solver.splr_step(st, cfg)
    x = st.x
    st2 = solver.splr_init(x, cfg)  # resumed from the downloaded point
    assert st2.cur.f == st.cur.f and st2.cur.marginal_error == st.cur.marginal_error
    its = 0
    while st2.cur.marginal_error > cfg.tol and its < 200:
        solver.splr_step(st2, cfg)
        its += 1
    assert st2.cur.marginal_error <= 1e-8 and its <= 40


def test_two_threads_two_handles(oracle):
    """bench.h:203-211 (`parallel_repeats`): the harness calls the solvers from several threads; entry points are
    re-entrant per handle (regot_b200.h).  Two contexts solve different problems concurrently; each result equals
    its single-threaded run bit for bit."""
    probs = [to_problem(oracle.gen_problem("synth2", 96, 80, 0.01)),
             to_problem(oracle.gen_problem("synth1-iid", 120, 90, 0.02, d=2, seed=5))]
    cfg = rg.SplrConfig(tol=1e-8, max_iter=150)
    base = []
    for p in probs:
        s = rg.Solver(0)
        s.set_problem(p)
        base.append((s.run_splr(rg.DualPoint.zeros(p.n, p.m), cfg), s.run_sinkhorn(rg.DualPoint.zeros(p.n, p.m), rg.SinkhornConfig(max_iter=50))))
        s.close()
    out, err = [None, None], []

    def work(i):
        try:
            s = rg.Solver(0)
            s.set_problem(probs[i])
            p = probs[i]
            rs = []
            for _ in range(3):
                rs.append((s.run_splr(rg.DualPoint.zeros(p.n, p.m), cfg), s.run_sinkhorn(rg.DualPoint.zeros(p.n, p.m), rg.SinkhornConfig(max_iter=50))))
            out[i] = rs
            s.close()
        except BaseException as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=work, args=(i,), daemon=True) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not err and all(o is not None for o in out), err
    for i in range(2):
        for splr, sk in out[i]:
            assert [r.f for r in splr.trace.rows] == [r.f for r in base[i][0].trace.rows]
            assert np.array_equal(splr.x.alpha, base[i][0].x.alpha) and np.array_equal(splr.x.beta, base[i][0].x.beta)
            assert np.array_equal(sk.x.alpha, base[i][1].x.alpha)
