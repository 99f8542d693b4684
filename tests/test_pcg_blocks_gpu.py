"""GPU: the block-resident Schur-complement PCG kernel (csrc/k6_pcg_blocks.cu) in all its forms -- exchanges through
L2 (flagged words), block rows as thread-block clusters (distributed shared memory), a single cluster -- against the
reference's sparse-Cholesky direction (test_splr.cpp:89-129: <= 1e-8 relative), against the older persistent kernel
and the kernel-by-kernel path, on odd grids and shapes; run-to-run bitwise; same trajectories through run_splr."""
import os

import numpy as np
import pytest

import paper_2605_08793_b200 as rg
from paper_2605_08793_b200 import problems

pytestmark = pytest.mark.gpu


def to_problem(p):
    return rg.ProblemInstance(p["n"], p["m"], np.ascontiguousarray(p["M"]), p["a"], p["b"], p["eta"])


def make_solver(**env):
    """A context created under the given REGOT_B200_* switches (they are read when the context is created)."""
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        return rg.Solver(0)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


FORMS = {
    "auto": {},
    "through-L2": {"REGOT_B200_PCG_BLOCKS_CLUSTER": 0},
    "L2 3x4": {"REGOT_B200_PCG_BLOCKS_CLUSTER": 0, "REGOT_B200_PCG_BLOCKS_GRID": "3x4"},
    "L2 7x5": {"REGOT_B200_PCG_BLOCKS_CLUSTER": 0, "REGOT_B200_PCG_BLOCKS_GRID": "7x5"},
    "clusters 5x4": {"REGOT_B200_PCG_BLOCKS_GRID": "5x4"},
    "clusters 2x3": {"REGOT_B200_PCG_BLOCKS_GRID": "2x3"},
    "clusters 9x8": {"REGOT_B200_PCG_BLOCKS_GRID": "9x8"},
    "one cluster 1x16": {"REGOT_B200_PCG_BLOCKS_GRID": "1x16"},
    "one cluster 1x3": {"REGOT_B200_PCG_BLOCKS_GRID": "1x3"},
    "older persistent kernel": {"REGOT_B200_PCG_BLOCKS": 0},
    "kernel by kernel": {"REGOT_B200_MULTIKERNEL_PCG": 1},
}


@pytest.fixture(scope="module")
def forms():
    made = {name: make_solver(**env) for name, env in FORMS.items()}
    yield made
    for s in made.values():
        s.close()


@pytest.mark.parametrize("n,m,k", [(300, 257, 6000), (90, 700, 9000), (1500, 1400, 30000), (37, 23, 200)])
def test_every_form_matches_the_cholesky_oracle(forms, oracle, n, m, k):
    # full first row / column (heavy lines in every block that meets them), ragged slices, two right-hand sides
    p = oracle.gen_problem("rand", n, m, 0.1, seed=6701)
    a0, b0 = oracle.rand_dual(n, m, 0.2, 6801)
    coords = oracle.select_topk(oracle.plan(p, a0, b0), k)
    x = rg.DualPoint(a0, b0)
    dim = n + m - 1
    gref = oracle.gradient(p, a0, b0)["grad"]
    rng = np.random.default_rng(7)
    sv = 0.05 * rng.uniform(-1, 1, dim)
    got = {}
    for name, s in forms.items():
        s.set_problem(to_problem(p))
        g = s.fused_gradient(x)
        tau = min(1.0, g.grad_norm2)
        A = s.assemble(x, rg.SparsityPattern(n, m - 1, coords), tau, g)
        R = oracle.assemble(p, a0, b0, coords, tau)
        d, its = s.compute_direction(A, g.grad, cg_rtol=1e-13)
        dr, _ = R.compute_direction(gref)
        assert its > 0 and g.grad @ d < 0, name
        assert np.linalg.norm(d - dr) <= 1e-8 * np.linalg.norm(dr), name
        # the residual through the (independent) full mat-vec kernel
        assert np.linalg.norm(A.matvec(d) + g.grad) <= 1e-9 * np.linalg.norm(g.grad), name
        # Woodbury branch: two systems in one launch
        u, v = R.matvec(sv) + 0.3 * sv, R.matvec(sv)
        xi, zeta = 1.0 / (u @ sv), -1.0 / (v @ sv)
        d2, _ = s.compute_direction(A, g.grad, u, v, xi, zeta, cg_rtol=1e-13)
        dr2, _ = R.compute_direction(gref, u, v, xi, zeta)
        assert np.linalg.norm(d2 - dr2) <= 1e-8 * np.linalg.norm(dr2), name
        # zero right-hand side: no iteration, zero direction
        d0, _ = s.compute_direction(A, np.zeros(dim))
        assert np.abs(d0).max() == 0.0, name
        got[name] = (d, d2, its)
        # bitwise run to run (the layout of a block and the dealing of its lines to threads are fixed by the pattern)
        again, _ = s.compute_direction(A, g.grad, cg_rtol=1e-13)
        assert np.array_equal(again, d), name
    ref = got["older persistent kernel"]
    for name, (d, d2, its) in got.items():
        assert np.linalg.norm(d - ref[0]) <= 1e-9 * np.linalg.norm(ref[0]), name
        assert abs(its - ref[2]) <= 1, name


def test_every_form_takes_the_same_trajectory(forms):
    p = problems.gen_synthetic1(300, 260, "iid", 2, 7, 0.01)
    cfg = rg.SplrConfig(max_iter=200, tol=1e-8)
    res = {}
    for name, s in forms.items():
        s.set_problem(p)
        res[name] = s.run_splr(rg.DualPoint.zeros(p.n, p.m), cfg)
        # and the same bits when asked again
        again = s.run_splr(rg.DualPoint.zeros(p.n, p.m), cfg)
        assert [r.f for r in again.trace.rows] == [r.f for r in res[name].trace.rows], name
        assert np.array_equal(again.x.alpha, res[name].x.alpha), name
    ref = res["older persistent kernel"]
    a = ref.trace.rows[-1]
    assert a.marginal_error <= 1e-8
    for name, r in res.items():
        b = r.trace.rows[-1]
        assert b.marginal_error <= 1e-8, name
        for u, v in zip(ref.steps[:15], r.steps[:15]):
            assert abs(u.f_after - v.f_after) <= 1e-11 * (1 + abs(u.f_after)), name
            assert abs(u.cg_iters - v.cg_iters) <= 1, name
        assert abs(a.f - b.f) <= 1e-9 * (1 + abs(a.f)), name


def test_breakdown_is_reported_like_a_failed_factorization(forms, oracle):
    # an indefinite matrix (negative shift through a negative tau is rejected, so: a pattern whose diagonal is made
    # tiny by scaling the sums) must come back as NotPositiveDefinite from every form, not hang or return garbage
    p = oracle.gen_problem("rand", 120, 100, 0.1, seed=5)
    a0, b0 = oracle.rand_dual(120, 100, 0.2, 6)
    coords = oracle.select_topk(oracle.plan(p, a0, b0), 3000)
    x = rg.DualPoint(a0, b0)
    for name in ("auto", "through-L2", "clusters 5x4", "one cluster 1x16"):
        s = forms[name]
        s.set_problem(to_problem(p))
        g = s.fused_gradient(x)
        # sums scaled down: diag = sums / eta + tau becomes much smaller than the off-diagonal row sums
        fake = rg.GradientResult(g.f, g.grad, 1e-3 * g.row_sums, 1e-3 * g.col_sums, g.marginal_error, g.duality_gap, g.grad_norm2)
        A = s.assemble(x, rg.SparsityPattern(120, 99, coords), 0.0, fake)
        with pytest.raises(rg.NotPositiveDefiniteError):
            s.compute_direction(A, g.grad, cg_rtol=1e-12)


def test_schur_diagonal_preconditioner_against_d2_on_clustered_clouds(oracle):
    """DESIGN.md K5: the PCG is preconditioned with diag(D2 - B' D1^-1 B); REGOT_B200_SCHUR_DIAG=0 keeps D2.  Both
    give the Cholesky direction (<= 1e-8); on clustered clouds (Gaussian mixtures, the family of config D), after the
    plan has concentrated, the true diagonal needs clearly fewer iterations (CPU restatement at this size: 165 -> 43)."""
    n = m = 700
    X, Y = problems.gen_gmm_points(n, m, 10, 21)
    P = problems.problem_from_points(X, Y, 0.001)
    p = {"n": n, "m": m, "M": np.ascontiguousarray(P.M), "a": P.a, "b": P.b, "eta": 0.001}
    al, be = np.zeros(n), np.zeros(m)
    for _ in range(300):
        al, be = oracle.sinkhorn_step(p, al, be)
    coords = oracle.select_topk(oracle.plan(p, al, be), oracle.topk_budget(n, m, 0.01))
    x = rg.DualPoint(al, be)
    gref = oracle.gradient(p, al, be)["grad"]
    its = {}
    for name, env in (("diag(S)", {}), ("D2", {"REGOT_B200_SCHUR_DIAG": 0}),
                      ("diag(S), kernel by kernel", {"REGOT_B200_MULTIKERNEL_PCG": 1}),
                      ("D2, kernel by kernel", {"REGOT_B200_MULTIKERNEL_PCG": 1, "REGOT_B200_SCHUR_DIAG": 0})):
        s = make_solver(**env)
        try:
            s.set_problem(to_problem(p))
            g = s.fused_gradient(x)
            tau = min(1.0, g.grad_norm2)
            A = s.assemble(x, rg.SparsityPattern(n, m - 1, coords), tau, g)
            d, its[name] = s.compute_direction(A, g.grad, cg_rtol=1e-12)
            dr, _ = oracle.assemble(p, al, be, coords, tau).compute_direction(gref)
            assert np.linalg.norm(d - dr) <= 1e-8 * np.linalg.norm(dr), name
        finally:
            s.close()
    assert 2 * its["diag(S)"] <= its["D2"], its
    assert abs(its["diag(S)"] - its["diag(S), kernel by kernel"]) <= 1 and abs(its["D2"] - its["D2, kernel by kernel"]) <= 1, its
