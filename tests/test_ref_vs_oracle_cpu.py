"""CPU: the oracle restatement against the reference's OWN code (oracle/_ref/libregot_ref.so: the
reference headers compiled unmodified over oracle/eigen_shim).  Every comparison is bitwise: the
restatement follows the reference's loop and summation order, and the Eigen stand-in reduces left to
right like the restatement does.  Skipped where oracle/_ref has not been built."""
import numpy as np
import pytest

from paper_2605_08793_b200._lib import SinkhornConfigC, SplrConfigC
from tests import oracle_lib

ref = oracle_lib.load_ref()
pytestmark = pytest.mark.skipif(ref is None, reason="oracle/_ref not built (needs /root/reference)")

GOLDEN_F = [1.6638586759335181, 0.29051373543167602, 0.21054519582141862, 0.095970055531796022,
            0.063997930975742745, 0.044099819557298296, 0.026713859915931643]


def cfg(**kw):
    c = SplrConfigC(1.0, 10, 5, 0.01, 1e-4, 0.9, 1000, 1e-8, 30, 1, 0, 8, 32, 0, 0.0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def test_reference_code_reproduces_its_golden_trajectory():
    # test_splr.cpp:380-402 through the reference's own run_splr
    p = ref.gen_problem("synth2", 32, 32, 0.01)
    res = ref.run_splr(p, np.zeros(32), np.zeros(32), cfg(S=1, J=0, max_iter=6, tol=0.0))
    assert len(res["trace"]) == 7
    for row, want in zip(res["trace"], GOLDEN_F):
        assert abs(row[2] - want) <= 1e-12 * want


@pytest.mark.parametrize("kind,n,m,eta,d,seed", [("synth2", 64, 50, 0.01, 2, 0), ("synth1-iid", 40, 30, 0.01, 2, 7),
                                                  ("synth1-diff", 33, 47, 0.05, 3, 9), ("synth2", 32, 32, 0.001, 2, 0)])
def test_generators_and_kernels_bitwise(oracle, kind, n, m, eta, d, seed):
    p, q = oracle.gen_problem(kind, n, m, eta, d=d, seed=seed), ref.gen_problem(kind, n, m, eta, d=d, seed=seed)
    assert np.array_equal(p["M"], q["M"]) and np.array_equal(p["a"], q["a"]) and np.array_equal(p["b"], q["b"])
    al, be = oracle.rand_dual(n, m, 0.05, 99)
    for naive in (False, True):
        g, h = oracle.gradient(p, al, be, naive=naive), ref.gradient(p, al, be, naive=naive)
        assert g["f"] == h["f"] and np.array_equal(g["grad"], h["grad"]) and np.array_equal(g["col"], h["col"])
        assert g["marginal_error"] == h["marginal_error"] and g["duality_gap"] == h["duality_gap"]
    for tr, tc in [(1, 1), (3, 5), (64, 64)]:
        assert np.array_equal(oracle.gradient(p, al, be, tr=tr, tc=tc)["grad"], ref.gradient(p, al, be, tr=tr, tc=tc)["grad"])
    assert np.array_equal(oracle.plan(p, al, be), ref.plan(p, al, be))
    assert np.array_equal(oracle.optimal_alpha(p, al, be), ref.optimal_alpha(p, al, be))
    assert np.array_equal(oracle.optimal_beta(p, al), ref.optimal_beta(p, al))
    xa, xb = oracle.sinkhorn_step(p, al, be)
    ya, yb = ref.sinkhorn_step(p, al, be)
    assert np.array_equal(xa, ya) and np.array_equal(xb, yb) and xb[-1] == 0.0


def test_topk_assemble_direction_bitwise(oracle):
    rng = np.random.default_rng(2024)
    for _ in range(8):
        n, m = int(2 + rng.random() * 62), int(2 + rng.random() * 62)
        T = np.where(rng.random((n, m)) < 0.3, 0.5, rng.random((n, m)))
        k = int(rng.random() * n * (m - 1))
        assert np.array_equal(oracle.select_topk(T, k), ref.select_topk(T, k))
    p = oracle.gen_problem("rand", 41, 29, 0.1, seed=3401)
    a0, b0 = oracle.rand_dual(41, 29, 0.2, 3402)
    a1, b1 = oracle.rand_dual(41, 29, 0.2, 3403)
    coords = oracle.select_topk(oracle.plan(p, a0, b0), 120)
    A, R = oracle.assemble(p, a0, b0, coords, 0.5), ref.assemble(p, a0, b0, coords, 0.5)
    assert A.info() == R.info()  # dim, nnz, |Omega|, FNV-1a pattern id
    assert all(np.array_equal(x, y) for x, y in zip(A.export(), R.export()))
    A.update_values(a1, b1, 0.25)
    R.update_values(a1, b1, 0.25)
    assert np.array_equal(A.export()[2], R.export()[2])
    v = rng.uniform(-1, 1, 69)
    assert np.array_equal(A.matvec(v), R.matvec(v))
    g = oracle.gradient(p, a1, b1)["grad"]
    d1, _ = A.compute_direction(g)
    d2, _ = R.compute_direction(g)
    assert np.array_equal(d1, d2)  # AMD ordering, symbolic, numeric factorisation and solve all agree bitwise
    s = 0.05 * rng.uniform(-1, 1, 69)
    u, w = A.matvec(s) + 0.3 * s, A.matvec(s)
    d3, _ = A.compute_direction(g, u, w, 1.0 / (u @ s), -1.0 / (w @ s))
    d4, _ = R.compute_direction(g, u, w, 1.0 / (u @ s), -1.0 / (w @ s))
    assert np.array_equal(d3, d4)


@pytest.mark.parametrize("kind,eta,kw", [("synth2", 0.01, {}), ("synth1-iid", 0.01, {}), ("synth2", 0.001, dict(max_iter=400)),
                                         ("synth2", 0.01, dict(S=4, J=3, max_iter=24, tol=0.0))])
def test_run_splr_traces_and_step_records_bitwise(oracle, kind, eta, kw):
    n = 64 if "S" not in kw else 32
    p = oracle.gen_problem(kind, n, n, eta, d=2, seed=7)
    c = cfg(max_iter=200)
    for k, v in kw.items():
        setattr(c, k, v)
    a, b = oracle.run_splr(p, np.zeros(n), np.zeros(n), c), ref.run_splr(p, np.zeros(n), np.zeros(n), c)
    assert [(r[0], r[2], r[3], r[4]) for r in a["trace"]] == [(r[0], r[2], r[3], r[4]) for r in b["trace"]]
    for s, t in zip(a["steps"], b["steps"]):
        for key in ("iter", "refresh", "sinkhorn_selected", "f_after", "f_cand_qn", "gamma", "g_dot_d", "gnew_dot_d",
                    "curvature_ok", "ls_failed", "lowrank_active", "tau", "factor_retries", "ls_evals"):
            assert s[key] == t[key], (s["iter"], key)
    assert np.array_equal(a["alpha"], b["alpha"]) and np.array_equal(a["beta"], b["beta"])


def test_run_sinkhorn_bitwise(oracle):
    p = oracle.gen_problem("synth2", 24, 24, 0.01)
    for c in (SinkhornConfigC(40, 1, 0.0), SinkhornConfigC(100000, 100000, 1e-6)):
        a, b = oracle.run_sinkhorn(p, np.zeros(24), np.zeros(24), c), ref.run_sinkhorn(p, np.zeros(24), np.zeros(24), c)
        assert [(r[0], r[2], r[3], r[4]) for r in a["trace"]] == [(r[0], r[2], r[3], r[4]) for r in b["trace"]]
        assert np.array_equal(a["alpha"], b["alpha"])


def test_error_classes_agree(oracle):
    p = oracle.gen_problem("rand", 6, 5, 0.1, seed=1)
    for o in (oracle, ref):
        be = np.zeros(5)
        be[4] = 1e-3
        with pytest.raises(RuntimeError, match="status 4.*gauge violated"):
            o.gradient(p, np.zeros(6), be)
        with pytest.raises(RuntimeError, match="status 4"):
            o.run_splr(p, np.zeros(6), np.zeros(5), cfg(c1=0.6))
