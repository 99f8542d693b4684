"""CPU: host-side logic of the product -- config structs, hashes, generators, value types."""
import ctypes as C

import numpy as np
import pytest

import paper_2605_08793_b200 as rg
from paper_2605_08793_b200 import _lib, problems


def fnv1a_hex(s: str) -> str:
    h = 0xCBF29CE484222325
    for ch in s.encode():
        h = ((h ^ ch) * 0x100000001B3) & ((1 << 64) - 1)
    return f"{h:016x}"


def test_config_defaults_match_reference():
    c = _lib.SplrConfigC()
    _lib.load().regot_b200_splr_config_default(C.byref(c))
    d = rg.SplrConfig()
    assert (c.tau_max, c.S, c.J, c.density, c.c1, c.c2, c.max_iter, c.tol, c.max_ls_trials, c.record_every, c.overlap,
            c.tile_rows, c.tile_cols) == (1.0, 10, 5, 0.01, 1e-4, 0.9, 1000, 1e-8, 30, 1, 0, 8, 32)  # splr.h:24-35
    assert (d.tau_max, d.S, d.J, d.density, d.c1, d.c2, d.max_iter, d.tol) == (1.0, 10, 5, 0.01, 1e-4, 0.9, 1000, 1e-8)
    k = _lib.SinkhornConfigC()
    _lib.load().regot_b200_sinkhorn_config_default(C.byref(k))
    assert (k.max_iter, k.record_every, k.tol) == (1000, 1, 0.0)  # sinkhorn.h:18-20


@pytest.mark.parametrize("bad", [dict(c1=0.6), dict(c2=1e-4), dict(S=0), dict(tau_max=0.0), dict(J=-1), dict(density=0.0),
                                 dict(density=1.5), dict(max_iter=0), dict(tol=-1.0), dict(max_ls_trials=0), dict(record_every=0)])
def test_splr_config_invariants(bad):
    # test_splr.cpp:404-421, splr.h:37-59
    with pytest.raises(rg.ValidationError, match="SplrConfig"):
        rg.SplrConfig(**bad).validate()
    rg.SplrConfig().validate()


def test_config_hashes_follow_reference_canonical_strings():
    # splr.h:62-70 / sinkhorn.h:33-39: FNV-1a of the streamed canonical string (default ostream formatting)
    assert rg.splr_config_hash(rg.SplrConfig()) == fnv1a_hex("tau_max=1;S=10;J=5;density=0.01;c1=0.0001;c2=0.9;tile=8x32")
    assert rg.splr_config_hash(rg.SplrConfig(S=4, J=3, max_iter=7, tol=0.0, overlap=True)) == \
        fnv1a_hex("tau_max=1;S=4;J=3;density=0.01;c1=0.0001;c2=0.9;tile=8x32")  # tol/max_iter/overlap not hashed
    assert rg.sinkhorn_config_hash(rg.SinkhornConfig(max_iter=40)) == fnv1a_hex("max_iter=40;tol=0")
    assert rg.sinkhorn_config_hash(rg.SinkhornConfig(max_iter=100000, tol=1e-6)) == fnv1a_hex("max_iter=100000;tol=1e-06")


def test_rng_is_mt19937_64():
    r = problems.Rng(5489)
    assert r.next_u64() == 14514284786278117030  # first output of std::mt19937_64 with the default seed
    r2 = problems.Rng(7)
    u = [r2.uniform() for _ in range(5)]
    assert all(0.0 <= v < 1.0 for v in u)


def test_generators_bit_exact_with_oracle(oracle):
    def same(p, q):
        return np.array_equal(p.M, q["M"]) and np.array_equal(p.a, q["a"]) and np.array_equal(p.b, q["b"])
    assert same(problems.gen_synthetic2(64, 50, 0.01), oracle.gen_problem("synth2", 64, 50, 0.01))
    assert same(problems.gen_synthetic1(40, 30, "iid", 2, 7, 0.01), oracle.gen_problem("synth1-iid", 40, 30, 0.01, d=2, seed=7))
    assert same(problems.gen_synthetic1(40, 30, "diff", 3, 9, 0.01), oracle.gen_problem("synth1-diff", 40, 30, 0.01, d=3, seed=9))
    assert same(problems.gen_image(12, 0.001), oracle.gen_problem("image", 144, 144, 0.001, d=12))
    assert same(problems.problem_from_points(*problems.gen_gmm_points(50, 40, 10, 21), 0.001),
                oracle.gen_problem("gmm", 50, 40, 0.001, d=10, seed=21))
    assert same(problems.problem_from_points(*problems.gen_uniform_points(50, 40, 3, 31), 0.01),
                oracle.gen_problem("uniform", 50, 40, 0.01, d=3, seed=31))


def test_generator_invariants():
    # test_problem.cpp:30-38, 122-141
    p = problems.gen_synthetic2(101, 101, 0.01)
    assert p.M.max() == 1.0 and p.M.min() >= 0.0 and (np.diff(p.a) < 0).all()
    assert p.b[20] > p.b[19] and p.b[20] > p.b[21] and p.b[60] > p.b[59] and p.b[60] > p.b[61]
    assert abs(p.a.sum() - 1) <= 1e-12 and abs(p.b.sum() - 1) <= 1e-12
    q = problems.gen_image(20, 0.001)
    assert q.M.max() == 1.0 and (q.a > 0).all() and (q.b > 0).all()
    with pytest.raises(rg.ValidationError):
        problems.gen_synthetic1(1, 5, "iid", 2, 0)
    with pytest.raises(rg.DegenerateCostError):
        problems.normalize_cost(np.zeros((2, 2)))


def test_dual_point_free_vector_round_trip():
    # test_dual.cpp:246-257
    rng = np.random.default_rng(601)
    x = rg.DualPoint(rng.normal(size=9), np.append(rng.normal(size=6), 0.0))
    xf = x.to_free()
    y = rg.DualPoint.from_free(xf, 9, 7)
    assert np.array_equal(y.alpha, x.alpha) and np.array_equal(y.beta, x.beta) and y.beta[6] == 0.0
    assert np.array_equal(y.to_free(), xf)
    with pytest.raises(rg.ValidationError):
        rg.DualPoint.from_free(np.zeros(5), 9, 7)


def test_solver_trace_ordering_invariants():
    # trace.h:26-36
    t = rg.SolverTrace()
    t.append(rg.TraceRow(0, 0.0))
    t.append(rg.TraceRow(1, 0.5))
    with pytest.raises(rg.ValidationError):
        t.append(rg.TraceRow(1, 0.6))
    with pytest.raises(rg.ValidationError):
        t.append(rg.TraceRow(2, 0.4))


def test_topk_budget_and_row_blocks():
    assert rg.topk_budget(rg.ProblemInstance(10000, 10000, None, None, None, 1.0), 0.01) == 999900  # splr.h:336-340
    assert rg.topk_budget(rg.ProblemInstance(20000, 5000, None, None, None, 1.0), 0.01) == 999800
    lib = _lib.load()
    covered = []
    for r in range(8):
        b, c = C.c_int64(), C.c_int64()
        lib.regot_b200_host_row_block(50000, r, 8, C.byref(b), C.byref(c))
        covered.append((b.value, c.value))
    assert covered[0][0] == 0 and sum(c for _, c in covered) == 50000
    assert all(covered[i][0] + covered[i][1] == covered[i + 1][0] for i in range(7))


def test_pick_bucket():
    lib = _lib.load()
    hist = (C.c_uint64 * 8)(5, 0, 3, 0, 0, 2, 0, 1)
    b, above = C.c_int(), C.c_int64()
    for need, want in [(1, (7, 0)), (2, (5, 1)), (3, (5, 1)), (4, (2, 3)), (6, (2, 3)), (7, (0, 6)), (11, (0, 6)), (12, (-1, 0))]:
        lib.regot_b200_host_pick_bucket(hist, 8, need, C.byref(b), C.byref(above))
        assert (b.value, above.value) == want, (need, b.value, above.value)
