"""Pattern reuse across refreshes (north_star item 2: "the symbolic structure is reused across iterations and rebuilt only
when the pattern drifts"; regot_b200_set_pattern_reuse).  The reference rebuilds at every k % S == 0 (splr.h:352, 359-364),
so there is no oracle for the reusing trajectory: the bar is (i) drift_tol = 0 IS the reference's rule, bit for bit, (ii) a
reusing solve reaches the same optimum (f within 1e-9, marginal error under the tolerance, the oracle's objective), (iii)
it rebuilds less often and never keeps a pattern more than max_skips refreshes in a row, (iv) validation of the arguments."""
import numpy as np
import pytest

import paper_2605_08793_b200 as rg
from paper_2605_08793_b200 import problems

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]


@pytest.fixture()
def own():
    s = rg.Solver(0)
    yield s
    s.close()


def test_zero_tolerance_is_the_fixed_rule_bit_for_bit(own, solver):
    p = problems.gen_synthetic1(300, 260, "iid", 2, 5, 0.01)
    cfg = rg.SplrConfig(tol=1e-8)
    x0 = rg.DualPoint.zeros(p.n, p.m)
    solver.set_problem(p)
    ref = solver.run_splr(x0, cfg)
    own.set_pattern_reuse(0.0, 4)
    own.set_problem(p)
    r = own.run_splr(x0, cfg)
    assert [t.f for t in r.trace.rows] == [t.f for t in ref.trace.rows]
    assert np.array_equal(r.x.alpha, ref.x.alpha) and np.array_equal(r.x.beta, ref.x.beta)
    rebuilds, reuses = own.pattern_counts()
    assert reuses == 0 and rebuilds == sum(1 for s in r.steps if s.refresh)


@pytest.mark.parametrize("make", [
    lambda: problems.gen_synthetic1(400, 400, "iid", 2, 7, 0.01),
    lambda: problems.gen_synthetic2(256, 192, 0.005),
    lambda: problems.gen_image(24, 0.005),
])
def test_reusing_solves_reach_the_same_optimum_with_fewer_rebuilds(own, solver, oracle, make):
    p = make()
    cfg = rg.SplrConfig(tol=1e-8)
    x0 = rg.DualPoint.zeros(p.n, p.m)
    solver.set_problem(p)
    ref = solver.run_splr(x0, cfg)
    own.set_pattern_reuse(0.5, 3)
    own.set_problem(p)
    r = own.run_splr(x0, cfg)
    last, last0 = r.trace.rows[-1], ref.trace.rows[-1]
    assert last.marginal_error <= 1e-8
    assert abs(last.f - last0.f) <= 1e-9 * (1 + abs(last0.f))
    # the oracle's objective at the point reached: the values are the reference's whatever the path
    op = dict(n=p.n, m=p.m, M=np.asfortranarray(p.M), a=p.a, b=p.b, eta=p.eta)
    g = oracle.gradient(op, r.x.alpha, r.x.beta)
    assert abs(g["f"] - last.f) <= 1e-11 * (1 + abs(last.f))
    rebuilds, reuses = own.pattern_counts()
    refreshes = [s.iter for s in r.steps if s.refresh]
    assert rebuilds + reuses == len(refreshes)
    assert rebuilds >= 1 and rebuilds >= (len(refreshes) + 3) // 4  # never more than 3 kept refreshes in a row
    print(f"refreshes {len(refreshes)}: {rebuilds} rebuilds, {reuses} reuses; iterations {last.iter} (fixed rule {last0.iter})")
    assert last.iter <= int(1.5 * last0.iter) + cfg.S, (last.iter, last0.iter)


def test_a_pattern_is_kept_once_the_duals_have_settled(own):
    """A solve continued from its own solution: the duals do not move any more, so every refresh after the first keeps the
    pattern until max_skips forces a rebuild."""
    p = problems.gen_synthetic2(200, 160, 0.01)
    own.set_problem(p)
    x = own.run_splr(rg.DualPoint.zeros(p.n, p.m), rg.SplrConfig(tol=1e-9)).x
    own.set_pattern_reuse(0.05, 2)
    st = own.splr_init(x, rg.SplrConfig(tol=0.0, S=2))
    cfg = rg.SplrConfig(tol=0.0, S=2)
    r0 = own.pattern_counts()
    for _ in range(8):  # refreshes at k = 0, 2, 4, 6
        own.splr_step(st, cfg)
    rebuilds, reuses = (a - b for a, b in zip(own.pattern_counts(), r0))
    assert (rebuilds, reuses) == (2, 2), (rebuilds, reuses)  # build, keep, keep, rebuild (max_skips = 2)


def test_repeated_solve_is_deterministic(own):
    p = problems.gen_synthetic2(200, 160, 0.005)
    cfg = rg.SplrConfig(tol=1e-8)
    x0 = rg.DualPoint.zeros(p.n, p.m)
    own.set_pattern_reuse(0.5, 4)
    own.set_problem(p)
    a = own.run_splr(x0, cfg)
    b = own.run_splr(x0, cfg)
    assert [t.f for t in a.trace.rows] == [t.f for t in b.trace.rows]
    assert np.array_equal(a.x.beta, b.x.beta)


def test_arguments_are_validated(own):
    for tol, skips in ((-0.1, 4), (1.0, 4), (float("nan"), 4), (0.1, -1)):
        with pytest.raises(rg.ValidationError):
            own.set_pattern_reuse(tol, skips)
