"""synth2 1600 x 1200 (eta = 0.001): CG iterations and the split of the solve with the Schur-diagonal preconditioner on / off."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08793_b200 as rg  # noqa: E402
from paper_2605_08793_b200 import problems  # noqa: E402

p = problems.gen_synthetic2(1600, 1200, 0.001)
for sd in ("1", "0"):
    os.environ["REGOT_B200_SCHUR_DIAG"] = sd
    s = rg.Solver(0)
    s.set_problem(p)
    x0 = rg.DualPoint.zeros(p.n, p.m)
    for rep in range(2):
        s.set_profiling(False)
        s.set_profiling(True)
        res = s.run_splr(x0, rg.SplrConfig(max_iter=1000))
    st = res.steps
    print(f"schur_diag={sd}: {res.stats.device_ms:.1f} ms, iterations {res.trace.rows[-1].iter}, cg {sum(q.cg_iters for q in st)}, evals {sum(q.ls_evals for q in st)},"
          f" failed {sum(q.ls_failed for q in st)}, sinkhorn selected {sum(q.sinkhorn_selected for q in st)}")
    for kind, name in enumerate(("gradient", "row_lse", "col_lse", "topk", "spmv", "pcg", "refresh")):
        n, ms = s.get_profile(kind)
        if n:
            print(f"   {name:9s} {n:5d} launches {ms:8.2f} ms avg {ms / n:.4f}")
    s.close()
