"""Time to marginal error 1e-8 of run_splr and run_sinkhorn at the paper's sizes, one B200.
The second solve of each is reported (the first one pays one-time allocations)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08793_b200 as rg  # noqa: E402
from paper_2605_08793_b200 import problems  # noqa: E402

s = rg.Solver(0)
print("| problem | SPLR: time to 1e-8 (iterations) | Sinkhorn: time to 1e-8 (iterations) |")
print("|---|---|---|")
for kind in ("synth1-iid", "synth2"):
    for n, m in ((1600, 1200), (3200, 2400), (6400, 4800)):
        p = problems.make_problem(kind, n, m, 0.001, 2, 7)
        s.set_problem(p)
        cells = []
        for algo in ("splr", "sinkhorn"):
            for rep in range(2):
                t0 = time.perf_counter()
                if algo == "splr":
                    res = s.run_splr(rg.DualPoint.zeros(n, m), rg.SplrConfig(max_iter=5000, tol=1e-8, record_every=5000))
                else:
                    res = s.run_sinkhorn(rg.DualPoint.zeros(n, m), rg.SinkhornConfig(max_iter=50000, tol=1e-8, record_every=50000))
                wall = 1e3 * (time.perf_counter() - t0)
            last = res.trace.rows[-1]
            ok = last.marginal_error <= 1e-8
            cells.append(f"{wall:.1f} ms ({last.iter})" if ok else f"not reached: {last.marginal_error:.1e} after {last.iter} its, {wall:.0f} ms")
        print(f"| {kind} {n}x{m}, eta=0.001 | {cells[0]} | {cells[1]} |", flush=True)
