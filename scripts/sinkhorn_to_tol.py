"""run_sinkhorn to marginal error 1e-8 on a BASELINE config (default B), for the comparison with run_splr.
Usage: python scripts/sinkhorn_to_tol.py [A|B] [max_iter]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08793_b200 as rg  # noqa: E402
from paper_2605_08793_b200 import problems  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "B"
max_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 30000
p = problems.gen_image(100, 0.001) if which == "B" else problems.gen_synthetic1(1000, 1000, "iid", 2, 7, 0.01)
s = rg.Solver(0)
s.set_problem(p)
t0 = time.perf_counter()
res = s.run_sinkhorn(rg.DualPoint.zeros(p.n, p.m), rg.SinkhornConfig(max_iter=max_iter, tol=1e-8, record_every=1000))
wall = time.perf_counter() - t0
last = res.trace.rows[-1]
print(f"config {which}: run_sinkhorn stopped at iteration {last.iter} with marginal error {last.marginal_error:.3e} after {wall:.3f} s "
      f"(device {res.stats.device_ms:.1f} ms)")
print("errors every 1000 iterations:", [f"{r.marginal_error:.2e}" for r in res.trace.rows])
