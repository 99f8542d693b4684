"""Times the stand-alone mat-vec (K4) on a config-B pattern; prints the line-length distribution."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08793_b200 as rg
from paper_2605_08793_b200 import problems
p = problems.gen_image(100, 0.001)
s = rg.Solver(0)
s.set_problem(p)
x = rg.DualPoint.zeros(p.n, p.m)
for _ in range(20):
    x = s.sinkhorn_step(x)
g = s.fused_gradient(x)
A = s.assemble_topk(x, rg.topk_budget(p, 0.01), min(1.0, g.grad_norm2), g)
cp, ri, va, co = A.export()
rows = np.bincount(co[:, 0], minlength=p.n)
cols = np.bincount(co[:, 1], minlength=p.m - 1)
for nm, L in (("rows", rows), ("cols", cols)):
    print(nm, "nnz", L.sum(), "max", L.max(), "mean", L.mean(), "<=64:", (L <= 64).sum(), "65..512:", ((L > 64) & (L <= 512)).sum(), ">512:", (L > 512).sum(),
          "pct", np.percentile(L, [50, 90, 99, 99.9]))
v = np.random.default_rng(0).normal(size=p.n + p.m - 1)
for _ in range(5):
    A.matvec(v)
s.set_profiling(True)
for _ in range(30):
    A.matvec(v)
n, ms = s.get_profile(4)
print(f"spmv dbg={os.environ.get('REGOT_B200_SPMV_DBG', '0')}: {n} launches avg {1e3 * ms / n:.2f} us")
