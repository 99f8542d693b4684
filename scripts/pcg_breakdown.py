"""Time of the direction solve (pattern of config B, or of PROBLEM=kind:n:m:eta, after 20 Sinkhorn steps): the persistent Schur-complement
PCG kernel to convergence and for a fixed 1000 iterations (REGOT_B200_PCG_FIXED_ITERS), and the former
full-system kernel (REGOT_B200_PCG_FULL=1 in the environment) for comparison.
Usage: python scripts/pcg_breakdown.py [nrhs=3]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08793_b200 as rg  # noqa: E402
from paper_2605_08793_b200 import problems  # noqa: E402

nrhs = int(sys.argv[1]) if len(sys.argv) > 1 else 3
spec = os.environ.get("PROBLEM", "")  # kind:n:m:eta (d = 2, seed = 7); default: config B
if spec:
    kind, n_, m_, eta_ = spec.split(":")
    p = problems.make_problem(kind, int(n_), int(m_), float(eta_), 2, 7)
else:
    p = problems.gen_image(100, 0.001)
s = rg.Solver(0)
s.set_problem(p)
x = rg.DualPoint.zeros(p.n, p.m)
for _ in range(20):
    x = s.sinkhorn_step(x)
g = s.fused_gradient(x)
A = s.assemble_topk(x, rg.topk_budget(p, 0.01), min(1.0, g.grad_norm2), g)
rng = np.random.default_rng(0)
dim = p.n + p.m - 1
u = rng.normal(size=dim) if nrhs == 3 else None
v = rng.normal(size=dim) if nrhs == 3 else None
for fixed in (0, 1000):
    if fixed:
        os.environ["REGOT_B200_PCG_FIXED_ITERS"] = str(fixed)
    best = 1e9
    for rep in range(3):
        s.set_profiling(True)
        try:
            d, its = s.compute_direction(A, g.grad, u, v, 1.0, -1.0, cg_rtol=1e-10)
        except rg.RegotError:
            its = -1  # fixed-iteration runs go past convergence; only the kernel time matters
        n, ms = s.get_profile(5)
        s.set_profiling(False)
        best = min(best, ms / max(n, 1))
    iters = fixed if fixed else its
    print(f"fixed={fixed} nrhs={nrhs}: kernel {best:.3f} ms, {iters} iterations -> {1e3 * best / max(iters, 1):.2f} us/iteration", flush=True)
