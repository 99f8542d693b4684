"""Debug helper: one direction solve through the block-resident PCG kernel on a small random pattern; prints errors in full.
Usage: python scripts/r2_blocks_dbg.py n m k"""
import os
import sys
import traceback

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08793_b200 as rg  # noqa: E402
from paper_2605_08793_b200 import problems  # noqa: E402

n, m = int(sys.argv[1]), int(sys.argv[2])
p = problems.gen_synthetic1(n, m, "iid", 2, 7, 0.01)
s = rg.Solver(0)
s.set_problem(p)
x = rg.DualPoint.zeros(p.n, p.m)
for _ in range(3):
    x = s.sinkhorn_step(x)
g = s.fused_gradient(x)
A = s.assemble_topk(x, rg.topk_budget(p, 0.01), min(1.0, g.grad_norm2), g)
try:
    d, its = s.compute_direction(A, g.grad, cg_rtol=1e-10)
    r = A.matvec(d) + g.grad
    print("ok: iterations", its, "relative residual", np.linalg.norm(r) / np.linalg.norm(g.grad), flush=True)
except Exception as e:  # noqa: BLE001
    print("FAILED:", repr(e), flush=True)
    traceback.print_exc()
