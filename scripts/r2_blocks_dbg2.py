"""Debug helper: an indefinite matrix through the direction solve (must come back as NotPositiveDefinite)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08793_b200 as rg  # noqa: E402
from tests import oracle_lib  # noqa: E402

oracle = oracle_lib.load()
p = oracle.gen_problem("rand", 120, 100, 0.1, seed=5)
a0, b0 = oracle.rand_dual(120, 100, 0.2, 6)
coords = oracle.select_topk(oracle.plan(p, a0, b0), 3000)
x = rg.DualPoint(a0, b0)
s = rg.Solver(0)
s.set_problem(rg.ProblemInstance(p["n"], p["m"], np.ascontiguousarray(p["M"]), p["a"], p["b"], p["eta"]))
g = s.fused_gradient(x)
sc = float(os.environ.get("SCALE", "1e-3"))
fake = rg.GradientResult(g.f, g.grad, sc * g.row_sums, sc * g.col_sums, g.marginal_error, g.duality_gap, g.grad_norm2)
A = s.assemble(x, rg.SparsityPattern(120, 99, coords), 0.0, fake)
print("assembled", flush=True)
try:
    d, its = s.compute_direction(A, g.grad, cg_rtol=1e-12)
    print("returned", its, np.isfinite(d).all(), flush=True)
except Exception as e:  # noqa: BLE001
    print("raised", type(e).__name__, e, flush=True)
os._exit(0)
