import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2605_08793_b200 as rg
from paper_2605_08793_b200 import problems
p = problems.gen_synthetic2(96, 80, 0.01)
cfg = rg.SplrConfig(max_iter=200, tol=1e-8)
s1 = rg.Solver(0)
os.environ["REGOT_B200_MULTIKERNEL_PCG"] = "1"
s2 = rg.Solver(0)
res = []
for s in (s1, s2):
    s.set_problem(p)
    res.append(s.run_splr(rg.DualPoint.zeros(p.n, p.m), cfg))
for a, b in zip(res[0].steps[:60], res[1].steps[:60]):
    flag = "" if (a.f_after == b.f_after) else ("  <-- differs %.3e" % abs(a.f_after - b.f_after))
    print(f"it {a.iter:3d} ls {a.ls_evals}/{b.ls_evals} cg {a.cg_iters}/{b.cg_iters} gamma {a.gamma:.4g}/{b.gamma:.4g} lr {a.lowrank_active}/{b.lowrank_active} sk {a.sinkhorn_selected}/{b.sinkhorn_selected} f {a.f_after:.15g} {b.f_after:.15g}{flag}")
