"""Marginal error and objective of the last iterations of run_splr (synthetic II, 96 x 80, eta = 0.01) next to the CPU
oracle: where the objective is flat to its last bits the crossing of the tolerance is decided by rounding noise.
Usage: python scripts/trajectory_tail.py"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2605_08793_b200 as rg
from paper_2605_08793_b200 import problems
from tests import oracle_lib
oracle = oracle_lib.load()
p = problems.gen_synthetic2(96, 80, 0.01)
op = dict(n=p.n, m=p.m, M=np.asfortranarray(p.M), a=p.a, b=p.b, eta=p.eta)
s = rg.Solver(0); s.set_problem(p)
cfg = rg.SplrConfig(max_iter=200, tol=1e-8)
res = s.run_splr(rg.DualPoint.zeros(p.n, p.m), cfg)
oref = oracle.run_splr(op, np.zeros(p.n), np.zeros(p.m), cfg._c())
g = {r.iter: r for r in res.trace.rows}
o = {r[0]: r for r in oref["trace"]}
for it in range(36, 52):
    a = g.get(it); b = o.get(it)
    print(it, ("%.6e %.15g" % (a.marginal_error, a.f)) if a else "-", "|", ("%.6e %.15g" % (b[3], b[2])) if b else "-")
