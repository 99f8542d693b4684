import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08793_b200 as rg
from paper_2605_08793_b200 import problems
p = problems.gen_image(60, 0.001)
s = rg.Solver(0)
s.set_problem(p)
x = rg.DualPoint.zeros(p.n, p.m)
for _ in range(10):
    x = s.sinkhorn_step(x)
g = s.fused_gradient(x)
A = s.assemble_topk(x, rg.topk_budget(p, 0.01), min(1.0, g.grad_norm2), g)
rng = np.random.default_rng(0)
v = rng.normal(size=p.n + p.m - 1)
ys = [A.matvec(v) for _ in range(4)]
print("matvec identical:", all(np.array_equal(ys[0], y) for y in ys[1:]))
ds = [s.compute_direction(A, g.grad, cg_rtol=1e-8) for _ in range(4)]
print("direction(1 rhs) identical:", all(np.array_equal(ds[0][0], d[0]) for d in ds[1:]), [d[1] for d in ds])
sv = 0.01 * rng.normal(size=p.n + p.m - 1)
u = A.matvec(sv) + 0.3 * sv
w = A.matvec(sv)
xi, zeta = 1.0 / (u @ sv), -1.0 / (w @ sv)
ds = [s.compute_direction(A, g.grad, u, w, xi, zeta, cg_rtol=1e-8) for _ in range(4)]
print("direction(3 rhs) identical:", all(np.array_equal(ds[0][0], d[0]) for d in ds[1:]), [d[1] for d in ds],
      [float(np.abs(ds[0][0] - d[0]).max()) for d in ds[1:]])
gs = [s.fused_gradient(x) for _ in range(3)]
print("gradient identical:", all(np.array_equal(gs[0].grad, q.grad) and gs[0].f == q.f for q in gs[1:]))
xs = [s.sinkhorn_step(x) for _ in range(3)]
print("sinkhorn identical:", all(np.array_equal(xs[0].alpha, q.alpha) and np.array_equal(xs[0].beta, q.beta) for q in xs[1:]))
As = [s.assemble_topk(x, rg.topk_budget(p, 0.01), 0.1, g).export() for _ in range(3)]
print("assemble identical:", all(all(np.array_equal(a, b) for a, b in zip(As[0], q)) for q in As[1:]))
cfg = rg.SplrConfig(max_iter=25, tol=0.0)
rs = [s.run_splr(rg.DualPoint.zeros(p.n, p.m), cfg) for _ in range(3)]
print("splr 25 its f:", [r.trace.rows[-1].f for r in rs], [sum(t.cg_iters for t in r.steps) for r in rs])
for k in range(25):
    fs = [r.trace.rows[k + 1].f for r in rs]
    if len(set(fs)) > 1:
        print(" first divergence at iter", k + 1, fs, [r.steps[k].cg_iters for r in rs], [r.steps[k].gamma for r in rs])
        break
