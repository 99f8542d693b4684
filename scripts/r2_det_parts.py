"""Config D, one iterate: is every stage the same bits when repeated?  gradient | top-k pattern + values | direction."""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08793_b200 as rg  # noqa: E402
from paper_2605_08793_b200 import problems  # noqa: E402

n = m = int(os.environ.get("N", "50000"))
X, Y = problems.gen_gmm_points(n, m, 10, 21)
a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
s = rg.Solver(0)
s.set_pointcloud(X, Y, a, b, 0.001, on_the_fly=False)
res = s.run_splr(rg.DualPoint.zeros(n, m), rg.SplrConfig(max_iter=int(os.environ.get("WARM", "25"))))
x = res.x
k = int(os.environ.get("K", str(int(0.01 * n * m))))


def h(*arrs):
    d = hashlib.sha1()
    for v in arrs:
        d.update(np.ascontiguousarray(v).tobytes())
    return d.hexdigest()[:12]


seen = {}
for rep in range(int(os.environ.get("REPS", "30"))):
    g = s.fused_gradient(x)
    hg = h(g.grad, g.row_sums, g.col_sums, np.array([g.f]))
    A = s.assemble_topk(x, k, min(1.0, g.grad_norm2), g)
    coords, vals = A.export_local()
    hp, hv = h(coords), h(vals)
    d, its = s.compute_direction(A, g.grad)
    hd = h(d)
    key = (hg, hp, hv, hd, its)
    seen[key] = seen.get(key, 0) + 1
    if len(seen) > 1 or rep == 0:
        print(rep, key, "nnz", len(vals), flush=True)
    A.free()
print("distinct outcomes:", len(seen), list(seen.values()))
