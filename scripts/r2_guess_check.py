"""Config D: the pattern of a refresh that starts from the previous refresh's threshold bin against the three-sweep path."""
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
k = int(np.ceil(0.01 * n * (m - 1)))


def h(v):
    return hashlib.sha1(np.ascontiguousarray(v).tobytes()).hexdigest()[:12]


x10 = None
for guess in ("1", "0"):
    os.environ["REGOT_B200_TOPK_GUESS"] = guess
    s = rg.Solver(0)
    s.set_pointcloud(X, Y, a, b, 0.001, on_the_fly=False)
    if x10 is None:
        x10 = s.run_splr(rg.DualPoint.zeros(n, m), rg.SplrConfig(max_iter=int(os.environ.get("WARM", "10")))).x
        s.close()
        s = rg.Solver(0)
        s.set_pointcloud(X, Y, a, b, 0.001, on_the_fly=False)
    x0 = rg.DualPoint.zeros(n, m)
    s.assemble_topk(x0, k, 1.0).free()
    A = s.assemble_topk(x10, k, 1.0)
    coords, vals = A.export_local()
    print(f"guess={guess}: nnz {len(vals)} coords {h(coords)} values {h(vals)}", flush=True)
    if guess == "1":
        keep = coords.copy()
    else:
        same = len(coords) == len(keep) and np.array_equal(coords, keep)
        print("patterns equal:", same)
        if not same:
            sa = set(map(tuple, keep.tolist())); sb = set(map(tuple, coords.tolist()))
            print("only with guess:", len(sa - sb), "only without:", len(sb - sa), list(sa - sb)[:5], list(sb - sa)[:5])
    s.close()
