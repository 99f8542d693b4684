"""Are the first iterations of config D the same bits run to run and across prefetch distances of the ELL stream?"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08793_b200 as rg  # noqa: E402
from paper_2605_08793_b200 import problems  # noqa: E402

n = m = int(os.environ.get("N", "50000"))
X, Y = problems.gen_gmm_points(n, m, 10, 21)
a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
ref = None
for ahead in os.environ.get("AHEADS", "0 512 0 512 1024").split():
    os.environ["REGOT_B200_PANEL_AHEAD"] = ahead
    s = rg.Solver(0)
    s.set_pointcloud(X, Y, a, b, 0.001, on_the_fly=False)
    res = s.run_splr(rg.DualPoint.zeros(n, m), rg.SplrConfig(max_iter=int(os.environ.get("MAXIT", "14"))))
    sig = [(st.cg_iters, st.ls_evals, st.f_after) for st in res.steps]
    if ref is None:
        ref = sig
    first = next((i for i, (u, v) in enumerate(zip(ref, sig)) if u != v), None)
    print(f"ahead {ahead}: first difference at step {first}", sig[first] if first is not None else "", ref[first] if first is not None else "", flush=True)
    s.close()
