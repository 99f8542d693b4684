"""Times the three sweep kernels (K1 gradient, K7 row LSE, K8 column LSE) alone on config B at two dual
points: the cold start x0 = 0 and a point after 30 Sinkhorn steps.  Usage: python scripts/time_sweeps.py [side]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08793_b200 as rg  # noqa: E402
from paper_2605_08793_b200 import problems  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 100
p = problems.gen_image(side, 0.001)
s = rg.Solver(0)
s.set_problem(p)
byts = 8.0 * p.n * p.m + 16.0 * (p.n + p.m)
x = rg.DualPoint.zeros(p.n, p.m)
for tag in ("x0", "after30"):
    if tag == "after30":
        for _ in range(30):
            x = s.sinkhorn_step(x)
    for which, nm in ((0, "K1 gradient"), (1, "K7 row lse"), (2, "K8 col lse")):
        ms = s.time_kernel(which, x, 20)[3:]
        med = float(np.median(ms))
        print(json.dumps({"point": tag, "kernel": nm, "ms_median": round(med, 5), "ms_min": round(float(ms.min()), 5),
                          "GBps_median": round(byts / med * 1e-6, 1), "frac_of_6447.8": round(byts / med * 1e-6 / 6447.8, 4)}),
              flush=True)
