"""Times the fused-gradient sweep kernel (K1) alone on a config-B-shaped problem.
Usage: python scripts/time_gradient.py [n] [m] [iters]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08793_b200 as rg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
rng = np.random.default_rng(0)
t0 = time.time()
M = rng.random((n, m))
M /= M.max()
a = np.full(n, 1.0 / n)
b = np.full(m, 1.0 / m)
eta = 0.05
s = rg.Solver(0)
s.set_problem(rg.ProblemInstance(n, m, M, a, b, eta))
print(f"setup {time.time() - t0:.1f}s", flush=True)
x = rg.DualPoint(rng.normal(size=n) * 0.01, np.append(rng.normal(size=m - 1) * 0.01, 0.0))
ms = s.time_kernel(0, x, iters)
byts = 8.0 * n * m + 16.0 * (n + m)
best, med = float(ms.min()), float(np.median(ms))
print(json.dumps({"n": n, "m": m, "ms_min": best, "ms_median": med, "GBps_median": byts / med * 1e-6,
                  "GBps_best": byts / best * 1e-6, "all_ms": [round(float(v), 4) for v in ms]}))
t0 = time.time()
g = s.fused_gradient(x)
print(f"full API gradient call {1e3 * (time.time() - t0):.2f} ms, f={g.f:.6g} err={g.marginal_error:.3e}")
