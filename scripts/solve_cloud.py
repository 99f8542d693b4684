"""Solve a point-cloud BASELINE config on one GPU through regot_b200_set_pointcloud and print where the
time goes.  Usage: python scripts/solve_cloud.py E|D|A [fly=1|0] [n]
  E: uniform clouds in R^3, eta = 0.01, n = m = 100,000, cost formed on the fly (never stored)
  D: Gaussian-mixture clouds in R^10, eta = 0.001, n = m = 50,000 (20 GB materialised on the device)
  A: gen_synthetic1 clouds in R^2 (seed 7), eta = 0.01, n = m = 1000"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08793_b200 as rg  # noqa: E402
from paper_2605_08793_b200 import problems  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "E"
fly = (sys.argv[2] == "1") if len(sys.argv) > 2 else (which == "E")
t0 = time.time()
if which == "E":
    n = m = int(sys.argv[3]) if len(sys.argv) > 3 else 100000
    X, Y = problems.gen_uniform_points(n, m, 3, 31)
    eta = 0.01
elif which == "D":
    n = m = int(sys.argv[3]) if len(sys.argv) > 3 else 50000
    X, Y = problems.gen_gmm_points(n, m, 10, 21)
    eta = 0.001
else:
    n = m = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
    rng = problems.Rng(7)
    X = np.array([rng.normal() for _ in range(n * 2)]).reshape(n, 2)
    Y = np.array([rng.normal() for _ in range(m * 2)]).reshape(m, 2)
    eta = 0.01
a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
print(f"clouds {which}: n={n} m={m} d={X.shape[1]} eta={eta} on_the_fly={fly} generated in {time.time() - t0:.1f}s", flush=True)
s = rg.Solver(0)
t0 = time.time()
s.set_pointcloud(X, Y, a, b, eta, on_the_fly=fly)
print(f"set_pointcloud {time.time() - t0:.3f}s", flush=True)
x0 = rg.DualPoint.zeros(n, m)
ms = s.time_kernel(0, x0, 5)
alg = 8.0 * n * m
print(f"K1 fused gradient pass: median {np.median(ms):.3f} ms = {n * m / np.median(ms) * 1e-6:.1f} G entries/s"
      f" ({alg / np.median(ms) * 1e-6:.0f} GB/s of materialised-equivalent traffic)", flush=True)
for k, nm in ((1, "K7 row lse"), (2, "K8 col lse")):
    ms = s.time_kernel(k, x0, 5)
    print(f"{nm}: median {np.median(ms):.3f} ms", flush=True)
cfg = rg.SplrConfig(max_iter=int(os.environ.get("MAXIT", "1000")))
for rep in range(int(os.environ.get("REPS", "1"))):  # REPS=2: the second solve excludes first-use costs
    s.set_profiling(False)
    s.set_profiling(True)
    t0 = time.time()
    res = s.run_splr(x0, cfg)
    wall = time.time() - t0
last = res.trace.rows[-1]
print(json.dumps({"wall_s": round(wall, 3), "device_ms": round(res.stats.device_ms, 1), "iters": last.iter,
                  "err": last.marginal_error, "f": last.f, "grad_passes": res.stats.gradient_passes,
                  "lse_passes": res.stats.lse_passes, "ls_evals": sum(x.ls_evals for x in res.steps),
                  "cg_iters": sum(x.cg_iters for x in res.steps), "ls_failed": sum(x.ls_failed for x in res.steps),
                  "sink_sel": sum(x.sinkhorn_selected for x in res.steps),
                  "pattern_rebuilds_reuses": s.pattern_counts()}), flush=True)
for k, nm in enumerate(["gradient", "row_lse", "col_lse", "topk", "spmv", "pcg"]):
    cnt, tot = s.get_profile(k)
    print(f"  {nm:9s} launches {cnt:6d} total {tot:10.2f} ms avg {tot / max(cnt, 1):.4f} ms")
print("trace errs:", [(r.iter, float(f"{r.marginal_error:.3g}")) for r in res.trace.rows[::10]])
