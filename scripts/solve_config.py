"""Solve one BASELINE config on the GPU and print where the time goes.
Usage: python scripts/solve_config.py A|B|C|D|Dsmall|<side> [overlap] [cg_rtol]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08793_b200 as rg  # noqa: E402
from paper_2605_08793_b200 import problems  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "B"
overlap = len(sys.argv) > 2 and sys.argv[2] == "1"
cg_rtol = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
t0 = time.time()
if which == "A":
    p = problems.gen_synthetic1(1000, 1000, "iid", 2, 7, 0.01)
elif which == "B":
    p = problems.gen_image(100, 0.001)
elif which == "C":
    p = problems.gen_synthetic2(20000, 5000, 0.0005)
elif which in ("D", "Dsmall"):
    # config D: Gaussian-mixture clouds in R^10, eta = 0.001; the 20 GB cost matrix is built in row chunks
    n = m = 50000 if which == "D" else 8000
    X, Y = problems.gen_gmm_points(n, m, 10, 21)
    M = np.empty((n, m))
    mx = 0.0
    for r0 in range(0, n, 2500):
        blk = problems.sqeuclid_cost(X[r0:r0 + 2500], Y)
        mx = max(mx, float(blk.max()))
        M[r0:r0 + 2500] = blk
    for r0 in range(0, n, 2500):
        M[r0:r0 + 2500] /= mx
    p = rg.ProblemInstance(n, m, M, np.full(n, 1.0 / n), np.full(m, 1.0 / m), 0.001)
elif ":" in which:  # kind:n:m:eta, e.g. synth1-iid:1600:1200:0.001 (d = 2, seed = 7)
    kind, n_, m_, eta_ = which.split(":")
    p = problems.make_problem(kind, int(n_), int(m_), float(eta_), 2, 7)
else:
    side = int(which)
    p = problems.gen_image(side, 0.001)
print(f"generated {which}: {p.n}x{p.m} eta={p.eta} in {time.time() - t0:.1f}s", flush=True)
s = rg.Solver(0)
t0 = time.time()
s.set_problem(p)
print(f"upload {time.time() - t0:.3f}s", flush=True)
cfg = rg.SplrConfig(overlap=overlap, cg_rtol=cg_rtol, max_iter=int(os.environ.get("MAXIT", "1000")))
for rep in range(2):
    s.set_profiling(rep == 1)
    t0 = time.time()
    try:
        res = s.run_splr(rg.DualPoint.zeros(p.n, p.m), cfg)
    except rg.RegotError as e:
        print("solve failed:", e)
        for k, nm in enumerate(["gradient", "row_lse", "col_lse", "topk", "spmv", "pcg"]):
            n, ms = s.get_profile(k)
            print(f"  {nm:9s} launches {n:6d} total {ms:9.2f} ms avg {ms / max(n, 1):.4f} ms")
        continue
    wall = time.time() - t0
    last = res.trace.rows[-1]
    print(json.dumps({"rep": rep, "wall_s": round(wall, 4), "device_ms": round(res.stats.device_ms, 2),
                      "iters": last.iter, "err": last.marginal_error, "f": last.f,
                      "grad_passes": res.stats.gradient_passes, "lse_passes": res.stats.lse_passes,
                      "launches": res.stats.kernel_launches,
                      "ls_evals": sum(x.ls_evals for x in res.steps), "cg_iters": sum(x.cg_iters for x in res.steps),
                      "ls_failed": sum(x.ls_failed for x in res.steps), "sink_sel": sum(x.sinkhorn_selected for x in res.steps),
                      "retries": sum(x.factor_retries for x in res.steps),
                      "pattern_rebuilds_reuses": s.pattern_counts()}), flush=True)
names = ["gradient", "row_lse", "col_lse", "topk", "spmv", "pcg", "refresh"]
for k, nm in enumerate(names):
    n, ms = s.get_profile(k)
    print(f"  {nm:9s} launches {n:6d} total {ms:9.2f} ms avg {ms / max(n, 1):.4f} ms")
for st in res.steps[:40]:
    print(f"   it {st.iter:3d} ref {int(st.refresh)} sk {int(st.sinkhorn_selected)} ls {st.ls_evals:2d} cg {st.cg_iters:5d} "
          f"gamma {st.gamma:8.3g} f {st.f_after:.10g} tau {st.tau:.3g} lr {int(st.lowrank_active)} fail {int(st.ls_failed)}")
print("trace errs:", [(r.iter, float(f"{r.marginal_error:.3g}")) for r in res.trace.rows[::10]])
sk = rg.SinkhornConfig(max_iter=200, record_every=50, tol=0.0)
t0 = time.time()
rk = s.run_sinkhorn(rg.DualPoint.zeros(p.n, p.m), sk)
print(f"sinkhorn 200 its: wall {time.time() - t0:.3f}s device {rk.stats.device_ms:.1f} ms err {rk.trace.rows[-1].marginal_error:.3e}")
