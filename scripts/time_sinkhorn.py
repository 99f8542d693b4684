"""run_sinkhorn on config B (n = m = 10,000, eta = 0.001): device time per iteration with the stopping test
evaluated every iteration (tol > 0: Sinkhorn update + gradient pass), for the gradient-sweep form of the
update (default) and the log-sum-exp kernels (REGOT_B200_EXACT_LSE=1).  Usage: python scripts/time_sinkhorn.py"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1:
    import paper_2605_08793_b200 as rg
    from paper_2605_08793_b200 import problems

    p = problems.gen_image(100, 0.001)
    s = rg.Solver(0)
    s.set_problem(p)
    cfg = rg.SinkhornConfig(max_iter=200, tol=1e-300, record_every=200)
    for rep in range(2):
        res = s.run_sinkhorn(rg.DualPoint.zeros(p.n, p.m), cfg)
    last = res.trace.rows[-1]
    print(f"{sys.argv[1]}: {res.stats.device_ms:.2f} ms for {last.iter} iterations = {res.stats.device_ms / last.iter:.4f} ms/iteration, "
          f"err {last.marginal_error:.6e}, f {last.f:.15g}")
else:
    for name, env in (("sweep form", {}), ("log-sum-exp", {"REGOT_B200_EXACT_LSE": "1"})):
        subprocess.run([sys.executable, __file__, name], env={**os.environ, **env}, check=True)
