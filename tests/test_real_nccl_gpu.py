"""GPU: the sharded path through the REAL libnccl on one GPU.  One rank, a one-rank communicator pair made from
ncclGetUniqueId / ncclCommInitRank, and REGOT_B200_SHARDED_SINGLE=1 so the context takes the row-block upload and
issues every collective (ncclAllReduce double sum / max, u64 sum; main and side communicators) instead of skipping
them as an unsharded context does.  The loopback tests (test_sharded_loopback_gpu.py) cover R > 1 ranks with a
stand-in library; this one covers the actual NCCL entry points, enums and stream usage.  It runs in a child
process: the function table is resolved once per process and the loopback tests point it elsewhere."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, sys
import numpy as np
import paper_2605_08793_b200 as rg
from paper_2605_08793_b200 import problems

def summary(s, p, x0, overlap):
    g = s.fused_gradient(x0)
    sk = s.sinkhorn_step(x0)
    rs = s.run_sinkhorn(x0, rg.SinkhornConfig(max_iter=40, tol=0.0, record_every=10))
    r = s.run_splr(x0, rg.SplrConfig(max_iter=200, tol=1e-8, overlap=overlap))
    last = r.trace.rows[-1]
    return {"f": g.f, "err": g.marginal_error, "cols": g.col_sums.tolist(), "rows": g.row_sums.tolist(),
            "sk_beta": sk.beta.tolist(), "sk_alpha": sk.alpha.tolist(), "rs_f": rs.trace.rows[-1].f,
            "its": last.iter, "splr_f": last.f, "splr_err": last.marginal_error,
            "steps": [[st.f_after, st.cg_iters, st.ls_evals] for st in r.steps]}

out = {}
for name, p in (("synth1", problems.gen_synthetic1(192, 160, "iid", 2, 7, 0.01)), ("synth2", problems.gen_synthetic2(128, 112, 0.01))):
    x0 = rg.DualPoint.zeros(p.n, p.m)
    plain = rg.Solver(0)
    plain.set_problem(p)
    sh = rg.Solver(0)
    ids = rg.Solver.comm_unique_id()
    sh.comm_init(0, 1, ids)
    sh.set_problem(p, rows=(0, p.n))
    out[name] = {"plain": summary(plain, p, x0, False), "sharded": summary(sh, p, x0, False), "sharded_overlap": summary(sh, p, x0, True)}
    sh.close(); plain.close()
print("RESULT " + json.dumps(out))
'''


def test_sharded_path_over_real_nccl_with_one_rank():
    env = dict(os.environ)
    env.pop("REGOT_B200_NCCL_LIB", None)
    env["REGOT_B200_SHARDED_SINGLE"] = "1"
    env["NCCL_DEBUG"] = "VERSION"  # the real library announces itself when a communicator is made
    env["PYTHONPATH"] = ROOT + os.pathsep + env.get("PYTHONPATH", "")
    out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=500, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    assert "NCCL version" in out.stdout + out.stderr, "the real libnccl was not the one initialised"
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("RESULT ")][-1]
    res = json.loads(line[len("RESULT "):])
    for name, r in res.items():
        a = r["plain"]
        for form in ("sharded", "sharded_overlap"):
            b = r[form]
            # one rank: the row side is the same arithmetic; the column side goes through the allreduced pack
            assert np.array_equal(a["rows"], b["rows"]), (name, form)
            np.testing.assert_allclose(b["cols"], a["cols"], rtol=1e-12)
            assert abs(a["f"] - b["f"]) <= 1e-12 * (1 + abs(a["f"])), (name, form)
            np.testing.assert_allclose(b["sk_beta"], a["sk_beta"], rtol=0, atol=1e-12)
            np.testing.assert_allclose(b["sk_alpha"], a["sk_alpha"], rtol=0, atol=1e-12)
            assert abs(a["rs_f"] - b["rs_f"]) <= 1e-11 * (1 + abs(a["rs_f"])), (name, form)
            # whole solves: converged, same objective, same count within the parity band (north_star: +-5 %, here +-2)
            assert b["splr_err"] <= 1e-8, (name, form)
            assert abs(a["splr_f"] - b["splr_f"]) <= 1e-9 * (1 + abs(a["splr_f"])), (name, form)
            assert abs(a["its"] - b["its"]) <= 2, (name, form, a["its"], b["its"])
            for u, v in zip(a["steps"][:8], b["steps"][:8]):
                assert abs(u[0] - v[0]) <= 1e-10 * (1 + abs(u[0])), (name, form)
