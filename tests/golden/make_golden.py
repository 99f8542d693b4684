"""Generates tests/golden/oracle_golden.json from the CPU oracle (run once in the authoring
container, after oracle/selfcheck passed against the reference's own known-answer tests)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2605_08793_b200._lib import SinkhornConfigC, SplrConfigC  # noqa: E402
from tests import oracle_lib  # noqa: E402

o = oracle_lib.load()
G = {"gradient": [], "sinkhorn": [], "splr": [], "topk": []}
for kind, n, m, eta, d, seed in [("rand", 33, 128, 0.1, 2, 303), ("synth2", 96, 80, 0.001, 2, 0),
                                 ("synth1-iid", 64, 64, 0.01, 2, 7), ("image", 144, 144, 0.001, 12, 0),
                                 ("gmm", 50, 40, 0.001, 10, 21), ("uniform", 50, 40, 0.01, 3, 31)]:
    p = o.gen_problem(kind, n, m, eta, d=d, seed=seed)
    al, be = o.rand_dual(n, m, 0.05, 99)
    g = o.gradient(p, al, be)
    G["gradient"].append(dict(kind=kind, n=n, m=m, eta=eta, d=d, seed=seed, scale=0.05, dual_seed=99, f=float(g["f"]).hex(),
                              marginal_error=float(g["marginal_error"]).hex(), row_head=[float(v).hex() for v in g["row"][:4]],
                              col_head=[float(v).hex() for v in g["col"][:4]]))
for kind, n, m, eta, d, seed, it in [("synth2", 24, 24, 0.01, 2, 0, 40), ("rand", 30, 20, 0.05, 2, 5, 25)]:
    p = o.gen_problem(kind, n, m, eta, d=d, seed=seed)
    r = o.run_sinkhorn(p, np.zeros(n), np.zeros(m), SinkhornConfigC(it, it, 0.0))
    G["sinkhorn"].append(dict(kind=kind, n=n, m=m, eta=eta, d=d, seed=seed, max_iter=it, final_err=float(r["trace"][-1][3]).hex()))
for kind, n, m, eta, d, seed, it in [("synth2", 64, 64, 0.01, 2, 0, 200), ("synth1-diff", 64, 64, 0.01, 2, 7, 200)]:
    p = o.gen_problem(kind, n, m, eta, d=d, seed=seed)
    c = SplrConfigC(1.0, 10, 5, 0.01, 1e-4, 0.9, it, 1e-8, 30, 1, 0, 8, 32, 0, 0.0)
    r = o.run_splr(p, np.zeros(n), np.zeros(m), c)
    G["splr"].append(dict(kind=kind, n=n, m=m, eta=eta, d=d, seed=seed, max_iter=it, iters=r["trace"][-1][0],
                          f_head=[float(t[2]).hex() for t in r["trace"][:5]]))
for seed, n, m, k in [(1, 40, 33, 200), (2, 63, 17, 500), (3, 9, 64, 10)]:
    rng = np.random.default_rng(seed)
    T = np.where(rng.random((n, m)) < 0.3, 0.5, rng.random((n, m)))
    c = o.select_topk(T, k)
    G["topk"].append(dict(seed=seed, n=n, m=m, k=k, count=len(c), checksum=int(np.sum(c[:, 0] * 1315423911 + c[:, 1]) % (2**61 - 1))))
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle_golden.json"), "w") as f:
    json.dump(G, f, indent=1)
print("wrote oracle_golden.json")
