"""Writes the I/O golden fixtures with the REFERENCE's own writers (oracle/_ref: save_problem
problem.h:221-241, emit_csv bench.h:243-256).  Run once in the authoring container (needs
/root/reference for `make -C oracle ref`); the fixtures are committed so the GPU box needs neither."""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from paper_2605_08793_b200._lib import TraceRowC  # noqa: E402
from tests import oracle_lib  # noqa: E402

ref = oracle_lib.load_ref()
assert ref is not None, "build oracle/_ref first (make -C oracle ref)"
lib = ref.lib
dp = C.POINTER(C.c_double)
p = ref.gen_problem("synth1-diff", 6, 5, 0.0125, d=3, seed=42)
M = np.asfortranarray(p["M"])
path = os.path.join(HERE, "ref_synth1diff_6x5.rotb")
st = lib.rgo_save_problem(path.encode(), C.c_long(6), C.c_long(5), M.ctypes.data_as(dp), p["a"].ctypes.data_as(dp),
                          p["b"].ctypes.data_as(dp), C.c_double(p["eta"]))
assert st == 0
rows = (TraceRowC * 4)()
vals = [(0, 0.0, 1.6638586759335181, 1.25, -0.5), (1, 0.1, 0.29051373543167602, 1e-3, 1e-300),
        (7, 123.456789012345678, -0.06647132208369197, 7.190629985496689e-09, -2.5e-17),
        (1000, 1e6, float(np.nextafter(1.0, 2.0)), 5e-324, float("inf"))]
for r, v in zip(rows, vals):
    r.iter, r.wall_ms, r.f, r.marginal_error, r.duality_gap = v
st = lib.rgo_emit_trace_csv(os.path.join(HERE, "ref_trace.csv").encode(), C.c_long(4), rows)
assert st == 0
print("wrote", path, os.path.getsize(path), "bytes and ref_trace.csv")
