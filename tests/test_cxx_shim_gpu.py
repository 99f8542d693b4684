"""GPU: the header-only C++ shim (include/regot_b200.hpp -- regot::run_splr-shaped wrappers and the reference's
exception classes over the C ABI) executes on the device and agrees with the ctypes mirror bit for bit: same
library, same calls.  The program reads a problem written by this test (raw doubles), runs fused_gradient,
sinkhorn_step, run_sinkhorn and run_splr through the shim's free functions, checks the gauge validation throws the
reference's exception class, and prints %.17g numbers."""
import os
import subprocess
import tempfile

import numpy as np
import pytest

import paper_2605_08793_b200 as rg
from paper_2605_08793_b200 import _lib, problems

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROG = r'''
#include "regot_b200.hpp"
#include <cstdio>
#include <fstream>
#include <vector>
namespace rb = regot_b200;
static std::vector<double> slurp(const char* path, size_t n) {
  std::vector<double> v(n);
  std::ifstream f(path, std::ios::binary);
  f.read(reinterpret_cast<char*>(v.data()), (std::streamsize)(8 * n));
  if (!f) throw std::runtime_error("short read");
  return v;
}
int main(int argc, char** argv) {
  const long n = std::atol(argv[1]), m = std::atol(argv[2]);
  rb::ProblemInstance p;
  p.n = n; p.m = m; p.layout = REGOT_LAYOUT_ROWMAJOR; p.eta = std::atof(argv[3]);
  p.M = slurp(argv[4], (size_t)(n * m)); p.a = slurp(argv[5], (size_t)n); p.b = slurp(argv[6], (size_t)m);
  rb::DualPoint x0 = rb::DualPoint::zeros(n, m);
  // free functions with the reference's signatures
  rb::GradientResult g = rb::fused_gradient(x0, p);
  std::printf("grad %.17g %.17g %.17g\n", g.f, g.marginal_error, g.row_sums[0]);
  rb::DualPoint x1 = rb::sinkhorn_step(x0, p);
  std::printf("sink %.17g %.17g\n", x1.alpha[0], x1.beta[0]);
  rb::SinkhornConfig sk; sk.max_iter = 50; sk.tol = 0.0; sk.record_every = 10;
  rb::SinkhornResult rs = rb::run_sinkhorn(x0, p, sk);
  std::printf("run_sinkhorn %zu %.17g %.17g\n", rs.trace.rows.size(), rs.trace.rows.back().f, rs.trace.rows.back().marginal_error);
  rb::SplrConfig cfg; cfg.max_iter = 200; cfg.tol = 1e-8;
  rb::SplrResult r = rb::run_splr(x0, p, cfg);
  std::printf("run_splr %ld %.17g %.17g %zu\n", r.trace.rows.back().iter, r.trace.rows.back().f, r.trace.rows.back().marginal_error, r.steps.size());
  for (size_t k = 0; k < r.steps.size() && k < 5; ++k) std::printf("step %.17g %d %d\n", r.steps[k].f_after, r.steps[k].ls_evals, r.steps[k].cg_iters);
  // validation: the gauge must hold exactly (dual.h:72-78) -> the reference's exception class
  rb::DualPoint bad = x0; bad.beta[(size_t)m - 1] = 1e-300;
  try { rb::fused_gradient(bad, p); std::printf("gauge accepted\n"); return 3; }
  catch (const rb::ValidationError& e) { std::printf("gauge ValidationError\n"); }
  return 0;
}
'''


def test_cxx_shim_runs_on_the_device_and_matches_the_python_mirror(solver):
    p = problems.gen_synthetic2(96, 80, 0.01)
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "shim.cpp"), os.path.join(d, "shim")
        open(src, "w").write(PROG)
        libdir = os.path.dirname(_lib.LIB_PATH)
        subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"), "-o", exe, src, "-L", libdir,
                        "-lregot_b200", f"-Wl,-rpath,{libdir}", "-L/usr/local/cuda/lib64", "-Wl,-rpath,/usr/local/cuda/lib64"], check=True)
        files = []
        for name, arr in (("M", np.ascontiguousarray(p.M)), ("a", p.a), ("b", p.b)):
            path = os.path.join(d, name + ".bin")
            np.asarray(arr, dtype=np.float64).tofile(path)
            files.append(path)
        out = subprocess.run([exe, str(p.n), str(p.m), repr(p.eta), *files], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    lines = {ln.split()[0]: ln.split()[1:] for ln in out.stdout.splitlines() if not ln.startswith("step")}
    steps = [ln.split()[1:] for ln in out.stdout.splitlines() if ln.startswith("step")]
    assert lines["gauge"] == ["ValidationError"]

    solver.set_problem(p)
    x0 = rg.DualPoint.zeros(p.n, p.m)
    g = solver.fused_gradient(x0)
    assert [float(v) for v in lines["grad"]] == [g.f, g.marginal_error, float(g.row_sums[0])]
    x1 = solver.sinkhorn_step(x0)
    assert [float(v) for v in lines["sink"]] == [float(x1.alpha[0]), float(x1.beta[0])]
    rs = solver.run_sinkhorn(x0, rg.SinkhornConfig(max_iter=50, tol=0.0, record_every=10))
    assert int(lines["run_sinkhorn"][0]) == len(rs.trace.rows)
    assert [float(v) for v in lines["run_sinkhorn"][1:]] == [rs.trace.rows[-1].f, rs.trace.rows[-1].marginal_error]
    r = solver.run_splr(x0, rg.SplrConfig(max_iter=200, tol=1e-8))
    last = r.trace.rows[-1]
    assert int(lines["run_splr"][0]) == last.iter and int(lines["run_splr"][3]) == len(r.steps)
    assert [float(v) for v in lines["run_splr"][1:3]] == [last.f, last.marginal_error]
    for got, st in zip(steps, r.steps):
        assert float(got[0]) == st.f_after and int(got[1]) == st.ls_evals and int(got[2]) == st.cg_iters
