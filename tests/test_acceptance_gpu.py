"""GPU: the reference's acceptance criteria that judge whole solves (tests/acceptance.cpp), run on the device
solver: (8) the linear-rate envelope against a high-accuracy reference run (acceptance.cpp:345-371) and (11)
benchmark-harness fidelity at 256 x 256, eta = 0.001 -- SPLR's error at checkpoint 200 below Sinkhorn's
(acceptance.cpp:421-472).  Criteria 5-7 and 10 live in test_splr_gpu.py."""
import numpy as np
import pytest

import paper_2605_08793_b200 as rg
from paper_2605_08793_b200 import io

pytestmark = pytest.mark.gpu


def to_problem(p):
    return rg.ProblemInstance(p["n"], p["m"], p["M"], p["a"], p["b"], p["eta"])


@pytest.mark.parametrize("kind", ["synth1-iid", "synth1-diff", "synth2"])
def test_criterion_8_linear_rate_envelope(solver, oracle, kind):
    # ConvergenceRuns (acceptance.cpp:72-96): 64 x 64, eta = 0.01, seed 7, defaults with max_iter 200, tol 1e-8
    p = to_problem(oracle.gen_problem(kind, 64, 64, 0.01, d=2, seed=7))
    solver.set_problem(p)
    x0 = rg.DualPoint.zeros(64, 64)
    run = solver.run_splr(x0, rg.SplrConfig(max_iter=200, tol=1e-8, record_every=1))
    ref = solver.run_splr(x0, rg.SplrConfig(max_iter=1000, tol=1e-12, record_every=1000))
    assert ref.trace.rows[-1].marginal_error <= 1e-12, ref.trace.rows[-1]
    fstar = ref.trace.rows[-1].f
    rows = run.trace.rows
    e0, eK = rows[0].f - fstar, rows[-1].f - fstar
    assert e0 > 0.0
    for a, b in zip(rows, rows[1:]):
        assert b.f - fstar <= (a.f - fstar) + 1e-12 * (1.0 + abs(a.f))
    assert eK <= 1e-10 * e0, eK / e0


def test_criterion_11_harness_fidelity_256(solver, tmp_path):
    spec = io.BenchSpec(gen=io.GeneratorSpec("synth2", 256, 256), eta=0.001, algos=["sinkhorn", "splr"],
                        checkpoints=[10, 50, 200], repeats=3, warmup=1)
    report = io.run_benchmark(spec, solver)
    path = tmp_path / "report.csv"
    io.emit_csv(report, str(path))
    with open(path) as f:
        assert f.readline().rstrip("\n") == io.CSV_HEADER
    series = io.parse_report_csv(str(path))
    assert len(series) == 2
    err = {}
    for ar in report.algos:
        for row in ar.rows:
            if row.iter == 200 and not row.failed:
                err[ar.algo] = row.marginal_error
    assert err.get("sinkhorn", -1.0) > 0.0 and err.get("splr", -1.0) >= 0.0
    assert err["splr"] < err["sinkhorn"], err


def test_parallel_repeats_keep_errors_deterministic(solver):
    # bench.h:203-211 / test_bench.cpp "parallel repeats": concurrent repeats, one thread and one context each;
    # errors and objectives are bit-identical to the sequential run's, only wall times differ
    spec = io.BenchSpec(gen=io.GeneratorSpec("synth2", 48, 40), eta=0.01, algos=["sinkhorn", "splr"], checkpoints=[5, 20],
                        repeats=6, warmup=0, splr=rg.SplrConfig(S=5, J=2))
    seq = io.run_benchmark(spec, solver)
    spec.parallel_repeats = True
    par = io.run_benchmark(spec, solver)
    for a, b in zip(seq.algos, par.algos):
        for ra, rb in zip(a.rows, b.rows):
            assert not rb.failed and len(rb.samples) == 6
            assert (ra.f, ra.marginal_error, ra.duality_gap) == (rb.f, rb.marginal_error, rb.duality_gap)
            assert all((q.f, q.marginal_error) == (ra.samples[0].f, ra.samples[0].marginal_error) for q in rb.samples)
