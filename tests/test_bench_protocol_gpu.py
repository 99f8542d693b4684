"""GPU: the fixed-checkpoint benchmark protocol and the command line --
test_bench.cpp:111-205 and the `solve` / `bench` subcommands of tools/regot.cpp, with the CPU oracle
solving the same problems beside them."""
import math
import struct

import numpy as np
import pytest

import paper_2605_08793_b200 as rg
from paper_2605_08793_b200 import io
from paper_2605_08793_b200.__main__ import main

pytestmark = pytest.mark.gpu


def small_spec():
    # test_bench.cpp:36-50
    return io.BenchSpec(gen=io.GeneratorSpec("synth2", 16, 16), eta=0.01, algos=["sinkhorn", "splr"], checkpoints=[5, 10],
                        repeats=2, warmup=0, splr=rg.SplrConfig(S=5, J=2))


def bits(v):
    return struct.pack("<d", v)


def test_protocol_reports_deterministic_errors_and_medians(solver):
    # test_bench.cpp:111-143
    spec = small_spec()
    report = io.run_benchmark(spec, solver)
    assert len(report.algos) == 2
    for ar in report.algos:
        assert len(ar.rows) == 2
        for row in ar.rows:
            assert not row.failed and len(row.samples) == 2
            for s in row.samples:
                assert bits(s.f) == bits(row.samples[0].f) and bits(s.marginal_error) == bits(row.samples[0].marginal_error)
            assert row.marginal_error == row.samples[0].marginal_error
        assert ar.rows[1].marginal_error <= ar.rows[0].marginal_error * (1.0 + 1e-12) + 1e-300
    spec.repeats, spec.checkpoints = 1, [5]
    for ar in io.run_benchmark(spec, solver).algos:
        assert ar.rows[0].wall_ms == ar.rows[0].samples[0].wall_ms


def test_checkpoints_match_the_oracle_and_the_gap_bound(solver, oracle):
    # test_bench.cpp:163-177, and the same fixed-iteration runs on the CPU oracle
    spec = small_spec()
    p = io.make_problem(spec.gen, spec.eta)
    op = oracle.gen_problem("synth2", 16, 16, 0.01)
    assert np.array_equal(op["M"], p.M)
    for algo in spec.algos:
        for cp in spec.checkpoints:
            x = io.bench_solve(algo, p, spec.splr, cp, solver)
            gr = solver.fused_gradient(x)
            bound = max(np.abs(x.alpha).max(), np.abs(x.beta).max()) * gr.marginal_error
            assert abs(gr.duality_gap) <= bound * (1.0 + 1e-12) + 1e-300
            z = np.zeros(16)
            if algo == "sinkhorn":
                want = oracle.run_sinkhorn(op, z, z, rg.SinkhornConfig(max_iter=cp, record_every=cp, tol=0.0)._c())
            else:
                want = oracle.run_splr(op, z, z, rg.SplrConfig(S=5, J=2, max_iter=cp, record_every=cp, tol=0.0)._c())
            _, _, f_ref, err_ref, _ = want["trace"][-1]
            assert want["trace"][-1][0] == cp
            assert abs(gr.f - f_ref) <= 1e-9 * abs(f_ref)
            assert abs(gr.marginal_error - err_ref) <= 1e-6 * err_ref + 1e-14


def test_report_csv_sections_parse_back(solver, tmp_path):
    # test_bench.cpp:179-205
    report = io.run_benchmark(small_spec(), solver)
    path = str(tmp_path / "report.csv")
    io.emit_csv(report, path)
    body = open(path).read()
    assert body.startswith("iter,wall_ms,f,marginal_error,duality_gap\n") and body.count("# algo=") == 2
    series = io.parse_report_csv(path)
    assert [s.algo for s in series] == ["sinkhorn", "splr"]
    for s, ar in zip(series, report.algos):
        assert len(s.rows) == len(ar.rows)
        for a, b in zip(ar.rows, s.rows):
            assert a.iter == b.iter and bits(a.f) == bits(b.f) and bits(a.marginal_error) == bits(b.marginal_error)


def test_command_line_solve_and_bench(tmp_path, capsys, oracle):
    # regot.cpp:114-172: generated problem, trace CSV, a stored file whose eta is kept / overridden, the spec-file bench
    trace = str(tmp_path / "t.csv")
    assert main(["solve", "--problem", "synth2", "--n", "48", "--m", "40", "--eta", "0.01", "--S", "5", "--J", "2", "--trace", trace]) == 0
    out = capsys.readouterr().out.split("\n")
    assert out[0].startswith("splr on synth2 48x40: iter=") and "marginal_error=" in out[0] and out[1] == f"trace written to {trace}"
    rows = io.parse_report_csv(trace)[0].rows
    want = oracle.run_splr(oracle.gen_problem("synth2", 48, 40, 0.01), np.zeros(48), np.zeros(40),
                           rg.SplrConfig(S=5, J=2, max_iter=1000, tol=1e-8)._c())["trace"]
    # the iterates agree until the objective is flat to its last bits (error < 1e-7 on synthetic II); where the error then
    # crosses 1e-8 is decided by rounding (iteration-count parity), hence the slack on the count
    assert rows[-1].marginal_error <= 1e-8 and abs(rows[-1].iter - want[-1][0]) <= math.ceil(0.15 * want[-1][0])
    early = [(r, w) for r, w in zip(rows, want) if w[3] >= 1e-7]
    assert len(early) >= 20
    for r, w in early:
        assert r.iter == w[0] and abs(r.f - w[2]) <= 1e-9 * abs(w[2]) and abs(r.marginal_error - w[3]) <= 1e-5 * w[3]

    rotb = str(tmp_path / "p.rotb")
    assert main(["gen", "synth1-diff", "--n", "32", "--m", "24", "--seed", "3", "--eta", "0.02", "-o", rotb]) == 0
    capsys.readouterr()
    assert main(["solve", "--problem", rotb, "--algo", "sinkhorn", "--max-iter", "40", "--tol", "0"]) == 0
    line_file = capsys.readouterr().out.split("\n")[0]
    assert line_file.startswith(f"sinkhorn on file:{rotb}: iter=40 ")
    ref = oracle.run_sinkhorn(oracle.gen_problem("synth1-diff", 32, 24, 0.02, d=2, seed=3), np.zeros(32), np.zeros(24),
                              rg.SinkhornConfig(max_iter=40, record_every=40, tol=0.0)._c())["trace"][-1]
    f_cli = float(line_file.split(" f=")[1].split(" ")[0])
    assert abs(f_cli - ref[2]) <= 1e-9 * abs(ref[2])  # printed with %.10g
    assert main(["solve", "--problem", rotb, "--algo", "sinkhorn", "--max-iter", "40", "--tol", "0", "--eta", "0.05"]) == 0
    assert capsys.readouterr().out.split("\n")[0] != line_file

    spec, rep = str(tmp_path / "b.cfg"), str(tmp_path / "r.csv")
    with open(spec, "w") as fh:
        fh.write("problem = synth2\nn = 16\nm = 16\neta = 0.01\ncheckpoints = 5,10\nrepeats = 2\nwarmup = 0\nS = 5\nJ = 2\n")
    assert main(["bench", "--spec", spec, "-o", rep]) == 0
    out = capsys.readouterr().out.split("\n")
    assert out[0] == f"report written to {rep}" and sum(1 for q in out if q.startswith("  sinkhorn") or q.startswith("  splr")) == 4
    assert [s.algo for s in io.parse_report_csv(rep)] == ["sinkhorn", "splr"]
    assert main(["solve", "--problem", str(tmp_path / "absent.rotb")]) == 1 and "error:" in capsys.readouterr().err
