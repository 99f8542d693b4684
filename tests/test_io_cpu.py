"""ROTB container + trace/report CSV: this repo's reader/writer against fixtures written
by the REFERENCE's own save_problem / emit_csv (tests/golden/make_io_golden.py), plus the error cases of
test_problem.cpp:153-223 and the CSV cases of test_bench.cpp:54-102.  CPU only."""
import math
import os

import numpy as np
import pytest

import paper_2605_08793_b200 as rg
from paper_2605_08793_b200 import io, problems

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_reads_the_reference_written_rotb_and_rewrites_it_byte_for_byte(tmp_path, oracle):
    src = os.path.join(GOLD, "ref_synth1diff_6x5.rotb")
    p = io.load_problem(src)
    assert (p.n, p.m, p.eta) == (6, 5, 0.0125)
    ref = oracle.gen_problem("synth1-diff", 6, 5, 0.0125, d=3, seed=42)  # the instance the fixture was made from
    assert np.array_equal(p.M, ref["M"]) and np.array_equal(p.a, ref["a"]) and np.array_equal(p.b, ref["b"])
    out = tmp_path / "again.rotb"
    io.save_problem(p, str(out))
    assert out.read_bytes() == open(src, "rb").read()


def test_round_trip_is_bit_exact(tmp_path):
    # test_problem.cpp:153-166
    p = problems.gen_synthetic1(13, 9, "iid", 2, 11, 0.07)
    f = str(tmp_path / "roundtrip.rotb")
    io.save_problem(p, f)
    q = io.load_problem(f)
    assert (q.n, q.m) == (p.n, p.m) and q.eta == p.eta
    assert q.M.tobytes() == np.ascontiguousarray(p.M).tobytes() and q.a.tobytes() == p.a.tobytes() and q.b.tobytes() == p.b.tobytes()
    assert os.path.getsize(f) == 5 + 24 + 8 * (13 + 9 + 13 * 9)


def test_load_error_classes(tmp_path):
    # test_problem.cpp:168-223
    bad = tmp_path / "badmagic.rotb"
    bad.write_bytes(b"XXXX" + bytes(64))
    with pytest.raises(rg.FormatError, match="bad magic"):
        io.load_problem(str(bad))
    good = tmp_path / "good.rotb"
    io.save_problem(problems.gen_synthetic2(6, 5, 0.1), str(good))
    raw = bytearray(good.read_bytes())
    v2 = tmp_path / "v2.rotb"
    v2.write_bytes(bytes(raw[:4]) + b"\x02" + bytes(raw[5:]))
    with pytest.raises(rg.FormatError, match="unsupported version"):
        io.load_problem(str(v2))
    half = tmp_path / "half.rotb"
    half.write_bytes(bytes(raw[: len(raw) // 2]))
    with pytest.raises(rg.TruncationError):
        io.load_problem(str(half))
    (tmp_path / "hdr.rotb").write_bytes(b"RO")
    with pytest.raises(rg.TruncationError, match="truncated header"):
        io.load_problem(str(tmp_path / "hdr.rotb"))
    zero = tmp_path / "dims.rotb"
    zero.write_bytes(b"ROTB\x01" + bytes(24))
    with pytest.raises(rg.FormatError, match="implausible"):
        io.load_problem(str(zero))
    p = problems.gen_synthetic2(5, 5, 0.1)
    p.a[0], p.a[1] = 0.0, 2.0 / 5.0  # sum stays 1: only positivity fails
    io.save_problem(p, str(tmp_path / "zeromass.rotb"))
    with pytest.raises(rg.ValidationError):
        io.load_problem(str(tmp_path / "zeromass.rotb"))
    with pytest.raises(rg.IoError):
        io.load_problem(str(tmp_path / "missing.rotb"))


def test_make_problem_file_kind_and_describe(tmp_path):
    p = problems.gen_synthetic2(8, 7, 0.02)
    f = str(tmp_path / "p.rotb")
    io.save_problem(p, f)
    spec = io.GeneratorSpec(kind="file", path=f)
    assert io.make_problem(spec, 0.0).eta == 0.02      # the file's eta wins unless one is given (regot.cpp:121-122)
    assert io.make_problem(spec, 0.5).eta == 0.5
    assert io.describe(spec) == "file:" + f
    assert io.describe(io.GeneratorSpec("synth2", 64, 32)) == "synth2 64x32"
    assert io.describe(io.GeneratorSpec("synth1-iid", 64, 32, 3, 9)) == "synth1-iid 64x32 d=3 seed=9"
    with pytest.raises(rg.ValidationError, match="unknown generator"):
        io.make_problem(io.GeneratorSpec(kind="nope"), 0.1)


def test_trace_csv_matches_the_reference_writer_byte_for_byte(tmp_path):
    want = open(os.path.join(GOLD, "ref_trace.csv"), "rb").read()
    t = rg.SolverTrace(algo="splr", eta=0.01, config_hash="")
    for v in [(0, 0.0, 1.6638586759335181, 1.25, -0.5), (1, 0.1, 0.29051373543167602, 1e-3, 1e-300),
              (7, 123.456789012345678, -0.06647132208369197, 7.190629985496689e-09, -2.5e-17),
              (1000, 1e6, float(np.nextafter(1.0, 2.0)), 5e-324, math.inf)]:
        t.rows.append(rg.TraceRow(*v))
    f = tmp_path / "t.csv"
    io.emit_csv(t, str(f))
    assert f.read_bytes() == want
    series = io.parse_report_csv(str(f))  # test_bench.cpp:69-92: %.17g round trip is bitwise
    assert len(series) == 1 and series[0].algo == "trace"
    for got, src in zip(series[0].rows, t.rows):
        assert (got.iter, got.wall_ms, got.f, got.marginal_error, got.duality_gap) == \
               (src.iter, src.wall_ms, src.f, src.marginal_error, src.duality_gap)


def test_report_csv_sections_and_parse_errors(tmp_path):
    rep = io.BenchReport("synth2 16x16", 0.001, [
        io.AlgoReport("sinkhorn", "sinkhorn", [io.CheckpointStat(10, False, 1.5, 0.25, 1e-3, 1e-4)]),
        io.AlgoReport("splr", "0123456789abcdef", [io.CheckpointStat(10, False, 2.5, 0.125, 1e-6, 1e-7),
                                                    io.CheckpointStat(20, True, math.nan, math.nan, math.nan, math.nan)])])
    f = tmp_path / "r.csv"
    io.emit_csv(rep, str(f))
    lines = f.read_text().split("\n")
    assert lines[0] == io.CSV_HEADER == "iter,wall_ms,f,marginal_error,duality_gap"   # frozen (test_bench.cpp:54-57)
    assert lines[1] == "# algo=sinkhorn problem=synth2 16x16 eta=0.001 config=sinkhorn"
    assert lines[3] == "# algo=splr problem=synth2 16x16 eta=0.001 config=0123456789abcdef"
    s = io.parse_report_csv(str(f))
    assert [q.algo for q in s] == ["sinkhorn", "splr"] and len(s[1].rows) == 2 and math.isnan(s[1].rows[1].f)
    (tmp_path / "e.csv").write_text("")
    with pytest.raises(rg.FormatError, match="empty"):
        io.parse_report_csv(str(tmp_path / "e.csv"))
    (tmp_path / "h.csv").write_text("a,b\n")
    with pytest.raises(rg.FormatError, match="header"):
        io.parse_report_csv(str(tmp_path / "h.csv"))
    (tmp_path / "m.csv").write_text(io.CSV_HEADER + "\n1,2,3\n")
    with pytest.raises(rg.FormatError, match="malformed"):
        io.parse_report_csv(str(tmp_path / "m.csv"))
    (tmp_path / "i.csv").write_text(io.CSV_HEADER + "\nx,1,2,3,4\n")
    with pytest.raises(rg.FormatError, match="iteration"):
        io.parse_report_csv(str(tmp_path / "i.csv"))


def test_medians_and_spec_validation():
    # test_bench.cpp:104-109, 304-348
    assert io.median([3.0, 1.0, 2.0]) == 2.0 and io.median([4.0, 1.0, 3.0, 2.0]) == 2.5 and math.isnan(io.median([]))
    io.BenchSpec().validate()
    for bad in (dict(repeats=0), dict(warmup=-1), dict(checkpoints=[]), dict(checkpoints=[10, 10]), dict(checkpoints=[0]),
                dict(algos=[]), dict(algos=["newton"])):
        with pytest.raises(rg.ValidationError):
            io.BenchSpec(**bad).validate()
    with pytest.raises(rg.ValidationError):
        io.BenchSpec(splr=rg.SplrConfig(c1=0.7)).validate()


def test_bench_spec_keyfiles_parse_and_validate(tmp_path):
    # test_bench.cpp:304-348 (same file contents, same expectations)
    path = str(tmp_path / "spec.cfg")
    with open(path, "w") as fh:
        fh.write("# benchmark configuration\nproblem = synth2\nn = 32\nm = 24\neta = 0.005\nalgo = sinkhorn,splr\n"
                 "checkpoints = 5, 10, 20\nrepeats = 3\nwarmup = 1\nS = 7\nJ = 2\ndensity = 0.05\n")
    spec = io.parse_bench_spec(path)
    assert (spec.gen.kind, spec.gen.n, spec.gen.m, spec.eta) == ("synth2", 32, 24, 0.005)
    assert spec.algos == ["sinkhorn", "splr"] and spec.checkpoints == [5, 10, 20]
    assert (spec.repeats, spec.warmup, spec.splr.S, spec.splr.J, spec.splr.density) == (3, 1, 7, 2, 0.05)
    for body in ("problem = synth2\nbogus = 1\n", "problem = synth2\ncheckpoints = 10,5\n", "problem = synth2\njust a line\n",
                 "problem = synth2\nn = many\n"):
        with open(path, "w") as fh:
            fh.write(body)
        with pytest.raises(rg.ValidationError):
            io.parse_bench_spec(path)
    with pytest.raises(rg.IoError):
        io.parse_bench_spec(str(tmp_path / "absent.cfg"))
    # bench.h:534-543, 580-583: anything else is a file path whose stored eta is kept; default algorithms
    with open(path, "w") as fh:
        fh.write("problem = some/file.rotb\ntau-max = 0.5\nmax-ls-trials = 12\noverlap = true\nparallel-repeats = 1\n")
    spec = io.parse_bench_spec(path)
    assert (spec.gen.kind, spec.gen.path, spec.eta) == ("file", "some/file.rotb", 0.0)
    assert spec.algos == ["sinkhorn", "splr"] and spec.splr.tau_max == 0.5 and spec.splr.max_ls_trials == 12 and spec.splr.overlap


def test_command_line_gen_and_errors(tmp_path, capsys):
    # regot.cpp:104-113, 185-189: `gen` writes the ROTB file and reports it; errors print "error: ..." and exit 1
    from paper_2605_08793_b200.__main__ import main
    out = str(tmp_path / "p.rotb")
    assert main(["gen", "synth1-iid", "--n", "12", "--m", "9", "--d", "3", "--seed", "5", "--eta", "0.01", "-o", out]) == 0
    assert capsys.readouterr().out == f"wrote synth1-iid 12x9 d=3 seed=5 eta=0.01 to {out}\n"
    p, q = io.load_problem(out), problems.gen_synthetic1(12, 9, "iid", 3, 5, 0.01)
    assert np.array_equal(p.M, q.M) and np.array_equal(p.a, q.a) and p.eta == 0.01
    assert main(["gen", "not-a-generator", "-o", out]) == 1
    assert "error: gen: kind must be a synthetic generator" in capsys.readouterr().err
    assert main(["bench", "--spec", str(tmp_path / "absent.cfg"), "-o", out]) == 1
    assert "cannot open" in capsys.readouterr().err
