"""Data formats either side of the hot path: the ROTB problem container,
the trace / report CSV, the generator selector and the fixed-checkpoint benchmark protocol.

Host-side mirror of proj/include/regot/problem.h:218-324 and bench.h:22-35, 62-279, 289-339 -- same
names, argument meaning, file bytes and error classes, so a `.rotb` problem or a `%.17g` CSV written by
the reference is read here (and vice versa) bit for bit.  Solves run on the GPU through `regot.Solver`.
"""
from __future__ import annotations

import math
import os
import queue
import struct
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Union

import numpy as np

from . import problems
from .regot import (DualPoint, FormatError, IoError, ProblemInstance, RegotError, SinkhornConfig, Solver, SolverTrace,
                    SplrConfig, TraceRow, TruncationError, ValidationError, default_solver, splr_config_hash)

ROTB_MAGIC = b"ROTB"
ROTB_VERSION = 1
_MAX_DIM = 1 << 24


# ---- ROTB (problem.h:218-280) ---------------------------------------------------------------------------------
def save_problem(p: ProblemInstance, path: str) -> None:
    """magic "ROTB", version byte 1, little-endian u64 n, u64 m, f64 eta, a[n], b[m], M row-major."""
    try:
        with open(path, "wb") as f:
            f.write(ROTB_MAGIC + bytes([ROTB_VERSION]))
            f.write(struct.pack("<QQd", p.n, p.m, p.eta))
            f.write(np.ascontiguousarray(p.a, dtype="<f8").tobytes())
            f.write(np.ascontiguousarray(p.b, dtype="<f8").tobytes())
            f.write(np.ascontiguousarray(p.M, dtype="<f8").tobytes())  # C order == row-major
    except OSError as e:
        raise IoError(f"save_problem: cannot open {path}") from e


def load_problem(path: str) -> ProblemInstance:
    try:
        f = open(path, "rb")
    except OSError as e:
        raise IoError(f"load_problem: cannot open {path}") from e
    with f:
        head = f.read(4)
        if len(head) < 4:
            raise TruncationError("load_problem: truncated header")
        if head != ROTB_MAGIC:
            raise FormatError("load_problem: bad magic")
        ver = f.read(1)
        if len(ver) < 1:
            raise TruncationError("load_problem: truncated header")
        if ver[0] != ROTB_VERSION:
            raise FormatError("load_problem: unsupported version")

        def take(nbytes: int) -> bytes:
            buf = f.read(nbytes)
            if len(buf) < nbytes:
                raise TruncationError("load_problem: truncated payload")
            return buf

        n, m = struct.unpack("<QQ", take(16))
        if n == 0 or m == 0 or n > _MAX_DIM or m > _MAX_DIM:
            raise FormatError("load_problem: implausible dimensions")
        (eta,) = struct.unpack("<d", take(8))
        # a crafted or truncated header must not drive an allocation: compare the payload with what is left
        try:
            left = os.fstat(f.fileno()).st_size - f.tell()
        except (OSError, AttributeError):
            left = None
        if left is not None and left < 8 * (n + m + n * m):
            raise TruncationError("load_problem: truncated payload")
        a = np.frombuffer(take(8 * n), dtype="<f8").astype(np.float64)
        b = np.frombuffer(take(8 * m), dtype="<f8").astype(np.float64)
        M = np.frombuffer(take(8 * n * m), dtype="<f8").astype(np.float64).reshape(n, m)
    p = ProblemInstance(int(n), int(m), M, a, b, float(eta))
    problems.validate_problem(p)
    return p


# ---- generator selector (problem.h:283-324) ---------------------------------------------------------------------
@dataclass
class GeneratorSpec:
    kind: str = "synth2"  # synth1-iid | synth1-diff | synth2 | file   (+ image | gmm | uniform: BASELINE configs B, D, E)
    n: int = 64
    m: int = 64
    d: int = 2
    seed: int = 0
    path: str = ""


def make_problem(spec: GeneratorSpec, eta: float) -> ProblemInstance:
    if spec.kind == "file":
        p = load_problem(spec.path)
        if eta > 0.0:
            p.eta = eta
        problems.validate_problem(p)
        return p
    return problems.make_problem(spec.kind, spec.n, spec.m, eta, spec.d, spec.seed)  # raises on unknown kinds


def describe(spec: GeneratorSpec) -> str:
    if spec.kind == "file":
        return f"file:{spec.path}"
    s = f"{spec.kind} {spec.n}x{spec.m}"
    if spec.kind != "synth2":
        s += f" d={spec.d} seed={spec.seed}"
    return s


# ---- CSV (bench.h:22-35, 243-279, 289-339) ------------------------------------------------------------------------
CSV_HEADER = "iter,wall_ms,f,marginal_error,duality_gap"


def fmt_g17(v: float) -> str:
    """printf("%.17g"): enough digits for a bit-exact strtod round trip."""
    return "%.17g" % v


def median(v: Sequence[float]) -> float:
    s = sorted(v)
    n = len(s)
    if n == 0:
        return math.nan
    return s[n // 2] if n % 2 == 1 else 0.5 * (s[n // 2 - 1] + s[n // 2])


@dataclass
class RepeatSample:
    wall_ms: float = 0.0
    f: float = 0.0
    marginal_error: float = 0.0
    duality_gap: float = 0.0


@dataclass
class CheckpointStat:
    iter: int = 0
    failed: bool = False
    wall_ms: float = 0.0
    f: float = 0.0
    marginal_error: float = 0.0
    duality_gap: float = 0.0
    samples: List[RepeatSample] = field(default_factory=list)


@dataclass
class AlgoReport:
    algo: str = ""
    config_hash: str = ""
    rows: List[CheckpointStat] = field(default_factory=list)


@dataclass
class BenchReport:
    problem: str = ""
    eta: float = 0.0
    algos: List[AlgoReport] = field(default_factory=list)


def _row(r) -> str:
    return f"{r.iter},{fmt_g17(r.wall_ms)},{fmt_g17(r.f)},{fmt_g17(r.marginal_error)},{fmt_g17(r.duality_gap)}\n"


def emit_csv(obj: Union[SolverTrace, BenchReport], path: str) -> None:
    """Trace CSV (one row per record) or report CSV ("# algo=..." comment per algorithm)."""
    try:
        with open(path, "w", newline="") as f:
            f.write(CSV_HEADER + "\n")
            if isinstance(obj, BenchReport):
                for ar in obj.algos:
                    f.write(f"# algo={ar.algo} problem={obj.problem} eta={fmt_g17(obj.eta)} config={ar.config_hash}\n")
                    for r in ar.rows:
                        f.write(_row(r))
            else:
                for r in obj.rows:
                    f.write(_row(r))
    except OSError as e:
        raise IoError(f"emit_csv: cannot open {path}") from e


@dataclass
class PlotSeries:
    algo: str
    rows: List[TraceRow] = field(default_factory=list)


def parse_report_csv(path: str) -> List[PlotSeries]:
    try:
        with open(path, "r") as f:
            lines = f.read().split("\n")
    except OSError as e:
        raise IoError(f"parse_report_csv: cannot open {path}") from e
    if lines and lines[-1] == "":
        lines.pop()
    if not lines:
        raise FormatError("parse_report_csv: empty file")
    if lines[0].strip(" \t\r\n") != CSV_HEADER:
        raise FormatError("parse_report_csv: unexpected header")
    series: List[PlotSeries] = []
    for line in lines[1:]:
        t = line.strip(" \t\r\n")
        if not t:
            continue
        if t[0] == "#":
            pos = t.find("algo=")
            if pos >= 0:
                end = t.find(" ", pos)
                if end < 0:
                    end = len(t)
                series.append(PlotSeries(t[pos + 5:end]))
            continue
        parts = [q.strip(" \t\r\n") for q in t.split(",")]
        if len(parts) != 5:
            raise FormatError(f"parse_report_csv: malformed row '{t}'")
        if not series:
            series.append(PlotSeries("trace"))
        try:
            it = int(parts[0])
        except ValueError as e:
            raise FormatError(f"parse_report_csv: bad iteration field '{parts[0]}'") from e

        def num(s: str) -> float:  # strtod semantics: unparsable -> 0
            try:
                return float(s)
            except ValueError:
                return 0.0

        series[-1].rows.append(TraceRow(it, num(parts[1]), num(parts[2]), num(parts[3]), num(parts[4])))
    return series


# ---- benchmark protocol (bench.h:75-240) --------------------------------------------------------------------------
@dataclass
class BenchSpec:
    gen: GeneratorSpec = field(default_factory=GeneratorSpec)
    eta: float = 0.001
    algos: List[str] = field(default_factory=lambda: ["sinkhorn", "splr"])
    splr: SplrConfig = field(default_factory=SplrConfig)
    checkpoints: List[int] = field(default_factory=lambda: [10, 20, 50, 100])
    repeats: int = 10
    warmup: int = 1
    parallel_repeats: bool = False  # concurrent repeats; timings not comparable (bench.h:84)

    def validate(self) -> None:
        if self.repeats < 1:
            raise ValidationError("BenchSpec: repeats must be >= 1")
        if self.warmup < 0:
            raise ValidationError("BenchSpec: warmup must be >= 0")
        if not self.checkpoints:
            raise ValidationError("BenchSpec: need at least one checkpoint")
        for i, c in enumerate(self.checkpoints):
            if c < 1:
                raise ValidationError("BenchSpec: checkpoints must be >= 1")
            if i > 0 and c <= self.checkpoints[i - 1]:
                raise ValidationError("BenchSpec: checkpoints must be strictly increasing")
        if not self.algos:
            raise ValidationError("BenchSpec: need at least one algorithm")
        for a in self.algos:
            if a not in ("sinkhorn", "splr"):
                raise ValidationError(f"BenchSpec: unknown algorithm '{a}'")
            if a == "splr":
                self.splr.validate()


def bench_solve(algo: str, p: ProblemInstance, splr_cfg: SplrConfig, iters: int, solver=None) -> DualPoint:
    """One run for exactly `iters` iterations (tolerance zero); bench.h:148-164."""
    s = solver or default_solver()
    s.ensure_problem(p)
    if algo == "sinkhorn":
        return s.run_sinkhorn(DualPoint.zeros(p.n, p.m), SinkhornConfig(max_iter=iters, record_every=iters, tol=0.0)).x
    c = SplrConfig(**{**splr_cfg.__dict__})
    c.max_iter, c.record_every, c.tol = iters, iters, 0.0
    return s.run_splr(DualPoint.zeros(p.n, p.m), c).x


_MAX_PARALLEL_CONTEXTS = 4
_pool_lock = threading.Lock()


def _context_pool(s, p: ProblemInstance, count: int):
    """Extra device contexts of the same problem for concurrent repeats, cached on the primary solver."""
    pool = getattr(s, "_bench_pool", None)
    if pool is None:
        pool = s._bench_pool = {"key": None, "free": queue.SimpleQueue(), "all": []}
    key = (id(p), p.n, p.m, p.eta)
    if pool["key"] != key:
        for sv in pool["all"]:
            sv.close()
        pool.update(key=key, free=queue.SimpleQueue(), all=[])
    while len(pool["all"]) < count:
        sv = Solver(s.device)
        sv.set_problem(p)
        pool["all"].append(sv)
        pool["free"].put(sv)
    return pool


def _with_context(pool, fn):
    sv = pool["free"].get()
    try:
        return fn(sv)
    finally:
        pool["free"].put(sv)


def run_benchmark(spec: BenchSpec, solver=None) -> BenchReport:
    """Per algorithm and checkpoint: `warmup` discarded runs, `repeats` timed runs of exactly that many
    iterations from x0 = 0, medians; a solver failure marks the cell failed (NaN) and the run goes on."""
    spec.validate()
    p = make_problem(spec.gen, spec.eta)
    s = solver or default_solver()
    s.ensure_problem(p)
    report = BenchReport(describe(spec.gen), p.eta)
    for algo in spec.algos:
        ar = AlgoReport(algo, splr_config_hash(spec.splr) if algo == "splr" else "sinkhorn")
        for cp in spec.checkpoints:
            stat = CheckpointStat(iter=cp)
            try:
                for _ in range(spec.warmup):
                    bench_solve(algo, p, spec.splr, cp, s)

                def one_repeat(sv):
                    t0 = time.perf_counter()
                    x = bench_solve(algo, p, spec.splr, cp, sv)
                    wall = 1e3 * (time.perf_counter() - t0)
                    g = sv.fused_gradient(x)
                    return RepeatSample(wall, g.f, g.marginal_error, g.duality_gap)

                if spec.parallel_repeats:
                    # property runs only (bench.h:203-211): the repeats run concurrently, one thread and one
                    # device context each (entry points are re-entrant per handle); errors stay deterministic,
                    # wall times reflect contention
                    pool = _context_pool(s, p, min(spec.repeats, _MAX_PARALLEL_CONTEXTS))
                    with ThreadPoolExecutor(max_workers=len(pool)) as ex:
                        futs = [ex.submit(_with_context, pool, one_repeat) for _ in range(spec.repeats)]
                        stat.samples.extend(f.result() for f in futs)
                else:
                    for _ in range(spec.repeats):
                        stat.samples.append(one_repeat(s))
                stat.wall_ms = median([q.wall_ms for q in stat.samples])
                stat.f = median([q.f for q in stat.samples])
                stat.marginal_error = median([q.marginal_error for q in stat.samples])
                stat.duality_gap = median([q.duality_gap for q in stat.samples])
            except RegotError:
                stat.failed = True
                stat.wall_ms = stat.f = stat.marginal_error = stat.duality_gap = math.nan
            ar.rows.append(stat)
        report.algos.append(ar)
    return report


# ---- spec file (bench.h:509-586) ------------------------------------------------------------------------------------
_GENERATED_KINDS = ("synth1-iid", "synth1-diff", "synth2")


def _stol(val: str, what: str) -> int:
    """std::stol: leading integer, trailing text ignored; nothing parsable is an error (the reference
    lets std::invalid_argument escape; here it is a ValidationError naming the key)."""
    s = val.lstrip()
    k = 1 if s[:1] in "+-" else 0
    e = k
    while e < len(s) and s[e].isdigit():
        e += 1
    if e == k:
        raise ValidationError(f"parse_bench_spec: '{what}' needs an integer, got '{val}'")
    return int(s[:e])


def _strtod(val: str) -> float:
    """strtod(val, nullptr): longest parsable prefix, 0 when there is none."""
    s = val.strip()
    for e in range(len(s), 0, -1):
        try:
            return float(s[:e])
        except ValueError:
            continue
    return 0.0


def parse_bench_spec(path: str) -> BenchSpec:
    """Flat `key = value` lines, `#` comments; same keys, defaults and errors as bench.h:509-586
    (`parallel-repeats` runs the repeats from several threads, one device context each)."""
    try:
        with open(path, "r") as fh:
            lines = fh.read().split("\n")
    except OSError as e:
        raise IoError(f"parse_bench_spec: cannot open {path}") from e
    spec = BenchSpec()
    spec.algos = []
    have_eta = False
    ws = " \t\r\n"
    for lineno, line in enumerate(lines, 1):
        t = line.strip(ws)
        if not t or t[0] == "#":
            continue
        eq = t.find("=")
        if eq < 0:
            raise ValidationError(f"parse_bench_spec: line {lineno} is not 'key = value'")
        key, val = t[:eq].strip(ws), t[eq + 1:].strip(ws)
        if key == "problem":
            if val in _GENERATED_KINDS:
                spec.gen.kind = val
            else:
                spec.gen.kind, spec.gen.path = "file", val
        elif key in ("n", "m", "d", "seed"):
            setattr(spec.gen, key, _stol(val, key))
        elif key == "eta":
            spec.eta, have_eta = _strtod(val), True
        elif key == "algo":
            spec.algos += [a.strip(ws) for a in val.split(",") if a.strip(ws)]
        elif key == "checkpoints":
            spec.checkpoints = [_stol(c, key) for c in val.split(",") if c.strip(ws)]
        elif key in ("repeats", "warmup"):
            setattr(spec, key, _stol(val, key))
        elif key == "tau-max":
            spec.splr.tau_max = _strtod(val)
        elif key in ("S", "J"):
            setattr(spec.splr, key, _stol(val, key))
        elif key in ("density", "c1", "c2"):
            setattr(spec.splr, key, _strtod(val))
        elif key == "max-ls-trials":
            spec.splr.max_ls_trials = _stol(val, key)
        elif key == "overlap":
            spec.splr.overlap = val in ("1", "true")
        elif key == "parallel-repeats":
            spec.parallel_repeats = val in ("1", "true")
        else:
            raise ValidationError(f"parse_bench_spec: unknown key '{key}'")
    if not spec.algos:
        spec.algos = ["sinkhorn", "splr"]
    if spec.gen.kind == "file" and not have_eta:
        spec.eta = 0.0  # keep the eta stored in the file
    spec.validate()
    return spec
