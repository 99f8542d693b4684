"""`python -m paper_2605_08793_b200 gen|solve|bench ...` -- the reference's command line for the solver
path (proj/tools/regot.cpp:35-190: same subcommands, options, defaults and printed lines), with the
solves on the GPU.  `plot` (SVG rendering) is outside the hot-path scope: the report CSV written by
`bench` is byte-compatible with the reference's, whose own `regot plot` renders it.
"""
from __future__ import annotations

import argparse
import sys

from . import io
from .regot import DualPoint, RegotError, SinkhornConfig, Solver, SplrConfig, ValidationError, default_solver

_KINDS = ("synth1-iid", "synth1-diff", "synth2")


def _gen_spec(problem: str, n: int, m: int, d: int, seed: int) -> io.GeneratorSpec:
    if problem in _KINDS:
        return io.GeneratorSpec(problem, n, m, d, seed)
    return io.GeneratorSpec("file", n, m, d, seed, problem)


def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="regot", description="Entropic-regularized optimal transport solvers and benchmarks")
    sub = ap.add_subparsers(dest="cmd", required=True)

    g = sub.add_parser("gen", help="Generate a problem instance and save it")
    g.add_argument("kind", help="synth1-iid | synth1-diff | synth2")
    g.add_argument("--n", type=int, default=64, help="source size")
    g.add_argument("--m", type=int, default=64, help="target size")
    g.add_argument("--d", type=int, default=2, help="point dimension (synth1)")
    g.add_argument("--seed", type=int, default=0, help="RNG seed (synth1)")
    g.add_argument("--eta", type=float, default=0.001, help="regularization strength")
    g.add_argument("-o", "--output", required=True, help="output .rotb file")

    s = sub.add_parser("solve", help="Run a solver on a problem")
    s.add_argument("--problem", required=True, help="file path or synth1-iid | synth1-diff | synth2")
    s.add_argument("--n", type=int, default=64, help="source size (generated problems)")
    s.add_argument("--m", type=int, default=64, help="target size (generated problems)")
    s.add_argument("--d", type=int, default=2, help="point dimension (synth1)")
    s.add_argument("--seed", type=int, default=0, help="RNG seed (synth1)")
    s.add_argument("--eta", type=float, default=None, help="regularization strength (overrides a file's eta)")
    s.add_argument("--algo", choices=("sinkhorn", "splr"), default="splr")
    s.add_argument("--max-iter", type=int, default=1000, help="iteration budget")
    s.add_argument("--tol", type=float, default=1e-8, help="marginal-error stopping threshold")
    s.add_argument("--record-every", type=int, default=1, help="trace stride")
    d0 = SplrConfig()
    s.add_argument("--tau-max", type=float, default=d0.tau_max, help="cap for the diagonal shift")
    s.add_argument("--S", type=int, default=d0.S, help="symbolic reuse period")
    s.add_argument("--J", type=int, default=d0.J, help="Sinkhorn candidate steps per refresh")
    s.add_argument("--density", type=float, default=d0.density, help="top-k density rho")
    s.add_argument("--c1", type=float, default=d0.c1, help="Wolfe sufficient-decrease constant")
    s.add_argument("--c2", type=float, default=d0.c2, help="Wolfe curvature constant")
    s.add_argument("--overlap", action="store_true", help="overlap pattern selection with candidate generation")
    s.add_argument("--trace", default="", help="write the iteration trace CSV here")
    s.add_argument("--device", type=int, default=0, help="CUDA device (extension)")

    b = sub.add_parser("bench", help="Run the benchmark protocol from a spec file")
    b.add_argument("--spec", required=True, help="flat key = value spec file")
    b.add_argument("-o", "--output", required=True, help="report CSV path")
    b.add_argument("--parallel-repeats", action="store_true", help="run repeats concurrently (one device context per thread); timings not comparable")

    p = sub.add_parser("plot", help="(not provided: render the report CSV with the reference's `regot plot`)")
    p.add_argument("rest", nargs="*")
    return ap


def main(argv=None) -> int:
    args = _parser().parse_args(argv)
    try:
        if args.cmd == "gen":
            spec = _gen_spec(args.kind, args.n, args.m, args.d, args.seed)
            if spec.kind == "file":
                raise ValidationError("gen: kind must be a synthetic generator")
            p = io.make_problem(spec, args.eta)
            io.save_problem(p, args.output)
            print(f"wrote {io.describe(spec)} eta={p.eta:g} to {args.output}")
        elif args.cmd == "solve":
            spec = _gen_spec(args.problem, args.n, args.m, args.d, args.seed)
            # a file's stored eta wins unless --eta was given explicitly
            eta = 0.0 if (spec.kind == "file" and args.eta is None) else (0.001 if args.eta is None else args.eta)
            p = io.make_problem(spec, eta)
            x0 = DualPoint.zeros(p.n, p.m)
            solver = default_solver() if args.device == 0 else Solver(args.device)
            solver.ensure_problem(p)
            if args.algo == "sinkhorn":
                res = solver.run_sinkhorn(x0, SinkhornConfig(max_iter=args.max_iter, record_every=args.record_every, tol=args.tol))
            else:
                cfg = SplrConfig(tau_max=args.tau_max, S=args.S, J=args.J, density=args.density, c1=args.c1, c2=args.c2,
                                 max_iter=args.max_iter, tol=args.tol, record_every=args.record_every, overlap=args.overlap)
                res = solver.run_splr(x0, cfg)
            trace = res.trace
            trace.problem = io.describe(spec)
            gr = solver.fused_gradient(res.x)
            last = trace.rows[-1]
            print("%s on %s: iter=%d wall=%.3f ms f=%.10g marginal_error=%.3e duality_gap=%.3e"
                  % (args.algo, trace.problem, last.iter, last.wall_ms, gr.f, gr.marginal_error, gr.duality_gap))
            if args.trace:
                io.emit_csv(trace, args.trace)
                print(f"trace written to {args.trace}")
        elif args.cmd == "bench":
            spec = io.parse_bench_spec(args.spec)
            if args.parallel_repeats:  # regot.cpp:165-166
                spec.parallel_repeats = True
            report = io.run_benchmark(spec)
            io.emit_csv(report, args.output)
            print(f"report written to {args.output}")
            for ar in report.algos:
                for row in ar.rows:
                    print("  %-10s iter=%-6d wall=%10.3f ms  error=%.3e%s"
                          % (ar.algo, row.iter, row.wall_ms, row.marginal_error, "  [failed]" if row.failed else ""))
        else:
            raise ValidationError("plot: SVG rendering is not part of this build; use the reference's `regot plot` on the report CSV")
    except RegotError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
