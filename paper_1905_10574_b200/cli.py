"""`rsylv-bench` on the B200 engine: verification, timed runs with CSV output, tile-size tuning.

    python -m paper_1905_10574_b200 verify [--sizes 6,10,16] [--count 3] [--seed 42]
            [--omega 1e4] [--mu 1e-3] [--nu 1e-2] [--growth-size 100] [--tile-size 8]
            [--tolerance 1e-11] [--inject-bug] [--quiet]
    python -m paper_1905_10574_b200 bench [--solver nonrobust|robust-scalar|robust-tiled]
            [--m 1024] [--n 1024] [--mu 1024,2048] [--nu N] [--omega W] [--tile-size 256]
            [--workers 0,8] [--reps 3] [--pattern mixed|ones] [--csv out.csv] [--dump prefix]
            [--gpus-column]
    python -m paper_1905_10574_b200 tune [--m] [--n] [--tile-min 32] [--tile-max 256]
            [--tile-step 32] [--workers 0] [--reps 3] [--pattern] [--csv]

Mirrors tools/rsylv_bench.cpp:22-272 (the reference's CLI11 driver):
same subcommands, options, defaults, generators (testgen.py), run records and CSV format
(records.py: the reference's 14 columns, byte-identical number format; `--gpus-column` adds
a 15th `gpus` column), lower-median marking, "best tile size" rule (ties keep the smaller
tile), exit codes (verify: 0 OK / 1 FAILED; errors: "error: ..." and 2). The solvers are the
GPU engine (api.py); `workers` is recorded as given (one GPU serves every worker count).
Wall time is the reference's convention: the solver call on host data (H2D, solve, D2H)
after one untimed warm-up call per configuration (CUDA context and buffers).
"""
from __future__ import annotations

import argparse
import math
import sys
import time

from . import api
from . import records as rec
from . import testgen as tg
from . import verify as vf


def _csv_list(conv):
    def parse(s: str):
        return [conv(x) for x in s.split(",") if x != ""]
    return parse


def _pattern(name: str, n: int):
    return tg.ones_pattern(n) if name == "ones" else tg.mixed_pattern(n)


def _mark_median(rows, first: int) -> None:
    """rsylv_bench.cpp:48-57: lower median by wall time within rows[first:]."""
    order = sorted(range(first, len(rows)), key=lambda i: rows[i].wall_time_seconds)
    if order:
        rows[order[(len(order) - 1) // 2]].median = True


def _solve(args, qa, qb, c, cfg, workers, probe=None):
    if args.solver == "nonrobust":
        return api.solve_nonrobust(qa, qb, c, device=args.device), None
    if args.solver == "robust-scalar":
        return None, api.solve_robust_scalar(qa, qb, c, cfg, device=args.device)
    mode = api.ExecutionMode.sequential() if workers == 0 else api.ExecutionMode.parallel(workers)
    return None, api.solve_tiled_robust(qa, qb, c, args.tile_size, cfg, mode, probe,
                                        device=args.device)


def _run_once(args, mu, nu, workers, a, ac, b, bc, c) -> rec.RunRecord:
    """rsylv_bench.cpp:59-108."""
    r = rec.RunRecord(solver=args.solver, m=args.m, n=args.n, tile_size=args.tile_size,
                      workers=workers if args.solver == "robust-tiled" else 0, mu=mu, nu=nu,
                      omega=args.omega, gpus=1)
    qa, qb = api.QuasiTriangular.from_codes(a, ac), api.QuasiTriangular.from_codes(b, bc)
    cfg = api.OverflowConfig(omega=args.omega)
    state = {"min": 1.0}

    def probe(k, l, al, norm):
        state["min"] = min(state["min"], al)

    t0 = time.perf_counter()
    y, res = _solve(args, qa, qb, c, cfg, workers, probe)
    r.wall_time_seconds = time.perf_counter() - t0
    if y is not None:
        r.residual = vf.relative_residual(a, b, c, y, 0, args.device)
    else:
        r.alpha = res.alpha
        r.min_local_alpha = res.alpha if args.solver == "robust-scalar" else state["min"]
        r.residual = vf.relative_residual(a, b, c, res.y, res.alpha_exp, args.device)
    r.scaling_events = cfg.scaling_events
    return r


def _emit(args, rows) -> None:
    """rsylv_bench.cpp:110-120."""
    if not args.csv:
        rec.write_csv(sys.stdout, rows, args.gpus_column)
    else:
        with open(args.csv, "w") as fh:
            rec.write_csv(fh, rows, args.gpus_column)
        print(f"wrote {len(rows)} rows to {args.csv}")


def _system(args, mu, nu):
    a, ac = tg.generate_quasi_triangular(args.m, mu, _pattern(args.pattern, args.m))
    b, bc = tg.generate_quasi_triangular(args.n, nu, _pattern(args.pattern, args.n))
    return a, ac, b, bc, tg.generate_rhs(args.m, args.n)


def cmd_bench(args) -> int:
    """rsylv_bench.cpp:122-158."""
    mus = args.mu or [float(args.m)]
    nu = float(args.n) if args.nu < 0 else args.nu
    rows = []
    for mu in mus:
        a, ac, b, bc, c = _system(args, mu, nu)
        for workers in args.workers:
            _run_once(args, mu, nu, workers, a, ac, b, bc, c)  # untimed warm-up
            first = len(rows)
            for _ in range(args.reps):
                rows.append(_run_once(args, mu, nu, workers, a, ac, b, bc, c))
            _mark_median(rows, first)
        if args.dump:
            tag = "_mu" + rec.format_double(mu)
            rec.write_matrix_file(args.dump + tag + "_a.txt", a)
            rec.write_matrix_file(args.dump + tag + "_b.txt", b)
            rec.write_matrix_file(args.dump + tag + "_c.txt", c)
            y, res = _solve(args, api.QuasiTriangular.from_codes(a, ac),
                            api.QuasiTriangular.from_codes(b, bc), c,
                            api.OverflowConfig(omega=args.omega), 0)
            rec.write_matrix_file(args.dump + tag + "_y.txt", y if y is not None else res.y)
    _emit(args, rows)
    return 0


def cmd_tune(args) -> int:
    """rsylv_bench.cpp:160-192."""
    if args.tile_min < 2 or args.tile_max < args.tile_min or args.tile_step < 1:
        raise ValueError("tune: bad tile range")
    args.solver = "robust-tiled"
    mu = args.mu[0] if args.mu else float(args.m)
    nu = float(args.n) if args.nu < 0 else args.nu
    a, ac, b, bc, c = _system(args, mu, nu)
    rows, best_tile, best = [], 0, math.inf
    sizes = list(range(args.tile_min, args.tile_max + 1, args.tile_step))
    above = [ts for ts in sizes if ts > api.INTERNAL_TILE]
    if above:
        # the device serves every request above 128 with 128-tiles (one CTA per tile): those
        # sizes run the same partition and time the same; they stay in the CSV for the record
        print(f"note: tile sizes {above[0]}..{above[-1]} exceed the internal tile "
              f"({api.INTERNAL_TILE}) and are served by {api.INTERNAL_TILE}-tiles", file=sys.stderr)
    for ts in sizes:
        args.tile_size = ts
        _run_once(args, mu, nu, args.workers[0], a, ac, b, bc, c)  # untimed warm-up
        first = len(rows)
        for _ in range(args.reps):
            rows.append(_run_once(args, mu, nu, args.workers[0], a, ac, b, bc, c))
        _mark_median(rows, first)
        for r in rows[first:]:
            if r.median and r.wall_time_seconds < best:  # ties keep the smaller tile
                best, best_tile = r.wall_time_seconds, ts
    _emit(args, rows)
    print(f"best tile size: {best_tile} (median {rec.format_double(best)} s)")
    return 0


def cmd_verify(args) -> int:
    """rsylv_bench.cpp:245-251."""
    opt = vf.VerifyOptions(sizes=args.sizes, systems_per_size=args.count, seed=args.seed,
                           omegas=args.omega, mu=args.mu, nu=args.nu,
                           growth_size=args.growth_size, tile_size=args.tile_size,
                           oracle_tol=args.tolerance, inject_bug=args.inject_bug)
    rep = vf.run_verification(opt, args.device)
    if not args.quiet:
        sys.stdout.write(rep.text)
    print(f"min-local-alpha {rec.format_double(rep.min_local_alpha)}")
    print("OK" if rep.ok else "FAILED")
    return 0 if rep.ok else 1


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="rsylv-bench",
                                description="robust triangular Sylvester equation solvers: "
                                            "verification and benchmarks (B200)")
    p.add_argument("--device", type=int, default=0, help="CUDA device")
    sub = p.add_subparsers(dest="cmd", required=True)

    d = vf.VerifyOptions()
    v = sub.add_parser("verify", help="run the self-verification suites")
    v.add_argument("--sizes", type=_csv_list(int), default=d.sizes)
    v.add_argument("--count", type=int, default=d.systems_per_size)
    v.add_argument("--seed", type=int, default=d.seed)
    v.add_argument("--omega", type=_csv_list(float), default=d.omegas)
    v.add_argument("--mu", type=float, default=d.mu)
    v.add_argument("--nu", type=float, default=d.nu)
    v.add_argument("--growth-size", type=int, default=d.growth_size)
    v.add_argument("--tile-size", type=int, default=d.tile_size)
    v.add_argument("--tolerance", type=float, default=d.oracle_tol)
    v.add_argument("--inject-bug", action="store_true")
    v.add_argument("--quiet", action="store_true")

    def common(q, tune: bool):
        q.add_argument("--m", type=int, default=1024)
        q.add_argument("--n", type=int, default=1024)
        q.add_argument("--mu", type=_csv_list(float), default=[])
        q.add_argument("--nu", type=float, default=-1.0)
        q.add_argument("--omega", type=float, default=api.default_omega())
        q.add_argument("--reps", type=int, default=3)
        q.add_argument("--pattern", choices=["mixed", "ones"], default="mixed")
        q.add_argument("--csv", default="")
        q.add_argument("--gpus-column", action="store_true",
                       help="append a 'gpus' column to the reference's 14 CSV columns")
        if tune:
            q.add_argument("--tile-min", type=int, default=32)
            q.add_argument("--tile-max", type=int, default=256)
            q.add_argument("--tile-step", type=int, default=32)
            q.add_argument("--workers", type=lambda s: [int(s)], default=[0])
        else:
            q.add_argument("--solver", choices=["nonrobust", "robust-scalar", "robust-tiled"],
                           default="robust-tiled")
            q.add_argument("--tile-size", type=int, default=256)
            q.add_argument("--workers", type=_csv_list(int), default=[0])
            q.add_argument("--dump", default="")

    common(sub.add_parser("bench", help="timed solver runs with CSV output"), False)
    common(sub.add_parser("tune", help="tile-size sweep; best median runtime wins"), True)
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        if args.cmd == "verify":
            return cmd_verify(args)
        if args.cmd == "bench":
            return cmd_bench(args)
        return cmd_tune(args)
    except Exception as e:  # rsylv_bench.cpp:265-268
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
