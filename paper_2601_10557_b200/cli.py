"""Command line drop-in for ``bsesolve generate / solve / bench`` (cli.py:93-361 of the
reference) on the GPU: same options, outputs (eigenvalues.csv, eigenvectors.bin, trace.csv,
manifest.json, bench.csv) and exit codes (0 ok, 2 validation, 3 I/O, 4 numerical).

    python -m paper_2601_10557_b200 solve --pchb ham.pchb --nev 50 --nex 20 --tol 1e-10 --out run/
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

EXIT_VALIDATION, EXIT_IO, EXIT_NUMERICAL = 2, 3, 4


def _load(args):
    from . import fileio
    from .hamiltonian import BseHamiltonian

    if args.pchb:
        if args.a or args.b:
            raise ValueError_("--pchb excludes --a/--b")
        ham = fileio.read_pchb(args.pchb)
        return ham, {str(args.pchb): fileio.digest64(args.pchb)}
    if not (args.a and args.b):
        raise ValueError_("provide --a and --b, or --pchb")
    ham = BseHamiltonian(fileio.read_matrix_market(args.a), fileio.read_matrix_market(args.b))
    return ham, {str(args.a): fileio.digest64(args.a), str(args.b): fileio.digest64(args.b)}


def ValueError_(msg):  # noqa: N802 - reference ValidationError under a short name
    from .errors import ValidationError

    return ValidationError(msg)


def _config(args):
    from .solver import SolverConfig

    deg = args.deg
    if deg % 2:
        print(f"warning: filter degree must be even, rounding {deg} up to {deg + 1}", file=sys.stderr)
        deg += 1
    return SolverConfig(nev=args.nev, nex=args.nex, deg=deg, tol=args.tol, maxiter=args.maxiter,
                        rr_variant=args.rr, seed=args.seed, lanczos_steps=args.lanczos_steps,
                        rel_res=args.rel_res, reproducible=args.reproducible)


def cmd_generate(args) -> None:
    from . import fileio
    from .generate import GeneratorSpec, generate

    spec = GeneratorSpec(m=args.m, seed=args.seed, alpha=args.alpha, coupling_ratio=args.coupling_ratio,
                         mode=args.mode)
    ham = generate(spec)
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    a, b = ham.host_blocks()
    if args.format == "mm":
        fileio.write_matrix_market(out / "A.mtx", a, comment=f" resonant block, seed={args.seed}")
        fileio.write_matrix_market(out / "B.mtx", b, comment=f" coupling block, seed={args.seed}")
        outputs = ["A.mtx", "B.mtx"]
    else:
        fileio.write_pchb(out / "ham.pchb", ham)
        outputs = ["ham.pchb"]
    fileio.write_manifest(out / "manifest.json", "generate",
                          {"m": args.m, "seed": args.seed, "coupling_ratio": args.coupling_ratio,
                           "alpha": args.alpha, "mode": args.mode, "format": args.format}, {}, outputs, args.seed)
    print(f"wrote {', '.join(outputs)} (n={ham.n}, definiteness={ham.definiteness.value})")


def cmd_solve(args) -> None:
    from . import fileio
    from .solver import mirror_largest, solve

    ham, inputs = _load(args)
    cfg = _config(args)
    result = solve(ham, cfg)
    report = mirror_largest(result) if args.largest else result
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    digest = "+".join(inputs[k] for k in sorted(inputs))
    fileio.write_eigenvalues_csv(out / "eigenvalues.csv", report.lambdas, report.residual_norms, digest,
                                 converged=result.converged)
    fileio.write_pchv(out / "eigenvectors.bin", report.v)
    fileio.write_trace_csv(out / "trace.csv", result, digest)
    fileio.write_manifest(out / "manifest.json", "solve",
                          {"nev": cfg.nev, "nex": cfg.nex, "deg": cfg.deg, "tol": cfg.tol, "maxiter": cfg.maxiter,
                           "rr_variant": cfg.rr_variant, "seed": cfg.seed, "lanczos_steps": cfg.lanczos_steps,
                           "rel_res": cfg.rel_res, "reproducible": cfg.reproducible, "largest": args.largest},
                          inputs, ["eigenvalues.csv", "eigenvectors.bin", "trace.csv"], args.seed)
    status = "converged" if result.converged else "NOT converged"
    print(f"{status} in {result.iterations_used} iterations (backup events: {result.backup_events})")


def cmd_bench(args) -> None:
    """Repeat a solve; per repetition and phase seconds, modeled flops, GFLOP/s, then min/avg/max
    summaries -- bench.csv and manifest.json in the reference's format (cli.py:291-361,
    FORMATS.md "bench.csv")."""
    from . import fileio
    from .solver import solve

    ham, inputs = _load(args)
    cfg = _config(args)
    if args.reps < 1:
        raise ValueError_(f"reps must be >= 1, got {args.reps}")
    runs = []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        res = solve(ham, cfg, keep_on_device=True)
        runs.append((res, time.perf_counter() - t0))
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    phases = sorted({ph for r, _ in runs for ph in r.ledger.flops})
    rows = ["# bsesolve bench v1", "# manifest: manifest.json", f"# input_digest: {'+'.join(inputs[k] for k in sorted(inputs))}",
            "rep,phase,seconds,flops,gflops"]
    for rep, (r, wall) in enumerate(runs):
        led = r.ledger
        for ph in phases:
            sec, fl = led.seconds.get(ph, 0.0), led.flops.get(ph, 0.0)
            rows.append(f"{rep},{ph},{sec:.6f},{fl:.0f},{(fl / sec / 1e9) if sec > 0 else 0.0:.3f}")
        rows.append(f"{rep},total,{wall:.6f},{led.total_flops():.0f},{led.total_flops() / wall / 1e9:.3f}")
    echo = []
    for ph in phases + ["total"]:
        if ph == "total":
            secs, fl = [w for _, w in runs], runs[0][0].ledger.total_flops()
        else:
            secs, fl = [r.ledger.seconds.get(ph, 0.0) for r, _ in runs], runs[0][0].ledger.flops.get(ph, 0.0)
        rows.append(f"summary,{ph},{min(secs):.6f}/{sum(secs) / len(secs):.6f}/{max(secs):.6f},{fl:.0f},")
        echo.append(f"{ph:10s} min/avg/max {min(secs):.4f}/{sum(secs) / len(secs):.4f}/{max(secs):.4f} s, "
                    f"modeled {fl / 1e9:.3f} GFLOP")
    (out / "bench.csv").write_text("\n".join(rows) + "\n")
    fileio.write_manifest(out / "manifest.json", "bench",
                          {"nev": cfg.nev, "nex": cfg.nex, "deg": cfg.deg, "tol": cfg.tol, "maxiter": cfg.maxiter,
                           "rr_variant": cfg.rr_variant, "seed": cfg.seed, "reps": args.reps},
                          inputs, ["bench.csv"], args.seed)
    print("\n".join(echo))


def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2601_10557_b200", description=__doc__.splitlines()[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("generate")
    g.add_argument("--m", type=int, required=True)
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("--coupling-ratio", type=float, default=0.5)
    g.add_argument("--alpha", type=float, default=1.0)
    g.add_argument("--mode", choices=["definite", "indefinite"], default="definite")
    g.add_argument("--format", choices=["mm", "pchb"], default="mm")
    g.add_argument("--out", default=".")
    for name in ("solve", "bench"):
        s = sub.add_parser(name)
        s.add_argument("--a")
        s.add_argument("--b")
        s.add_argument("--pchb")
        s.add_argument("--nev", type=int, required=True)
        s.add_argument("--nex", type=int, default=None)
        s.add_argument("--deg", type=int, default=20)
        s.add_argument("--tol", type=float, default=1e-8)
        s.add_argument("--maxiter", type=int, default=25)
        s.add_argument("--rr", choices=["auto", "hermitian", "backup"], default="auto")
        s.add_argument("--seed", type=int, default=0)
        s.add_argument("--lanczos-steps", type=int, default=24)
        s.add_argument("--rel-res", action="store_true")
        s.add_argument("--reproducible", action=argparse.BooleanOptionalAction, default=True)
        s.add_argument("--out", default=".")
        if name == "solve":
            s.add_argument("--largest", action="store_true")
        else:
            s.add_argument("--reps", type=int, default=5)
    return ap


def main(argv=None) -> int:
    from .errors import NumericalError, ValidationError

    args = _parser().parse_args(argv)
    try:
        {"generate": cmd_generate, "solve": cmd_solve, "bench": cmd_bench}[args.cmd](args)
    except ValidationError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_VALIDATION
    except OSError as exc:
        print(f"i/o error: {exc}", file=sys.stderr)
        return EXIT_IO
    except NumericalError as exc:
        print(f"numerical error: {exc}", file=sys.stderr)
        return EXIT_NUMERICAL
    return 0
