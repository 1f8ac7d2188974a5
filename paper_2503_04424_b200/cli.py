"""Command line of the drop-in (the hot-path subcommands of `oocdet`, reference cli.py:1-318).

    python -m paper_2503_04424_b200 memdet --in K.mdm --assume spd --num-blocks 8 --json
    python -m paper_2503_04424_b200 gen --kind rbf --n 4096 --out K.mdm
    python -m paper_2503_04424_b200 cost --m 4096 --nb 4 [--case gen|sym] --json
    python -m paper_2503_04424_b200 flodance --prefix K.pfx --d 1 --n0 5 --ns 3000 --q 1 --predict 4096
    python -m paper_2503_04424_b200 pipeline --kind rbf --n 4096 --out K.mdm --assume spd --ns 3000 --json

Same flags, JSON payload (schema_version 1) and exit codes as the reference: 0 success,
2 usage error, 3 numerical failure, 4 I/O failure.  The SLQ / block-diagonal baselines are
outside this engine's scope; `gen` / `pipeline` generate the
BASELINE families (one output per datapoint, so FLODANCE runs with d = 1 in `pipeline`) instead
of the reference's Matern-LMC generator.
"""

from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

from . import __version__, gen
from .cost import predicted_cost
from .errors import NumericalError, OocdetError, StorageError
from .flodance import fit_prefix, predict, predict_interval, scaling_ratio_trace
from .memdet import memdet_cholesky, memdet_ldl, memdet_lu
from .prefixio import read_prefix
from .storage import write_matrix

SCHEMA_VERSION = 1
_SUFFIXES = {"k": 1 << 10, "m": 1 << 20, "g": 1 << 30}


def parse_size(text: str) -> int:
    """Byte count with an optional K/M/G suffix (powers of 1024), as reference cli.py:35-48."""
    s = text.strip().lower().removesuffix("b")
    mult = 1
    if s and s[-1] in _SUFFIXES:
        mult, s = _SUFFIXES[s[-1]], s[:-1]
    try:
        value = int(float(s) * mult) if "." in s else int(s) * mult
    except ValueError:
        raise argparse.ArgumentTypeError(f"cannot parse size {text!r}") from None
    if value < 0:
        raise argparse.ArgumentTypeError(f"size must be non-negative: {text!r}")
    return value


def _emit(args, payload: dict, lines):
    if args.json:
        json.dump(payload, sys.stdout, sort_keys=True)
        sys.stdout.write("\n")
    else:
        for line in lines:
            print(line)


def cmd_memdet(args) -> int:
    kwargs = dict(max_mem=args.max_mem, num_blocks=args.num_blocks, scratch_dir=args.scratch_dir)
    if args.assume == "gen":  # reference cli.py:81-88
        if args.prefix_out:
            raise ValueError("--prefix-out requires --assume sym or spd")
        res = memdet_lu(args.infile, **kwargs)
    else:
        driver = memdet_cholesky if args.assume == "spd" else memdet_ldl
        res = driver(args.infile, prefix_out=args.prefix_out, **kwargs)
    info = res.info
    payload = {
        "schema_version": SCHEMA_VERSION, "logabsdet": res.logabsdet, "sign": res.sign,
        "n_b": info.n_b, "b": info.b, "blocks_read": info.blocks_read,
        "blocks_written": info.blocks_written, "scratch_slots": info.scratch_slots,
        "wall_seconds": info.wall_seconds,
        "engine": {"device_ms": info.device_ms, "h2d_bytes": info.h2d_bytes,
                   "d2h_bytes": info.d2h_bytes, "kernel_launches": info.kernel_launches,
                   "out_of_core": info.out_of_core, "ooc_blocks": info.ooc_blocks,
                   "ooc_reads": info.ooc_reads, "ooc_writes": info.ooc_writes},
    }
    _emit(args, payload, [
        f"logabsdet = {res.logabsdet:.12e} (sign {res.sign:+d})",
        f"n_b = {info.n_b}, b = {info.b}, reads = {info.blocks_read}, writes = {info.blocks_written}, "
        f"scratch slots = {info.scratch_slots}",
        f"wall time {info.wall_seconds:.3f} s (device {info.device_ms:.1f} ms)",
    ])
    return 0


def _generate(args):
    kinds = {
        "wishart": lambda: (gen.spd_wishart(args.n, args.k or args.n, args.seed, args.jitter or 1e-3), "spd"),
        "rbf": lambda: (gen.rbf(args.n, args.d, args.ell, args.jitter or 1e-6, args.seed), "spd"),
        "ntk-like": lambda: (gen.ntk_like(args.n, args.k or 2 * args.n, args.alpha, args.jitter or 1e-8,
                                          args.seed), "spd"),
        "spd-random": lambda: (gen.random_spd(args.n, args.seed), "spd"),
        "sym-random": lambda: (gen.random_symmetric(args.n, args.seed), "symmetric"),
    }
    a, sym = kinds[args.kind]()
    return write_matrix(args.out, a, sym)


def cmd_gen(args) -> int:
    mf = _generate(args)
    _emit(args, {"schema_version": SCHEMA_VERSION, "path": mf.path, "m": mf.m, "dtype": str(mf.dtype),
                 "symmetry": mf.symmetry, "kind": args.kind, "seed": args.seed},
          [f"wrote {mf.symmetry} {mf.m}x{mf.m} matrix to {mf.path}"])
    return 0


def cmd_cost(args) -> int:
    case = {"gen": "generic", "sym": "symmetric"}[args.case]
    pc = predicted_cost(args.m, args.nb, case)
    def num(x):  # exact counts stay JSON integers (reference cost.py:58-60)
        return int(x) if x.denominator == 1 else float(x)

    ops = {}
    for name in ("decomposition", "lower_solve", "upper_solve", "full_multiply", "gramian_multiply"):
        op = getattr(pc, name)
        ops[name] = {"count": num(op.count), "flops_per_op": num(op.flops_per_op), "total": num(op.total)}
    payload = {"schema_version": SCHEMA_VERSION, "m": pc.m, "n_b": pc.n_b, "b": pc.m // pc.n_b,
               "case": pc.case, "operations": ops, "total_flops": num(pc.total_flops),
               "blocks_read": pc.blocks_read, "blocks_written": pc.blocks_written,
               "scratch_slots": pc.scratch_slots}
    _emit(args, payload, [f"total FMA {float(pc.total_flops):.6g}, reads {pc.blocks_read}, "
                          f"writes {pc.blocks_written}, scratch slots {pc.scratch_slots}"])
    return 0


def cmd_flodance(args) -> int:
    """Fit and extrapolate a prefix sidecar (reference cli.py:107-135)."""
    ell, _ = read_prefix(args.prefix)
    fit = fit_prefix(ell, args.d, args.n0, args.ns, args.q)
    L_hat, ell_hat = predict(fit, args.predict)
    payload = {"schema_version": SCHEMA_VERSION, **fit.to_json_dict(), "n": args.predict,
               "L_hat": float(L_hat), "logdet_hat": float(ell_hat)}
    lines = [f"fit on [{args.n0}, {args.ns}], q = {args.q}: c0 = {fit.c0:.6g}, "
             f"nu = {np.array2string(fit.nu, precision=6)}, sigma_hat = {fit.sigma_hat:.6g}",
             f"L_hat({args.predict}) = {float(L_hat):.12e}",
             f"logdet_hat({args.predict}) = {float(ell_hat):.12e}"]
    if args.interval is not None:
        lo, hi = predict_interval(fit, args.predict, args.interval)
        payload["interval"] = {"level": args.interval, "lower": lo, "upper": hi}
        lines.append(f"{args.interval:.0%} interval [{lo:.12e}, {hi:.12e}]")
    if args.trace_out:
        trace = scaling_ratio_trace(ell, args.d)
        with open(args.trace_out, "w") as f:
            f.write("n,log_ratio\n")
            for n, v in enumerate(trace, start=2):
                f.write(f"{n},{v!r}\n")
        lines.append(f"wrote ratio trace to {args.trace_out}")
    _emit(args, payload, lines)
    return 0


def cmd_pipeline(args) -> int:
    """Generate, factor on the B200 engine, fit and extrapolate (reference cli.py:169-199)."""
    started = time.perf_counter()
    inputs = {"kind": args.kind, "n": args.n, "k": args.k, "d": args.d, "ell": args.ell, "alpha": args.alpha,
              "seed": args.seed, "jitter": args.jitter}
    mf = _generate(args)
    driver = memdet_cholesky if args.assume == "spd" else memdet_ldl
    res = driver(mf, max_mem=args.max_mem, num_blocks=args.num_blocks, scratch_dir=args.scratch_dir)
    truth = res.logabsdet
    fit = fit_prefix(res.prefix, 1, args.n0, args.ns, args.q)
    _, ell_hat = predict(fit, args.n)
    rel_error = abs(float(ell_hat) - truth) / max(1.0, abs(truth))
    outputs = {
        "matrix": {"path": mf.path, "m": mf.m, "symmetry": mf.symmetry},
        "memdet": {"logabsdet": truth, "sign": res.sign, **res.info.to_json_dict()},
        "flodance": {**fit.to_json_dict(), "n": args.n, "logdet_hat": float(ell_hat)},
        "rel_error": rel_error,
    }
    payload = {"schema_version": SCHEMA_VERSION, "command": "pipeline", "inputs": inputs, "outputs": outputs,
               "timing": {"wall_seconds": time.perf_counter() - started}}
    _emit(args, payload, [f"generated {mf.m}x{mf.m} {args.kind} matrix",
                          f"memdet logabsdet = {truth:.12e}",
                          f"extrapolated logdet_hat({args.n}) = {float(ell_hat):.12e}",
                          f"relative error = {rel_error:.3e}"])
    return 0


def _add_gen_args(p):
    p.add_argument("--kind", default="rbf", choices=("wishart", "rbf", "ntk-like", "spd-random", "sym-random"))
    p.add_argument("--n", type=int, required=True)
    p.add_argument("--k", type=int, default=None, help="inner dimension (wishart / ntk-like)")
    p.add_argument("--d", type=int, default=16, help="RBF point dimension")
    p.add_argument("--ell", type=float, default=4.0, help="RBF length scale")
    p.add_argument("--alpha", type=float, default=0.75, help="NTK-like power-law exponent")
    p.add_argument("--jitter", type=float, default=None)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out", required=True)


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_2503_04424_b200",
                                     description="B200 MEMDET log-determinants (drop-in for oocdet memdet)")
    parser.add_argument("--version", action="version", version=__version__)
    sub = parser.add_subparsers(dest="command", required=True)

    p = sub.add_parser("memdet", help="exact log-determinant and prefixes on the B200 engine")
    p.add_argument("--in", dest="infile", required=True)
    p.add_argument("--assume", choices=("gen", "sym", "spd"), required=True)
    p.add_argument("--max-mem", type=parse_size, default=None)
    p.add_argument("--num-blocks", type=int, default=None)
    p.add_argument("--scratch-dir", default=None)
    p.add_argument("--prefix-out", default=None)
    p.add_argument("--json", action="store_true")
    p.set_defaults(func=cmd_memdet)

    p = sub.add_parser("gen", help="write a seeded BASELINE-family matrix (MEMDET01)")
    _add_gen_args(p)
    p.add_argument("--json", action="store_true")
    p.set_defaults(func=cmd_gen)

    p = sub.add_parser("cost", help="analytical cost model query")
    p.add_argument("--m", type=int, required=True)
    p.add_argument("--nb", type=int, required=True)
    p.add_argument("--case", choices=("gen", "sym"), default="gen")  # reference cli.py:276-279
    p.add_argument("--json", action="store_true")
    p.set_defaults(func=cmd_cost)

    p = sub.add_parser("flodance", help="fit and extrapolate a prefix sequence")
    p.add_argument("--prefix", required=True, help="prefix sidecar file")
    p.add_argument("--d", type=int, required=True)
    p.add_argument("--n0", type=int, required=True, help="burn-in start")
    p.add_argument("--ns", type=int, required=True, help="fit window end")
    p.add_argument("--q", type=int, required=True, help="exponent correction order")
    p.add_argument("--predict", type=int, required=True, metavar="N")
    p.add_argument("--interval", type=float, default=None, metavar="LEVEL")
    p.add_argument("--trace-out", default=None, help="write the determinant-ratio trace as CSV")
    p.add_argument("--json", action="store_true")
    p.set_defaults(func=cmd_flodance)

    p = sub.add_parser("pipeline", help="generate, factorize on the B200 engine, fit, and extrapolate")
    _add_gen_args(p)
    p.add_argument("--assume", choices=("sym", "spd"), default="sym")
    p.add_argument("--max-mem", type=parse_size, default=None)
    p.add_argument("--num-blocks", type=int, default=None)
    p.add_argument("--scratch-dir", default=None)
    p.add_argument("--n0", type=int, default=1)
    p.add_argument("--ns", type=int, required=True)
    p.add_argument("--q", type=int, default=0)
    p.add_argument("--json", action="store_true")
    p.set_defaults(func=cmd_pipeline)
    return parser


def main(argv=None) -> int:
    """Exit codes as reference cli.py:298-314."""
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (ValueError, argparse.ArgumentTypeError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except NumericalError as exc:
        print(f"numerical failure: {exc}", file=sys.stderr)
        return 3
    except (StorageError, OSError) as exc:
        print(f"I/O failure: {exc}", file=sys.stderr)
        return 4
    except OocdetError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return exc.exit_code


if __name__ == "__main__":
    sys.exit(main())
