"""``python -m paper_2307_14774_b200 bench --device cuda ...`` -- the GPU form of
the reference's ``spc5 bench`` command (cli.py:155-185).

Same loop and output as the reference command -- validate, then time, one
line per record, CSV v1 records plus the scatter companion -- with the
products on the GPU (``run_bench`` -> K1/K2 through the C ABI) and a second
CSV holding the roofline fields per record.  Matrices are the synthetic specs
of the reference CLI (``dense:N``, ``identity:N``,
``random:rows,cols,nnz_per_row,clustering,seed``) plus ``config:N[:LO-HI]`` for
the seeded BASELINE workloads (optionally a row slice); Matrix Market files and the SuiteSparse fetch are
out of scope.  Only ``--device cuda`` exists: there is no CPU path.
"""

from __future__ import annotations

import argparse
import os
import sys

from .blocks import VALID_R, VALID_VS
from .harness import (ValidationError, gpu_record, run_bench, write_gpu_records, write_records,
                      write_scatter)
from .kernels import KernelConfig

_STRATEGIES = ("scalar", "expand", "compact")
_REDUCTIONS = ("hsum", "multi")
_X_LOADS = ("partial", "single")


def _formats(text: str) -> list[int]:
    out = []
    for tok in text.split(","):
        tok = tok.strip().lower()
        if not tok.startswith("b") or not tok[1:].isdigit() or int(tok[1:]) not in VALID_R:
            raise argparse.ArgumentTypeError(
                f"bad format {tok!r}; expected a comma list from b1,b2,b4,b8")
        out.append(int(tok[1:]))
    return out


def _choices(allowed, what):
    def parse(text: str) -> list[str]:
        if text == "all":
            return list(allowed)
        out = [t.strip() for t in text.split(",")]
        for t in out:
            if t not in allowed:
                raise argparse.ArgumentTypeError(
                    f"bad {what} {t!r}; expected 'all' or a comma list from {allowed}")
        return out
    return parse


def load_matrix(spec: str, precision: str):
    """(label, CsrMatrix) for a synthetic spec of the reference CLI or config:N."""
    from .mmio import make_dense, make_identity, make_random
    kind, _, arg = spec.partition(":")
    if kind == "dense":
        return spec, make_dense(int(arg), precision)
    if kind == "identity":
        return spec, make_identity(int(arg), precision)
    if kind == "random":
        rows, cols, per_row, clustering, seed = arg.split(",")
        return spec, make_random(int(rows), int(cols), int(per_row), float(clustering), int(seed),
                                 precision)
    if kind == "config":  # config:N or config:N:LO-HI (a row slice of the seeded workload)
        from . import workloads
        num, _, rng = arg.partition(":")
        cfg = workloads.CONFIGS[int(num)]
        if cfg["precision"] != precision:
            raise ValueError(f"config {num} is {cfg['precision']}; pass --precision {cfg['precision']}")
        if int(num) == 1:
            return cfg["name"], workloads.config1()
        rows, _ = workloads.config_shape(cfg)
        lo, hi = (int(v) for v in rng.split("-")) if rng else (0, rows)
        return f"{cfg['name']}[{lo}:{hi}]", workloads.host_rows(cfg, lo, min(hi, rows))
    raise ValueError(f"unsupported matrix spec {spec!r} (dense:N, identity:N, random:..., config:N)")


def cmd_bench(args) -> int:
    if args.device != "cuda":
        print("error: only --device cuda exists (no CPU path)", file=sys.stderr)
        return 2
    label, m = load_matrix(args.matrix, args.precision)
    vs = args.vs or (8 if args.precision == "f64" else 16)
    from .blocks import csr_to_spc5
    peak = args.peak_gbs
    records, gpu_records, status = [], [], 0
    for r in args.format:
        s = csr_to_spc5(m, r, vs)  # for the roofline fields (run_bench converts its own)
        for strategy in args.strategy:
            for reduction in args.reduction:
                for x_load in args.xload:
                    cfg = KernelConfig(strategy=strategy, reduction=reduction, x_load=x_load,
                                       precision=args.precision)
                    try:
                        rec = run_bench(label, m, r, vs, cfg, workers=args.threads,
                                        reps=args.reps, warmup=args.warmup, seed=args.seed)
                    except ValidationError as exc:
                        print(f"error: validation failed, not timing: {exc}", file=sys.stderr)
                        status = 1
                        continue
                    g = gpu_record(rec, s, peak)
                    records.append(rec)
                    gpu_records.append(g)
                    print(f"{rec.matrix},{rec.precision},b{rec.r},vs={rec.vs},"
                          f"{rec.strategy}/{rec.reduction}/{rec.x_load},"
                          f"workers={rec.workers},median={rec.median_seconds:.3e}s,"
                          f"gflops={rec.gflops:.4f},filling={rec.filling:.4f},"
                          f"gbs={g.achieved_gbs:.1f},roofline={g.roofline_frac:.3f}")
    if args.out:
        write_records(args.out, records)
        stem = os.path.splitext(args.out)[0]
        write_scatter(stem + ".scatter.csv", records)
        write_gpu_records(stem + ".gpu.csv", gpu_records)
        print(f"wrote {len(records)} records to {args.out}, {stem}.scatter.csv and {stem}.gpu.csv")
    return status


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="python -m paper_2307_14774_b200")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("bench", help="time the GPU kernels and emit CSV records")
    p.add_argument("--device", default="cuda", help="only 'cuda'")
    p.add_argument("--matrix", required=True,
                   help="dense:N | identity:N | random:rows,cols,nnz_per_row,clustering,seed | "
                        "config:N[:LO-HI]")
    p.add_argument("--precision", choices=("f32", "f64"), default="f64")
    p.add_argument("--format", type=_formats, default=list(VALID_R))
    p.add_argument("--vs", type=int, choices=VALID_VS, default=None)
    p.add_argument("--strategy", type=_choices(_STRATEGIES, "strategy"), default=["expand"])
    p.add_argument("--reduction", type=_choices(_REDUCTIONS, "reduction"), default=["hsum"])
    p.add_argument("--xload", type=_choices(_X_LOADS, "x_load"), default=["partial"])
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--threads", type=int, default=int(os.environ.get("SPC5_THREADS", "1")),
                   help="workers of spmv_parallel (concurrent panel-range launches)")
    p.add_argument("--reps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--out", default=None, help="CSV output path")
    p.add_argument("--peak-gbs", type=float, default=_default_peak(),
                   help="HBM peak for the roofline column (default: MEASURED_PEAKS.json, else 6500)")
    p.set_defaults(func=cmd_bench)
    return parser


def _default_peak() -> float:
    import json
    from pathlib import Path
    f = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(f.read_text())["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6500.0


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    return args.func(args)


if __name__ == "__main__":
    sys.exit(main())
