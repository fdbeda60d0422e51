"""``python -m paper_2307_14774_b200 bench --device cuda ...`` -- the GPU form of
the reference's ``spc5 bench`` command (cli.py:155-185), plus its
``stats`` (cli.py:81-111), ``verify`` (cli.py:130-152, with the mask
fault-injection self-test) and ``fit`` (cli.py:188-199) commands over the same
GPU functions.

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


def cmd_stats(args) -> int:
    """Dimensions, NNZ and block filling per matrix and format (cli.py:81-111)."""
    from .blocks import csr_to_spc5, filling_stats
    columns = []
    if args.precision in ("f64", "both"):
        columns.append(("f64", args.vs or 8))
    if args.precision in ("f32", "both"):
        columns.append(("f32", args.vs or 16))
    tag = "|".join(p for p, _ in columns)
    print(f"{'matrix':24s} {'dim':>10s} {'nnz':>12s} {'nnz/row':>10s}  "
          + "  ".join(f"{'b' + str(r) + ' ' + tag:>12s}" for r in args.format))
    status = 0
    for spec in args.matrix:
        try:
            label, m = load_matrix(spec, "f64")  # filling is structural
        except Exception as exc:  # noqa: BLE001  (one bad spec must not stop the table)
            print(f"{spec:24s} error: {exc}", file=sys.stderr)
            status = 1
            continue
        dim = str(m.num_rows) if m.num_rows == m.num_cols else f"{m.num_rows}x{m.num_cols}"
        per_row = m.nnz / m.num_rows if m.num_rows else 0.0
        cells = ["|".join(f"{filling_stats(csr_to_spc5(m, r, vs)).filling * 100:.0f}%"
                          for _, vs in columns).rjust(12) for r in args.format]
        print(f"{label:24s} {dim:>10s} {m.nnz:>12d} {per_row:>10.4g}  " + "  ".join(cells))
    return status


def corrupt_one_mask(s, slot: int) -> None:
    """Fault injection for `verify`: starting at row mask `slot` (cyclic), take the
    first mask that is neither empty nor full and move its lowest set bit to its
    lowest clear lane, so every popcount survives but one value is paired with
    the wrong x entry; if there is no such mask, shift the first block's column."""
    import numpy as np
    masks = s.block_masks
    full = (1 << s.vs) - 1
    v = np.asarray(masks).astype(np.int64)
    cand = np.flatnonzero((v != 0) & (v != full))
    if cand.size == 0:
        s.block_colidx[0] += 1
        return
    n = len(v)
    i = int(cand[np.argmin((cand - slot % n) % n)])
    mask = int(v[i])
    low_set = mask & -mask
    low_clear = ~mask & (mask + 1) & full
    if low_clear == 0:  # the clear lanes are all below the set ones
        low_clear = 1 << ((~mask & full).bit_length() - 1)
    masks[i] = mask ^ low_set ^ low_clear


def cmd_verify(args) -> int:
    """Every kernel config against the exact oracle (cli.py:130-152)."""
    from .blocks import csr_to_spc5
    from .kernels import verify_against_oracle
    label, m = load_matrix(args.matrix, args.precision)
    vs = args.vs or (8 if args.precision == "f64" else 16)
    failures = 0
    for r in args.format:
        s = csr_to_spc5(m, r, vs)
        if args.inject_mask_corruption is not None:
            corrupt_one_mask(s, args.inject_mask_corruption)
        for strategy in args.strategy:
            for reduction in args.reduction:
                for x_load in args.xload:
                    cfg = KernelConfig(strategy=strategy, reduction=reduction, x_load=x_load,
                                       precision=args.precision)
                    try:
                        report = verify_against_oracle(m, r, vs, cfg, trials=args.trials,
                                                       seed=args.seed, spc5=s)
                        ok, text = report.passed, str(report)
                    except (ValueError, RuntimeError, IndexError) as exc:
                        # the library validates structure before a product: a
                        # corrupted mask may already be refused there
                        ok, text = False, f"refused: {exc}"
                    print(f"{label} r={r} vs={vs} {strategy}/{reduction}/{x_load}: {text}")
                    failures += 0 if ok else 1
    if failures:
        print(f"{failures} configuration(s) failed", file=sys.stderr)
        return 1
    return 0


def cmd_fit(args) -> int:
    """Per-block cost model from bench records (cli.py:188-199)."""
    from .harness import InsufficientDataError, fit_cost_model, read_records
    try:
        fits = fit_cost_model(read_records(args.csv), min_records=args.min_records)
    except InsufficientDataError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    for (r, vs, precision), fit in sorted(fits.items()):
        flag = "constant-cost" if fit.constant_cost else "NOT constant-cost (R2 < 0.9)"
        print(f"r={r} vs={vs} {precision}: cost/block = {fit.cost_per_block_seconds:.3e} s, "
              f"R2 = {fit.r_squared:.4f}  [{flag}]")
    return 0


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

    ps = sub.add_parser("stats", help="per-matrix dimensions, NNZ and block filling")
    ps.add_argument("--matrix", action="append", required=True)
    ps.add_argument("--format", type=_formats, default=list(VALID_R))
    ps.add_argument("--precision", choices=("f32", "f64", "both"), default="both")
    ps.add_argument("--vs", type=int, choices=VALID_VS, default=None)
    ps.set_defaults(func=cmd_stats)

    pv = sub.add_parser("verify", help="check every kernel config against the exact oracle")
    pv.add_argument("--matrix", required=True)
    pv.add_argument("--precision", choices=("f32", "f64"), default="f64")
    pv.add_argument("--format", type=_formats, default=list(VALID_R))
    pv.add_argument("--vs", type=int, choices=VALID_VS, default=None)
    pv.add_argument("--strategy", type=_choices(_STRATEGIES, "strategy"), default=list(_STRATEGIES))
    pv.add_argument("--reduction", type=_choices(_REDUCTIONS, "reduction"), default=list(_REDUCTIONS))
    pv.add_argument("--xload", type=_choices(_X_LOADS, "x_load"), default=list(_X_LOADS))
    pv.add_argument("--seed", type=int, default=0)
    pv.add_argument("--trials", type=int, default=3)
    pv.add_argument("--inject-mask-corruption", type=int, default=None, metavar="SLOT",
                    help="fault-injection self-test: corrupt a mask before verifying")
    pv.set_defaults(func=cmd_verify)

    pf = sub.add_parser("fit", help="fit the per-block cost model from bench CSV")
    pf.add_argument("csv")
    pf.add_argument("--min-records", type=int, default=5)
    pf.set_defaults(func=cmd_fit)
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
