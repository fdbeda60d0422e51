"""Timing harness: ``run_kernel`` / ``run_bench`` of the reference (bench.py:140-184).

Same protocol -- convert, verify against the exact oracle (refuse to time on
failure, bench.py:163-167), warm up, take the median of the repetitions,
GFLOP/s = 2*nnz/median (bench.py:183) -- with the GPU timed by CUDA events on
the launching stream (device arrays, no host copies in the timed region).
``run_kernel`` keeps the reference's host-clock semantics for drop-in callers.
"""

from __future__ import annotations

import csv
import io
import statistics
import time
from dataclasses import dataclass
from dataclasses import fields as dataclass_fields
from pathlib import Path

import numpy as np

from .blocks import csr_to_spc5, filling_stats
from .kernels import (KernelConfig, SpmvResult, spmv_spc5_scalar, spmv_spc5_vector,
                      verify_against_oracle)
from .parallel import spmv_parallel

__all__ = ["BenchRecord", "CostModelFit", "CSV_VERSION_LINE", "GpuRecord", "InsufficientDataError",
           "ValidationError", "fit_cost_model", "gpu_record", "read_records", "run_bench",
           "run_kernel", "spearman_rank_correlation", "time_device_spmv", "write_gpu_records",
           "write_records", "write_scatter"]

# Schema line of the reference's CSV v1 (bench.py:43).  Records written here
# parse with the reference's read_records and vice versa; GPU-only fields go to
# a companion file (write_gpu_records) so the v1 columns stay unchanged.
CSV_VERSION_LINE = "# spc5 bench csv v1 (fma=unfused, tree=adjacent-pair, numa=none)"


class ValidationError(RuntimeError):
    """A kernel failed oracle verification; its timings would be meaningless."""


class InsufficientDataError(ValueError):
    """A (r, vs, precision) group has too few records for the cost fit (bench.py:206-213)."""


@dataclass
class BenchRecord:
    """One measurement row (bench.py:54-79 fields)."""

    matrix: str
    precision: str
    r: int
    vs: int
    strategy: str
    reduction: str
    x_load: str
    workers: int
    reps: int
    median_seconds: float
    gflops: float
    filling: float
    num_blocks: int

    @property
    def nnz(self) -> int:
        return round(self.filling * self.num_blocks * self.r * self.vs)

    @property
    def avg_nnz_per_block(self) -> float:
        return self.filling * self.r * self.vs


def run_kernel(s, x, y, cfg: KernelConfig, workers: int = 1) -> SpmvResult:
    """One SpMV (bench.py:140-150): parallel only when more than one worker is asked."""
    if workers > 1:
        return spmv_parallel(s, x, y, cfg, workers)
    t0 = time.perf_counter()
    if cfg.strategy == "scalar":
        spmv_spc5_scalar(s, x, y)
    else:
        spmv_spc5_vector(s, x, y, cfg)
    return SpmvResult(y=y, flops=2 * s.nnz, elapsed=time.perf_counter() - t0)


def time_device_spmv(s, reps: int = 100, warmup: int = 20, seed: int = 0,
                     flush_bytes: int = 0) -> list[float]:
    """Per-launch device times (s) of y = A.x with x, y resident, CUDA events on the stream."""
    import torch

    from . import _native as nat
    from .blocks import torch_stream
    h = s.handle()
    tdt = torch.float64 if s.dtype == np.float64 else torch.float32
    rng = np.random.default_rng(seed)
    x = torch.from_numpy(rng.uniform(-1, 1, s.num_cols).astype(s.dtype)).to("cuda", tdt)
    y = torch.zeros(s.num_rows, dtype=tdt, device="cuda")
    flush = torch.empty(flush_bytes // 4, dtype=torch.int32, device="cuda") if flush_bytes else None
    times = []
    for i in range(warmup + reps):
        if flush is not None:
            flush.fill_(i)
        st = torch_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        nat.check(nat.lib.spc5_spmv(h.ptr, x.data_ptr(), y.data_ptr(), 0, st))
        e1.record()
        e1.synchronize()
        if i >= warmup:
            times.append(e0.elapsed_time(e1) * 1e-3)
    return times


def run_bench(label: str, m, r: int, vs: int, cfg: KernelConfig, workers: int = 1,
              reps: int = 10, warmup: int = 3, seed: int = 0) -> BenchRecord:
    """Validate, then time: median device time of ``reps`` products (bench.py:153-184)."""
    s = csr_to_spc5(m, r, vs)
    report = verify_against_oracle(m, r, vs, cfg, trials=1, seed=seed, spc5=s)
    if not report.passed:
        raise ValidationError(
            f"{label} r={r} vs={vs} {cfg.strategy}/{cfg.reduction}/{cfg.x_load}: {report}")
    if workers > 1:
        rng = np.random.default_rng(seed)
        x = rng.uniform(-1.0, 1.0, size=m.num_cols).astype(m.values.dtype)
        times = []
        for i in range(warmup + reps):
            y = np.zeros(m.num_rows, dtype=m.values.dtype)
            res = run_kernel(s, x, y, cfg, workers)
            if i >= warmup:
                times.append(res.elapsed)
    else:
        times = time_device_spmv(s, reps=reps, warmup=warmup, seed=seed)
    median = statistics.median(times)
    st = filling_stats(s)
    return BenchRecord(matrix=label, precision=cfg.precision, r=r, vs=vs,
                       strategy=cfg.strategy, reduction=cfg.reduction, x_load=cfg.x_load,
                       workers=workers, reps=reps, median_seconds=median,
                       gflops=2 * m.nnz / median / 1e9, filling=st.filling,
                       num_blocks=st.num_blocks)


# ---------------------------------------------------------------- CSV records
_INTS = ("r", "vs", "workers", "reps", "num_blocks")
_FLOATS = ("median_seconds", "gflops", "filling")


def _columns() -> list[str]:
    return [f.name for f in dataclass_fields(BenchRecord)]


def _cell(name: str, v) -> str:
    # floats as shortest round-trip repr: a parsed file is field-identical
    return repr(float(v)) if name in _FLOATS else str(v)


def _write_csv(path, head: str, columns, rows) -> None:
    buf = io.StringIO()
    buf.write(head + "\n")
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(columns)
    w.writerows(rows)
    Path(path).write_text(buf.getvalue(), encoding="utf-8")


def write_records(path, records) -> None:
    """CSV v1 (bench.py:86-96): version line, header, one row per record."""
    cols = _columns()
    _write_csv(path, CSV_VERSION_LINE, cols,
               ([_cell(c, getattr(rec, c)) for c in cols] for rec in records))


def write_scatter(path, records) -> None:
    """Plot-ready companion (bench.py:99-108): GFLOP/s against entries per block."""
    _write_csv(path, "# spc5 bench scatter v1",
               ["matrix", "precision", "r", "vs", "avg_nnz_per_block", "gflops"],
               ([rec.matrix, rec.precision, rec.r, rec.vs, repr(rec.avg_nnz_per_block),
                 repr(rec.gflops)] for rec in records))


def read_records(path) -> list[BenchRecord]:
    """Parse a CSV v1 file (bench.py:111-137); ValueError on a foreign header or row."""
    cols = _columns()
    body = [ln for ln in Path(path).read_text(encoding="utf-8").splitlines()
            if ln.strip() and not ln.startswith("#")]
    out: list[BenchRecord] = []
    rows = csv.reader(body)
    head = next(rows, None)
    if head is None:
        return out
    if head != cols:
        raise ValueError(f"unexpected CSV header {head}")
    for cells in rows:
        if len(cells) != len(cols):
            raise ValueError(f"row has {len(cells)} cells, expected {len(cols)}")
        kw = {}
        for c, v in zip(cols, cells):
            kw[c] = int(v) if c in _INTS else float(v) if c in _FLOATS else v
        out.append(BenchRecord(**kw))
    return out


@dataclass
class GpuRecord:
    """GPU fields of one measurement (companion of a BenchRecord, same order)."""

    matrix: str
    r: int
    vs: int
    device: str
    median_us: float
    alg_bytes: int
    achieved_gbs: float
    peak_gbs: float
    roofline_frac: float


def gpu_record(rec: BenchRecord, s, peak_gbs: float, device: str = "cuda:0") -> GpuRecord:
    """Roofline fields for ``rec``: algorithmic bytes = footprint + x + y."""
    vb = np.dtype(s.dtype).itemsize
    alg = filling_stats(s).footprint_bytes + vb * (s.num_cols + s.num_rows)
    gbs = alg / rec.median_seconds / 1e9
    return GpuRecord(matrix=rec.matrix, r=rec.r, vs=rec.vs, device=device,
                     median_us=rec.median_seconds * 1e6, alg_bytes=int(alg), achieved_gbs=gbs,
                     peak_gbs=float(peak_gbs), roofline_frac=gbs / peak_gbs)


def write_gpu_records(path, records) -> None:
    cols = [f.name for f in dataclass_fields(GpuRecord)]
    _write_csv(path, "# spc5 bench gpu v1", cols,
               ([repr(v) if isinstance(v, float) else str(v)
                 for v in (getattr(g, c) for c in cols)] for g in records))


# ----------------------------------------------------------- per-block cost fit
@dataclass
class CostModelFit:
    """time = cost_per_block * num_blocks, least squares through 0 (bench.py:187-197)."""

    cost_per_block_seconds: float
    r_squared: float

    @property
    def constant_cost(self) -> bool:
        return self.r_squared >= 0.9


def fit_cost_model(records, min_records: int = 5) -> dict:
    """Per (r, vs, precision) group fit of median time on num_blocks (bench.py:200-224).

    On the GPU the time per block is the quantity the roofline explains: a
    group whose fit is not ``constant_cost`` is one whose blocks cost different
    amounts (filling, x locality), which the per-config table shows.
    """
    groups: dict = {}
    for rec in records:
        groups.setdefault((rec.r, rec.vs, rec.precision), []).append(rec)
    short = sorted(k for k, v in groups.items() if len(v) < min_records)
    if short:
        raise InsufficientDataError(
            "insufficient data: need >= %d records per group; " % min_records
            + ", ".join(f"r={k[0]} vs={k[1]} {k[2]} ({len(groups[k])} records)" for k in short))
    fits = {}
    for key, recs in groups.items():
        nb = np.array([rec.num_blocks for rec in recs], dtype=np.float64)
        t = np.array([rec.median_seconds for rec in recs], dtype=np.float64)
        den = float(nb @ nb)
        a = float(nb @ t) / den if den > 0 else 0.0
        res = float(((t - a * nb) ** 2).sum())
        tot = float(((t - t.mean()) ** 2).sum())
        r2 = 1.0 - res / tot if tot > 0 else (1.0 if res == 0.0 else 0.0)
        fits[key] = CostModelFit(cost_per_block_seconds=a, r_squared=r2)
    return fits


def _ranks(v) -> np.ndarray:
    v = np.asarray(v, dtype=np.float64)
    order = np.argsort(v, kind="stable")
    rk = np.empty(len(v))
    rk[order] = np.arange(len(v), dtype=np.float64)
    u, inv, cnt = np.unique(v, return_inverse=True, return_counts=True)
    if len(u) != len(v):  # ties share their mean rank
        sums = np.bincount(inv, weights=rk, minlength=len(u))
        rk = (sums / cnt)[inv]
    return rk


def spearman_rank_correlation(a, b) -> float:
    """Rank correlation with average ranks for ties (bench.py:227-248)."""
    ra, rb = _ranks(a), _ranks(b)
    ra -= ra.mean()
    rb -= rb.mean()
    den = float(np.sqrt((ra @ ra) * (rb @ rb)))
    return float(ra @ rb / den) if den else 0.0
