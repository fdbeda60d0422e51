"""Timing harness: ``run_kernel`` / ``run_bench`` of the reference (bench.py:140-184).

Same protocol -- convert, verify against the exact oracle (refuse to time on
failure, bench.py:163-167), warm up, take the median of the repetitions,
GFLOP/s = 2*nnz/median (bench.py:183) -- with the GPU timed by CUDA events on
the launching stream (device arrays, no host copies in the timed region).
``run_kernel`` keeps the reference's host-clock semantics for drop-in callers.
"""

from __future__ import annotations

import statistics
import time
from dataclasses import dataclass

import numpy as np

from .blocks import csr_to_spc5, filling_stats
from .kernels import (KernelConfig, SpmvResult, spmv_spc5_scalar, spmv_spc5_vector,
                      verify_against_oracle)
from .parallel import spmv_parallel

__all__ = ["BenchRecord", "ValidationError", "run_kernel", "run_bench", "time_device_spmv"]


class ValidationError(RuntimeError):
    """A kernel failed oracle verification; its timings would be meaningless."""


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
