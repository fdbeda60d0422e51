"""nnz-balanced panel partition and the partitioned product (parallel.py:1-92).

``partition_by_nnz`` returns exactly the reference's ranges (the greedy prefix
split of parallel.py:31-52), computed on the device from the per-tile
popcount prefix.  ``spmv_parallel`` runs one K2 launch per range, each on its
own CUDA stream -- the GPU analogue of the reference's thread pool -- into
disjoint y rows; because K2 sums every panel in an order fixed by global block
positions, the result is bitwise equal to the single-launch product for any
worker count (the property tests/test_parallel.py:67-108 checks).
Multi-GPU row-panel sharding over NCCL lives in :mod:`.distributed`.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .blocks import as_spc5, torch_stream
from .kernels import KernelConfig, SpmvResult, _check_xy

__all__ = ["Partition", "partition_by_nnz", "spmv_parallel"]


@dataclass
class Partition:
    """Contiguous, disjoint panel ranges covering the matrix, one per worker."""

    ranges: list[tuple[int, int]]


def partition_by_nnz(s, workers: int) -> Partition:
    """Greedy prefix split: each share lands within one panel's nnz of the ideal."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    s = as_spc5(s)
    h = s.handle()
    out = np.zeros(2 * workers, dtype=np.int64)
    nat.check(nat.lib.spc5_partition_by_nnz(h.ptr, workers, out.ctypes.data, torch_stream()))
    return Partition(ranges=[(int(out[2 * k]), int(out[2 * k + 1])) for k in range(workers)])


def spmv_parallel(m, x, y, cfg: KernelConfig, workers: int) -> SpmvResult:
    """y[:num_rows] += A.x with panels divided among ``workers`` concurrent launches."""
    import torch
    m = as_spc5(m)
    if m.dtype != cfg.dtype:
        raise ValueError(f"matrix is {m.precision} but config asks for {cfg.precision}")
    _check_xy(m.num_rows, m.num_cols, x, y)
    part = partition_by_nnz(m, workers)
    h = m.handle()
    tdt = torch.float64 if m.dtype == np.float64 else torch.float32
    t0 = time.perf_counter()
    xd = torch.as_tensor(np.ascontiguousarray(np.asarray(x)[:m.num_cols], dtype=m.dtype)).to(
        "cuda", tdt) if not torch.is_tensor(x) else x.to("cuda", tdt).contiguous()
    yd = torch.as_tensor(np.ascontiguousarray(np.asarray(y)[:m.num_rows], dtype=m.dtype)).to(
        "cuda", tdt) if not torch.is_tensor(y) else y[:m.num_rows].to("cuda", tdt).contiguous()
    main = torch.cuda.current_stream()
    live = [(lo, hi) for lo, hi in part.ranges if hi > lo]
    streams = [torch.cuda.Stream() for _ in live]
    for (lo, hi), st in zip(live, streams):
        st.wait_stream(main)
        nat.check(nat.lib.spc5_spmv_panels(h.ptr, lo, hi, xd.data_ptr(), yd.data_ptr(), 1,
                                           int(st.cuda_stream)))
    for st in streams:
        main.wait_stream(st)
    if torch.is_tensor(y):
        y[:m.num_rows] = yd.to(y.device, y.dtype)
    else:
        y[:m.num_rows] = yd.cpu().numpy()
    elapsed = time.perf_counter() - t0
    return SpmvResult(y=y, flops=2 * m.nnz, elapsed=elapsed)
