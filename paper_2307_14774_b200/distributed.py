"""Row-panel sharding of one SPC5 product over several GPUs.

The reference parallelises with a thread pool over contiguous, nnz-balanced
panel ranges (parallel.py:31-92).  Here the same ranges become ranks of one
process group (one process per GPU, torch.distributed with NCCL over
NVLink/NVSwitch):

* ``panel_partition`` reproduces ``partition_by_nnz`` (parallel.py:31-52)
  from the CSR row pointers alone -- the nnz of a panel is the nnz of its
  rows -- so every rank derives identical ranges without converting or
  owning the global matrix.
* each rank converts only its own rows (K1 on the device); the shard's block
  array equals the global conversion's slice bit for bit (conversion is
  panel-local), and ``block_base`` keeps the warp windows on the global grid.
* iterated products (BASELINE config 5): the local K2 writes its y-slice
  straight into the next x buffer, then an all-gather of the unequal slices
  (one broadcast per owner rank, batched) fills the rest and the buffers swap.

The local product is a callable so the host logic is testable on CPU with the
gloo backend (tests/test_distributed.py); on GPUs it is the C-ABI SpMV.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

__all__ = ["panel_partition", "ShardLayout", "shard_layout", "allgather_slices",
           "iterate_products", "bench_distributed"]


def panel_partition(row_ptr, r: int, workers: int) -> list[tuple[int, int]]:
    """partition_by_nnz (parallel.py:31-52) computed from CSR row pointers.

    cum[p] = nnz of panels 0..p = row_ptr[min((p+1)*r, n)]; boundary_k =
    searchsorted(cum, total*k/P, 'left') + 1, clamped to num_panels.  Works on
    numpy arrays or torch tensors (device searchsorted for 64M-row matrices).
    """
    if workers < 1:
        raise ValueError("workers must be >= 1")
    n = len(row_ptr) - 1
    num_panels = (n + r - 1) // r
    if num_panels == 0:
        return [(0, 0)] * workers
    if type(row_ptr).__module__.startswith("torch"):  # torch tensor (device search)
        import torch
        idx = torch.clamp((torch.arange(num_panels, device=row_ptr.device) + 1) * r, max=n)
        cum = row_ptr[idx].to(torch.float64)
        total = int(row_ptr[n])
        targets = torch.tensor([total * k / workers for k in range(1, workers)],
                               dtype=torch.float64, device=row_ptr.device)
        pos = torch.searchsorted(cum, targets, right=False).cpu().numpy() if workers > 1 else []
    else:
        rp = np.asarray(row_ptr, dtype=np.int64)
        idx = np.minimum((np.arange(num_panels, dtype=np.int64) + 1) * r, n)
        cum = rp[idx].astype(np.float64)
        total = int(rp[n])
        targets = np.array([total * k / workers for k in range(1, workers)], dtype=np.float64)
        pos = np.searchsorted(cum, targets, side="left")
    bounds = [0]
    for k in range(1, workers):
        target = total * k / workers
        bounds.append(0 if target <= 0 else int(pos[k - 1]) + 1)
    bounds.append(num_panels)
    bounds = [min(b, num_panels) for b in bounds]
    return [(bounds[i], bounds[i + 1]) for i in range(workers)]


@dataclass
class ShardLayout:
    """Rows owned by each rank for a panel partition."""

    r: int
    num_rows: int
    panel_ranges: list[tuple[int, int]]

    def rows(self, k: int) -> tuple[int, int]:
        lo, hi = self.panel_ranges[k]
        return min(lo * self.r, self.num_rows), min(hi * self.r, self.num_rows)


def shard_layout(row_ptr, r: int, workers: int) -> ShardLayout:
    return ShardLayout(r, len(row_ptr) - 1, panel_partition(row_ptr, r, workers))


def allgather_slices(x, layout: ShardLayout, rank: int, world: int) -> None:
    """Fill every rank's copy of x with the owners' slices (allgatherv in place).

    The slices are unequal (nnz-balanced), so each owner broadcasts its slice
    into the same view on every rank; the P broadcasts are issued together and
    waited on once (NCCL runs them as one batch of collectives).
    """
    import torch.distributed as dist
    reqs = []
    for k in range(world):
        lo, hi = layout.rows(k)
        if hi > lo:
            reqs.append(dist.broadcast(x[lo:hi], src=k, async_op=True))
    for q in reqs:
        q.wait()


def iterate_products(x0, steps: int, layout: ShardLayout, rank: int, world: int,
                     local_spmv: Callable, scale: float = 1.0):
    """x_{t+1} = scale * A x_t for `steps` products, A split by row panels.

    local_spmv(x_full, y_out) computes this rank's rows of A.x into y_out
    (a view of the next x buffer).  Returns the final x (replicated).
    """
    import torch
    xa = x0.clone()
    xb = torch.empty_like(xa)
    lo, hi = layout.rows(rank)
    for _ in range(steps):
        local_spmv(xa, xb[lo:hi])
        if scale != 1.0:
            xb[lo:hi] *= scale
        allgather_slices(xb, layout, rank, world)
        xa, xb = xb, xa
    return xa


# ----------------------------------------------------------------------------- bench
def bench_distributed(args, formats) -> None:
    """bench.py for N > 1: config-2/5 stencil split over the ranks; one step is
    one iterated product per format (local K2 + all-gather of x over NCCL)."""
    import json
    import os
    import time

    import torch
    import torch.distributed as dist

    from . import _native as nat
    from .blocks import csr_to_spc5_device, filling_stats, torch_stream
    from .workloads import CONFIGS, x_vector

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = CONFIGS[args.config]
    if "n" not in cfg:
        raise SystemExit("multi-GPU bench supports the stencil configs (2, 5)")
    n = cfg["n"]
    N = n ** 3
    prec = cfg["precision"]
    tdt = torch.float64 if prec == "f64" else torch.float32
    vb = 8 if prec == "f64" else 4
    rp_all = torch.empty(N + 1, dtype=torch.int64, device="cuda")
    nat.check(nat.lib.spc5_gen_stencil27_rowptr(n, 0, N, rp_all.data_ptr(), 0))
    x0 = torch.from_numpy(x_vector(N, prec)).to("cuda")
    results = {}
    for (r, vs) in formats:
        layout = shard_layout(rp_all, r, world)
        lo, hi = layout.rows(rank)
        rows = hi - lo
        rp = torch.empty(rows + 1, dtype=torch.int64, device="cuda")
        nat.check(nat.lib.spc5_gen_stencil27_rowptr(n, lo, hi, rp.data_ptr(), 0))
        nnz = int(rp[-1])
        ci = torch.empty(max(nnz, 1), dtype=torch.int32, device="cuda")
        va = torch.empty(max(nnz, 1), dtype=tdt, device="cuda")
        nat.check(nat.lib.spc5_gen_stencil27_fill(n, lo, hi, 1 if prec == "f64" else 0, 0, 27.0,
                                                  rp.data_ptr(), ci.data_ptr(), va.data_ptr(), 0))
        torch.cuda.synchronize()
        s = csr_to_spc5_device(rows, N, rp, ci, va, r, vs)
        del rp, ci, va
        h = s.handle()
        nnz_all = torch.tensor([h.info.nnz], device="cuda")
        dist.all_reduce(nnz_all)

        def local_spmv(xf, yout, h=h):
            nat.check(nat.lib.spc5_spmv(h.ptr, xf.data_ptr(), yout.data_ptr(), 0, torch_stream()))

        # rescale by an exact power of two each step so 100 iterations stay finite
        scale = 1.0 / 64.0
        for _ in range(args.warmup):
            iterate_products(x0, 1, layout, rank, world, local_spmv, scale)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        iterate_products(x0, args.steps, layout, rank, world, local_spmv, scale)
        e1.record()
        torch.cuda.synchronize()
        el = torch.tensor([e0.elapsed_time(e1) * 1e-3], device="cuda")
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
        dist.barrier()
        results[f"b({r},{vs})"] = {"seconds": float(el), "nnz": int(nnz_all),
                                   "local_footprint": filling_stats(s).footprint_bytes}
        del s, h
        torch.cuda.empty_cache()
    if rank == 0:
        tot_flops = sum(2.0 * v["nnz"] * args.steps for v in results.values())
        tot_t = sum(v["seconds"] for v in results.values())
        line = {"metric": "SpMV GFLOP/s (2*nnz/t)", "value": tot_flops / tot_t / 1e9,
                "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": tot_t / args.steps * 1e3, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": prec, "data": "synthetic",
                "config": {"workload": cfg["name"], "formats": list(results),
                           "step": "x <- A.x per format: local K2 + allgather of x (NCCL)",
                           "parallelism": f"row-panel shards x{world}"},
                "formats": {k: {"gflops": 2.0 * v["nnz"] * args.steps / v["seconds"] / 1e9}
                            for k, v in results.items()}}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
