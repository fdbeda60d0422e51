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
  (one NCCL group of point-to-point sends/receives) fills the rest and the
  buffers swap.

The local product is a callable so the host logic is testable on CPU with the
gloo backend (tests/test_distributed.py); on GPUs it is the C-ABI SpMV.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

__all__ = ["panel_partition", "ShardLayout", "shard_layout", "allgather_slices",
           "iterate_products", "FusedExchange", "iterate_products_fused", "NcclShard",
           "bench_distributed"]


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


def allgather_slices(x, layout: ShardLayout, rank: int, world: int, mode: str = "p2p") -> None:
    """Fill every rank's copy of x with the owners' slices (allgatherv in place).

    The slices are unequal (nnz-balanced row-panel shards), so this is an
    all-gather-v.  mode "p2p" (default): one batch of point-to-point
    operations -- this rank's slice sent to every peer, every peer's slice
    received into its place in x -- issued as ONE NCCL group
    (``batch_isend_irecv`` -> ncclGroupStart/End), so every transfer is in
    flight at once over NVSwitch.  mode "bcast": one broadcast per owner,
    coalesced (the A/B alternative).  No staging copies either way.
    """
    import torch.distributed as dist
    if world == 1:
        return
    mine = layout.rows(rank)
    if mode == "bcast":
        reqs = []
        for k in range(world):
            lo, hi = layout.rows(k)
            if hi > lo:
                reqs.append(dist.broadcast(x[lo:hi], src=k, async_op=True))
        for q in reqs:
            q.wait()
        return
    ops = []
    for k in range(world):
        if k == rank:
            continue
        lo, hi = layout.rows(k)
        if mine[1] > mine[0]:
            ops.append(dist.P2POp(dist.isend, x[mine[0]:mine[1]], k))
        if hi > lo:
            ops.append(dist.P2POp(dist.irecv, x[lo:hi], k))
    if ops:
        for q in dist.batch_isend_irecv(ops):
            q.wait()


def iterate_products(x0, steps: int, layout: ShardLayout, rank: int, world: int,
                     local_spmv: Callable, scale: float = 1.0, mode: str = "p2p"):
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
        allgather_slices(xb, layout, rank, world, mode)
        xa, xb = xb, xa
    return xa


class FusedExchange:
    """Symmetric-memory x buffers for iterated products with the exchange fused
    into K2 (spc5_spmv_mirrored).  Set up once (allocation + rendezvous), then
    run() any number of iterations: K2 stores every row of this rank's slice
    into its own next-x buffer and, over NVLink, into every peer's (no
    all-gather after the product); a device-side barrier on the symmetric
    handle orders iterations."""

    def __init__(self, n: int, dtype, layout: ShardLayout, rank: int, group=None):
        import ctypes

        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        group = group or dist.group.WORLD
        dev = torch.device("cuda", torch.cuda.current_device())
        self.bufs = [symm.empty(n, dtype=dtype, device=dev) for _ in range(2)]
        self.hdls = [symm.rendezvous(b, group) for b in self.bufs]
        self.lo, _ = layout.rows(rank)
        self.esz = self.bufs[0].element_size()
        self.peers = []
        for h in self.hdls:
            ptrs = [int(p) for i, p in enumerate(h.buffer_ptrs) if i != rank]
            self.peers.append(((ctypes.c_void_p * max(len(ptrs), 1))(*ptrs), len(ptrs)))

    def run(self, handle, x0, steps: int, scale: float = 1.0):
        from . import _native as nat
        from .blocks import torch_stream
        self.bufs[0].copy_(x0)
        self.hdls[0].barrier(channel=0)
        cur = 0
        for _ in range(steps):
            nxt = 1 - cur
            arr, npeer = self.peers[nxt]
            nat.check(nat.lib.spc5_spmv_mirrored(
                handle.ptr, self.bufs[cur].data_ptr(),
                self.bufs[nxt].data_ptr() + self.lo * self.esz, float(scale), arr, npeer,
                self.lo, torch_stream()))
            self.hdls[nxt].barrier(channel=0)
            cur = nxt
        return self.bufs[cur]


def iterate_products_fused(x0, steps: int, layout: ShardLayout, rank: int, world: int, handle,
                           scale: float = 1.0, group=None):
    """x_{t+1} = scale * A x_t with the exchange fused into K2 (see FusedExchange)."""
    ex = FusedExchange(x0.numel(), x0.dtype, layout, rank, group)
    return ex.run(handle, x0, steps, scale).clone()




class NcclShard:
    """This rank's shard of an iterated product through the C ABI's spc5_mg_*
    entry points (NCCL driven from libspc5_b200.so, no torch.distributed on
    the data path): ``step`` is x_next = scale * A.x, the local K2 into this
    rank's rows of x_next, then the all-gather-v of the slices in one NCCL
    group.  ``nccl_id`` is the 128-byte id of rank 0 (``NcclShard.unique_id()``),
    shipped to the other ranks by any means."""

    @staticmethod
    def unique_id() -> bytes:
        import ctypes

        from . import _native as nat
        buf = ctypes.create_string_buffer(128)
        nat.check(nat.lib.spc5_mg_unique_id(buf))
        return buf.raw

    @staticmethod
    def partition(row_ptr_dev, r: int, workers: int) -> list[tuple[int, int]]:
        """partition_by_nnz panel ranges from device CSR row pointers (C ABI)."""
        from . import _native as nat
        from .blocks import torch_stream
        out = np.zeros(2 * workers, dtype=np.int64)
        nat.check(nat.lib.spc5_mg_partition(row_ptr_dev.data_ptr(), row_ptr_dev.numel() - 1, r,
                                            workers, out.ctypes.data, torch_stream()))
        return [(int(out[2 * k]), int(out[2 * k + 1])) for k in range(workers)]

    def __init__(self, nccl_id: bytes, world: int, rank: int):
        import ctypes

        from . import _native as nat
        self._nat = nat
        self._h = ctypes.c_void_p()
        nat.check(nat.lib.spc5_mg_init(ctypes.c_char_p(nccl_id), world, rank,
                                       ctypes.byref(self._h)))
        self.world, self.rank = world, rank
        self._keep = None

    def shard(self, matrix, layout: ShardLayout) -> None:
        rows = np.array([v for k in range(self.world) for v in layout.rows(k)], dtype=np.int64)
        self._keep = (matrix, rows)  # the C side borrows the matrix handle
        self._nat.check(self._nat.lib.spc5_mg_shard(self._h, matrix.handle().ptr,
                                                    rows.ctypes.data))

    def step(self, x, x_next, scale: float = 1.0) -> None:
        from .blocks import torch_stream
        self._nat.check(self._nat.lib.spc5_mg_spmv_step(self._h, x.data_ptr(), x_next.data_ptr(),
                                                        float(scale), torch_stream()))

    def close(self) -> None:
        if self._h:
            self._nat.lib.spc5_mg_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ----------------------------------------------------------------------------- bench
def _timed(fn, stream):
    """Device time of fn() on `stream` (CUDA events), max over ranks."""
    import torch
    import torch.distributed as dist
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    out = fn()
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) * 1e-3], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t), out


def bench_distributed(args, formats) -> None:
    """bench.py for N > 1 (one process per GPU, torchrun, NCCL).

    --scaling strong (the default): the config's one matrix (BASELINE config
    5: the 400^3 stencil) is split into nnz-balanced row-panel shards
    (panel_partition == partition_by_nnz, computed from the generator's row
    pointers alone) and every rank generates and converts only its rows.
    --scaling weak: the 27-point stencil on an n x n x (n * N) box, one n^3
    cube of rows per GPU.  One step = one product per format with x
    replicated and each rank writing its own y-slice: no data-path
    collective (the bench `value`).  The iterated form -- x <- A.x/64 for
    --iters products (BASELINE: 100), x refreshed between products by the
    all-gather-v of the y-slices in one NCCL group -- is timed after it, A/B
    against coalesced broadcasts and against the exchange fused into K2
    (FusedExchange).  Times are device times (CUDA events), the max over
    ranks."""
    import json
    import os
    import time

    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    import torch
    import torch.distributed as dist

    from . import _native as nat
    from .blocks import csr_to_spc5_device, filling_stats, torch_stream
    from .kernels import spmv
    from .workloads import CONFIGS, config_shape, device_rowptr, device_rows, x_vector

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = CONFIGS[args.config]
    if cfg.get("gen") is None and "n" not in cfg:
        raise SystemExit(f"config {args.config}: no device generator for the multi-GPU bench")
    weak = "n" in cfg and args.scaling == "weak"
    if weak:
        cfg = dict(cfg, nz=cfg["n"] * world)
    prec = cfg["precision"]
    tdt = torch.float64 if prec == "f64" else torch.float32
    vb = 8 if prec == "f64" else 4
    N, C = config_shape(cfg)
    rp_all = device_rowptr(cfg, 0, N)  # structure only: the partition needs nothing else
    x_np = x_vector(C, prec)
    x0 = torch.from_numpy(x_np).to("cuda")
    st = torch_stream()
    stream = torch.cuda.current_stream()
    results, launches = {}, 0
    from bench import ClockSampler, config_dict, peaks  # noqa: E402  (repo root on sys.path)
    sampler = ClockSampler(local) if rank == 0 else None
    iters = max(1, args.iters)
    for (r, vs) in formats:
        layout = shard_layout(rp_all, r, world)
        lo, hi = layout.rows(rank)
        rp, ci, va = device_rows(cfg, lo, hi)
        s = csr_to_spc5_device(hi - lo, C, rp, ci, va, r, vs)
        del rp, ci, va
        torch.cuda.empty_cache()
        h = s.handle()
        y = torch.empty(max(hi - lo, 1), dtype=tdt, device="cuda")
        counts = torch.tensor([h.info.nnz, filling_stats(s).footprint_bytes + vb * (hi - lo)],
                              dtype=torch.int64, device="cuda")
        dist.all_reduce(counts)
        nnz_all, bytes_all = int(counts[0]), int(counts[1]) + vb * C * world

        def products(n):
            c = 0
            for _ in range(n):
                nat.check(nat.lib.spc5_spmv(h.ptr, x0.data_ptr(), y.data_ptr(), 0, st))
                c += nat.last_launch_count()
            return c

        products(args.warmup)
        if sampler is not None and not results:
            sampler.start()
            time.sleep(0.3)
        el, n_l = _timed(lambda: products(args.steps), stream)
        launches += n_l

        # iterated products: local K2 into the next x buffer + all-gather-v of the slices
        def local_spmv(xf, yout, h=h):
            nat.check(nat.lib.spc5_spmv(h.ptr, xf.data_ptr(), yout.data_ptr(), 0, st))

        iterate_products(x0, 2, layout, rank, world, local_spmv, 1.0 / 64.0)
        it, xr = _timed(lambda: iterate_products(x0, iters, layout, rank, world, local_spmv,
                                                 1.0 / 64.0), stream)
        itb, xb = _timed(lambda: iterate_products(x0, iters, layout, rank, world, local_spmv,
                                                  1.0 / 64.0, mode="bcast"), stream)
        same_b = bool(torch.equal(xr, xb))
        # the same iterations with the exchange fused into K2 (NVLink stores)
        try:
            if world > 1 and not (getattr(args, "fused", False) or os.environ.get("SPC5_BENCH_FUSED")):
                # never run on more than one rank in this environment (one GPU per call):
                # a hang here would lose the whole line, so it is opt-in (--fused)
                raise RuntimeError("skipped at N > 1 (pass --fused)")
            ex = FusedExchange(C, tdt, layout, rank)
            ex.run(h, x0, 2, 1.0 / 64.0)
            ft, xf = _timed(lambda: ex.run(h, x0, iters, 1.0 / 64.0).clone(), stream)
            fused = {"seconds": ft, "bitwise_equal_to_allgather": bool(torch.equal(xf, xr))}
        except Exception as e:  # symmetric memory unavailable: report, keep the line
            fused = {"error": f"{type(e).__name__}: {e}"[:200]}
        del xr, xb

        # end to end through the public API on pinned host buffers
        xp = torch.empty(C, dtype=tdt, pin_memory=True)
        xp.numpy()[:] = x_np
        yp = torch.empty(max(hi - lo, 1), dtype=tdt, pin_memory=True)
        e2e_steps = max(3, min(args.steps, 20))
        spmv(s, xp.numpy(), yp.numpy()[:hi - lo])
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            spmv(s, xp.numpy(), yp.numpy()[:hi - lo])
        te = torch.tensor([time.perf_counter() - t0], device="cuda")
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        results[f"b({r},{vs})"] = {"seconds": el, "nnz": nnz_all, "bytes": bytes_all,
                                   "iter_seconds": it, "iter_bcast_seconds": itb,
                                   "bcast_bitwise_equal": same_b, "iters": iters,
                                   "e2e_seconds": float(te), "e2e_steps": e2e_steps,
                                   "fused": fused, "h2d": vb * C, "d2h": vb * (hi - lo)}
        del s, h, y, xp, yp
        torch.cuda.empty_cache()
    clocks = sampler.stop() if sampler is not None else None
    h2d = torch.tensor([sum(v["h2d"] for v in results.values())], device="cuda")
    d2h = torch.tensor([sum(v["d2h"] for v in results.values())], device="cuda")
    dist.all_reduce(h2d)
    dist.all_reduce(d2h)
    lc = torch.tensor([launches], device="cuda")
    dist.all_reduce(lc)
    if rank == 0:
        peak, peak_kind = peaks()
        flops = sum(2.0 * v["nnz"] for v in results.values())
        tot_t = sum(v["seconds"] for v in results.values())
        tot_b = sum(v["bytes"] for v in results.values()) * args.steps
        achieved = tot_b / tot_t / 1e9
        conf = config_dict(args.config, formats, world, "weak" if weak else "strong")
        if weak:
            conf["workload"] = (f"stencil27_{cfg['n']}x{cfg['n']}x{cfg['nz']}_{prec} "
                                f"({cfg['n']}^3 rows per GPU)")
            conf["num_rows"] = conf["num_cols"] = N
        line = {"metric": "SpMV GFLOP/s (2*nnz/t)", "value": flops * args.steps / tot_t / 1e9,
                "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": tot_t / args.steps * 1e3,
                "higher_is_better": True, "scaling": "weak" if weak else "strong",
                "vs_baseline": None, "dtype": prec, "data": "synthetic",
                "config": conf,
                "matrix": {"nnz": results[next(iter(results))]["nnz"],
                           "step": "x replicated, each rank writes its nnz-balanced "
                                   "row-panel slice of y"},
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak * world,
                             "unit": "GB/s", "frac": achieved / (peak * world),
                             "traffic": None,
                             "peak_source": f"{peak_kind} hbm_gbs x {world} GPUs",
                             "alg_bytes_per_step": sum(v["bytes"] for v in results.values())},
                "formats": {k: {"gflops": 2.0 * v["nnz"] * args.steps / v["seconds"] / 1e9,
                                "us": v["seconds"] / args.steps * 1e6,
                                "iterated_gflops": 2.0 * v["nnz"] * v["iters"]
                                / v["iter_seconds"] / 1e9,
                                "iterated_us": v["iter_seconds"] / v["iters"] * 1e6,
                                "iterated_bcast_us": v["iter_bcast_seconds"] / v["iters"] * 1e6,
                                "bcast_bitwise_equal": v["bcast_bitwise_equal"],
                                "iterated_fused_us": (v["fused"]["seconds"] / v["iters"] * 1e6
                                                      if "seconds" in v["fused"] else None),
                                "fused": v["fused"]}
                            for k, v in results.items()},
                "iterated": {"step": "x <- A.x/64: local K2 into the next x + all-gather-v of "
                                     "the y-slices in one NCCL group (BASELINE config 5 form)",
                             "iters_per_format": iters,
                             "value": sum(2.0 * v["nnz"] * v["iters"] for v in results.values())
                             / sum(v["iter_seconds"] for v in results.values()) / 1e9,
                             "unit": "GFLOP/s"},
                "gpu_launches": int(lc),
                "clocks": clocks,
                "e2e": {"value": sum(2.0 * v["nnz"] * v["e2e_steps"] for v in results.values())
                        / sum(v["e2e_seconds"] for v in results.values()) / 1e9,
                        "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
                        "d2h_bytes_per_step": int(d2h),
                        "path": "paper_2307_14774_b200.spmv(numpy pinned) per rank, max over ranks"},
                "cpu_baseline": None}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
