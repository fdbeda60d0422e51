"""Multi-rank host logic of the row-panel sharding (paper_2307_14774_b200.distributed)
on CPU: gloo backend, world_size 2, the C oracle standing in for the local GPU
product.  The GPU kernels are covered by the -m gpu parity tests (including
shard-vs-full equality on one GPU)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from golden_io import expected_small, fmt_keys, small_case
from oracle import oracle
from paper_2307_14774_b200.distributed import allgather_slices, iterate_products, shard_layout, panel_partition
from paper_2307_14774_b200.workloads import stencil27, stencil27_rows, x_vector


def test_panel_partition_matches_reference():
    # parallel.py:31-52 computed from row pointers == the reference's ranges
    for name in ("tall", "longrows", "rand04", "rand17", "dense16", "lastpanel", "empty"):
        m = small_case(name)
        rec = expected_small()["cases"][name]
        for r, vs, f in fmt_keys(rec):
            for w, ranges in f["partition"].items():
                assert panel_partition(m.row_ptr, r, int(w)) == [tuple(t) for t in ranges], \
                    (name, r, w)
                assert panel_partition(torch.from_numpy(m.row_ptr), r, int(w)) == \
                    [tuple(t) for t in ranges], (name, r, w, "torch")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, r, steps, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full = stencil27(n)
    layout = shard_layout(full.row_ptr, r, world)
    lo, hi = layout.rows(rank)
    shard = oracle.csr_to_spc5(stencil27_rows(n, lo, hi), r, 8)

    def local_spmv(xf, yout):
        y = np.zeros(hi - lo)
        oracle.spmv_spc5_scalar(shard, xf.numpy(), y)
        yout.copy_(torch.from_numpy(y))

    x0 = torch.from_numpy(x_vector(full.num_cols))
    xf = iterate_products(x0, steps, layout, rank, world, local_spmv, scale=1.0 / 64)
    out[rank] = xf.numpy().tobytes()
    dist.destroy_process_group()


@pytest.mark.parametrize("r", [1, 2, 8])
def test_iterated_products_gloo(r):
    n, steps, world = 8, 3, 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n, r, steps, out), nprocs=world, join=True)
    # single-process reference: the oracle on the whole matrix, same scaling
    full = stencil27(n)
    s = oracle.csr_to_spc5(full, r, 8)
    x = x_vector(full.num_cols)
    for _ in range(steps):
        y = np.zeros(full.num_rows)
        oracle.spmv_spc5_scalar(s, x, y)
        x = y * (1.0 / 64)
    assert out[0] == out[1]  # replicated after the all-gather
    assert np.frombuffer(out[0], dtype=np.float64).tobytes() == x.tobytes()


def _worker_gather(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rp = np.array([0, 5, 5, 9, 20, 21, 30, 31], np.int64)  # uneven panel nnz
    layout = shard_layout(rp, 1, world)
    x = torch.full((7,), -1.0)
    lo, hi = layout.rows(rank)
    x[lo:hi] = float(rank + 1)
    allgather_slices(x, layout, rank, world)
    out[rank] = (x.tolist(), layout.panel_ranges)
    dist.destroy_process_group()


def test_allgather_uneven_slices():
    world = 3
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_gather, args=(world, _free_port(), out), nprocs=world, join=True)
    xs = [out[k][0] for k in range(world)]
    assert xs[0] == xs[1] == xs[2]
    ranges = out[0][1]
    expect = []
    for k, (lo, hi) in enumerate(ranges):
        expect += [float(k + 1)] * (hi - lo)
    assert xs[0] == expect
