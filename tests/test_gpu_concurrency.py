"""One matrix handle under concurrent use (header contract).

The matrix has split chunks (a giant row: carry slots + fixup), the state a
shared per-handle buffer would corrupt.  Products on two streams from two
threads with different x, the host-buffer path from two threads, range
products, and a CUDA-graph replay must all equal the serial product bit for
bit.
"""

import threading

import numpy as np
import pytest

from test_gpu_parity import giant_row_matrix

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mats(cuda_device):
    import paper_2307_14774_b200 as pkg
    out = {}
    for prec in ("f64", "f32"):
        m = giant_row_matrix(prec)
        for r, vs in ((1, 4), (2, 8), (4, 16)):
            s = pkg.csr_to_spc5(m, r, vs)
            assert s.handle().info.num_split_chunks > 0  # the carry path is live
            out[(prec, r, vs)] = (m, s)
    return out


def _xs(m, k):
    rng = np.random.default_rng(100 + k)
    return rng.uniform(-1, 1, m.num_cols).astype(m.values.dtype)


def test_two_streams_two_threads_bitwise(mats):
    import torch

    from paper_2307_14774_b200 import _native as nat
    for key, (m, s) in mats.items():
        h = s.handle().ptr
        tdt = torch.float64 if key[0] == "f64" else torch.float32
        xs = [torch.from_numpy(_xs(m, k)).cuda() for k in range(2)]
        ref = []
        for k in range(2):  # serial products
            y = torch.empty(m.num_rows, dtype=tdt, device="cuda")
            nat.check(nat.lib.spc5_spmv(h, xs[k].data_ptr(), y.data_ptr(), 0,
                                        int(torch.cuda.current_stream().cuda_stream)))
            ref.append(y)
        torch.cuda.synchronize()
        outs = [[torch.empty(m.num_rows, dtype=tdt, device="cuda") for _ in range(50)]
                for _ in range(2)]
        errs = []

        def worker(k):
            try:
                st = torch.cuda.Stream()
                for y in outs[k]:
                    nat.check(nat.lib.spc5_spmv(h, xs[k].data_ptr(), y.data_ptr(), 0,
                                                int(st.cuda_stream)))
                st.synchronize()
            except Exception as e:  # pragma: no cover - reported below
                errs.append(e)

        ts = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not errs, errs
        for k in range(2):
            for y in outs[k]:
                assert torch.equal(y, ref[k]), key


def test_host_path_two_threads_bitwise(mats):
    import paper_2307_14774_b200 as pkg
    for key, (m, s) in mats.items():
        xs = [_xs(m, k) for k in range(2)]
        ref = [pkg.spmv(s, xs[k]) for k in range(2)]
        got = [[None] * 20 for _ in range(2)]
        errs = []

        def worker(k):
            try:
                for i in range(20):
                    got[k][i] = pkg.spmv(s, xs[k])
            except Exception as e:  # pragma: no cover
                errs.append(e)

        ts = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not errs, errs
        for k in range(2):
            for y in got[k]:
                assert y.tobytes() == ref[k].tobytes(), key


def test_range_products_no_host_sync_bitwise(mats):
    """spc5_spmv_panels resolves its block range on the device: every range of
    a partition, each on its own stream, reassembles the full product."""
    import torch

    import paper_2307_14774_b200 as pkg
    from paper_2307_14774_b200 import _native as nat
    for key, (m, s) in mats.items():
        h = s.handle().ptr
        tdt = torch.float64 if key[0] == "f64" else torch.float32
        x = torch.from_numpy(_xs(m, 0)).cuda()
        full = torch.from_numpy(pkg.spmv(s, _xs(m, 0))).cuda()
        for w in (2, 3, 7):
            y = torch.full((m.num_rows,), float("nan"), dtype=tdt, device="cuda")
            streams = [torch.cuda.Stream() for _ in range(w)]
            for (lo, hi), st in zip(pkg.partition_by_nnz(s, w).ranges, streams):
                st.wait_stream(torch.cuda.current_stream())
                nat.check(nat.lib.spc5_spmv_panels(h, lo, hi, x.data_ptr(), y.data_ptr(), 0,
                                                   int(st.cuda_stream)))
            for st in streams:
                torch.cuda.current_stream().wait_stream(st)
            assert torch.equal(y, full), (key, w)


def test_graph_capture_replay_bitwise(mats):
    import torch

    from paper_2307_14774_b200 import _native as nat
    for key, (m, s) in mats.items():
        h = s.handle().ptr
        tdt = torch.float64 if key[0] == "f64" else torch.float32
        x = torch.from_numpy(_xs(m, 1)).cuda()
        y0 = torch.empty(m.num_rows, dtype=tdt, device="cuda")
        nat.check(nat.lib.spc5_spmv(h, x.data_ptr(), y0.data_ptr(), 0,
                                    int(torch.cuda.current_stream().cuda_stream)))
        y = torch.empty_like(y0)
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            nat.check(nat.lib.spc5_spmv(h, x.data_ptr(), y.data_ptr(), 0, int(cap.cuda_stream)))
            nat.check(nat.lib.spc5_spmv_panels(h, 0, s.num_panels // 2, x.data_ptr(),
                                               y.data_ptr(), 0, int(cap.cuda_stream)))
        for _ in range(3):
            y.zero_()
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(y, y0), key


def test_c_abi_nccl_single_rank(cuda_device):
    """spc5_mg_* on a one-rank NCCL communicator: the C-ABI partition equals
    partition_by_nnz, and a step x_next = A.x/64 equals the plain product
    scaled (the all-gather is empty at one rank)."""
    import torch

    import paper_2307_14774_b200 as spc5
    from paper_2307_14774_b200.distributed import NcclShard, shard_layout
    from paper_2307_14774_b200.workloads import stencil27, x_vector
    m = stencil27(24)
    rp = torch.from_numpy(m.row_ptr).cuda()
    for r in (1, 2, 4, 8):
        s = spc5.csr_to_spc5(m, r, 8)
        for w in (1, 2, 3, 8):
            assert NcclShard.partition(rp, r, w) == spc5.partition_by_nnz(s, w).ranges, (r, w)
        mg = NcclShard(NcclShard.unique_id(), 1, 0)
        mg.shard(s, shard_layout(m.row_ptr, r, 1))
        x = torch.from_numpy(x_vector(m.num_cols)).cuda()
        xn = torch.empty_like(x)
        mg.step(x, xn, 1.0 / 64.0)
        y = torch.from_numpy(spc5.spmv(s, x.cpu().numpy())).cuda() / 64.0
        assert torch.equal(xn, y), r
        mg.close()
