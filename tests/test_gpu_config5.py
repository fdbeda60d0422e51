"""BASELINE config 5 at full size on one GPU: the 27-point stencil on 400^3
(64,000,000 rows, 1,719,374,392 nnz), all eight (precision, r) pairs -- f64
beta(1|2|4|8, 8) and f32 beta(1|2|4|8, 16).

Conversion and product are panel-local (blocks.py:112-123, kernels.py:130-142),
so the reference's own conversion of an r-aligned row slice equals the slice
of the full conversion bit for bit, and its product equals the slice of y
(the sliced oracle).  For every format, on nine 2^18-row slices
-- the first rows, the last rows, and one straddling every rank boundary of
the P = 2/4/8 partition (parallel.py:31-52) -- the test asserts:

* the GPU matrix's four arrays over the slice equal the oracle's conversion of
  the host-generated slice (rowptr offset by the slice's first block);
* y = A.x (product 1) and A.(A.x/64) (product 2 of the iterated loop, with the
  GPU's validated product 1 as input) are within 1e-12 (f64) / 1e-5 (f32) of
  the oracle's scalar path, relative to sum_j |a_ij x_j|;

and over all 64M rows, y against the exact double-double row sums of the
generator's CSR.
"""

import ctypes

import numpy as np
import pytest

from oracle import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N3 = 400
N = N3 ** 3
SLICE = 1 << 18
TOL = {"f64": 1e-12, "f32": 1e-5}
FORMATS = [("f64", r, 8) for r in (1, 2, 4, 8)] + [("f32", r, 16) for r in (1, 2, 4, 8)]


@pytest.fixture(scope="module")
def host_slices():
    """Host CSR of every slice, per precision (generated once)."""
    return {}


@pytest.fixture(scope="module")
def xs(cuda_device):
    from paper_2307_14774_b200.workloads import x_vector
    return {p: x_vector(N, p) for p in ("f64", "f32")}


def _export_device(s):
    """The matrix's four arrays as device tensors (D2D copies)."""
    import torch

    from paper_2307_14774_b200 import _native as nat
    from paper_2307_14774_b200.blocks import torch_stream
    h = s.handle()
    info = h.info
    rp = torch.empty(info.num_panels + 1, dtype=torch.int64, device="cuda")
    ci = torch.empty(info.num_blocks, dtype=torch.int32, device="cuda")
    mk = torch.empty(info.num_blocks * info.r,
                     dtype=torch.uint8 if info.mask_bytes == 1 else torch.int16, device="cuda")
    va = torch.empty(info.nnz, dtype=torch.float64 if info.precision == nat.F64
                     else torch.float32, device="cuda")
    nat.check(nat.lib.spc5_export(h.ptr, rp.data_ptr(), ci.data_ptr(), mk.data_ptr(),
                                  va.data_ptr(), 0, torch_stream()))
    return rp, ci, mk, va


def _slices(s, r):
    starts = {0, N - SLICE}
    import paper_2307_14774_b200 as spc5
    for P in (2, 4, 8):
        for lo, _ in spc5.partition_by_nnz(s, P).ranges[1:]:
            b = lo * r
            starts.add(min(max(0, (b - SLICE // 2) // 8 * 8), N - SLICE))
    return sorted(starts)


@pytest.mark.parametrize("prec,r,vs", FORMATS)
def test_config5_format(cuda_device, host_slices, xs, prec, r, vs):
    import torch

    from paper_2307_14774_b200 import _native as nat
    from paper_2307_14774_b200.blocks import csr_to_spc5_device, torch_stream
    from paper_2307_14774_b200.workloads import CONFIGS, device_rows, stencil27_nnz, stencil27_rows
    cfg = dict(CONFIGS[5 if prec == "f64" else 7])
    tdt = torch.float64 if prec == "f64" else torch.float32
    rp, ci, va = device_rows(cfg, 0, N)
    assert int(rp[-1]) == stencil27_nnz(N3)
    s = csr_to_spc5_device(N, N, rp, ci, va, r, vs)
    st = torch_stream()
    x = torch.from_numpy(xs[prec]).to("cuda")
    y1 = torch.empty(N, dtype=tdt, device="cuda")
    y2 = torch.empty(N, dtype=tdt, device="cuda")
    h = s.handle().ptr
    nat.check(nat.lib.spc5_spmv(h, x.data_ptr(), y1.data_ptr(), 0, st))
    x1 = y1 * (1.0 / 64.0)  # exact scaling (the iterated loop's rescale)
    nat.check(nat.lib.spc5_spmv(h, x1.data_ptr(), y2.data_ptr(), 0, st))
    # all rows: exact double-double sums of the generator's CSR
    ye = torch.empty(N, dtype=torch.float64, device="cuda")
    ya = torch.empty(N, dtype=torch.float64, device="cuda")
    nat.check(nat.lib.spc5_csr_exact(N, nat.F64 if prec == "f64" else nat.F32, rp.data_ptr(),
                                     ci.data_ptr(), va.data_ptr(), x.data_ptr(), ye.data_ptr(),
                                     ya.data_ptr(), st))
    err = ((y1.to(torch.float64) - ye).abs() / ya.clamp(min=1e-300)).max().item()
    assert err <= TOL[prec], ("all rows vs exact", err)
    row_ptr = rp.cpu().numpy()
    del ci, va, rp, ye, ya
    torch.cuda.empty_cache()
    drp, dci, dmk, dva = _export_device(s)
    y1h, x1h, y2h = y1.cpu().numpy(), x1.cpu().numpy(), y2.cpu().numpy()
    for lo in _slices(s, r):
        hi = lo + SLICE
        key = (prec, lo)
        if key not in host_slices:
            host_slices[key] = stencil27_rows(N3, lo, hi, prec)
        m = host_slices[key]
        ref = oracle.csr_to_spc5(m, r, vs)
        p0, p1 = lo // r, hi // r
        b0, b1 = int(drp[p0]), int(drp[p1])
        v0, v1 = int(row_ptr[lo]), int(row_ptr[hi])
        assert np.array_equal((drp[p0:p1 + 1] - b0).cpu().numpy(), ref.block_rowptr), (lo, "rowptr")
        assert np.array_equal(dci[b0:b1].cpu().numpy().view(np.uint32), ref.block_colidx), (lo, "colidx")
        assert np.array_equal(dmk[b0 * r:b1 * r].cpu().numpy().view(ref.block_masks.dtype),
                              ref.block_masks), (lo, "masks")
        assert dva[v0:v1].cpu().numpy().tobytes() == ref.values.tobytes(), (lo, "values")
        for xin, ygpu, what in ((xs[prec], y1h, "product 1"), (x1h, y2h, "product 2")):
            yref = np.zeros(SLICE, dtype=xin.dtype)
            oracle.spmv_spc5_scalar(ref, xin, yref, threads=oracle.threads())
            _, a = oracle.csr_reference(m, xin)
            e = oracle.relative_error(ygpu[lo:hi], yref, a)
            assert float(e.max()) <= TOL[prec], (lo, what, float(e.max()))
    del s, drp, dci, dmk, dva, x, y1, y2, x1
    torch.cuda.empty_cache()
