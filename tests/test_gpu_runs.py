"""K2 run plans (csrc/spmv_kernel.cuh row_slots RUN; plan.cu runs_kernel): when
every row mask of a matrix is one contiguous run of bits (stencils, bands,
dense sub-blocks) the lane-per-panel-row steps gather x at immediate offsets
from each run's top instead of walking the bits.  Same products, same order:
y must be BITWISE the general walk's (plan knob SPC5_NO_RUN=1), and within the
oracle tolerance like every other mode.
"""
import numpy as np
import pytest

from golden_io import Csr
from oracle import oracle
from test_gpu_parity import assert_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spc5(cuda_device):
    import paper_2307_14774_b200 as pkg
    return pkg


def _banded(n, offsets, dtype, seed):
    rng = np.random.default_rng(seed)
    rows = [np.array(sorted({min(max(i + o, 0), n - 1) for o in offsets})) for i in range(n)]
    rp = np.zeros(n + 1, np.int64)
    np.cumsum([len(c) for c in rows], out=rp[1:])
    ci = np.concatenate(rows).astype(np.int32)
    return Csr(n, n, rp, ci, rng.uniform(-1, 1, ci.size).astype(dtype))


def _cases():
    from paper_2307_14774_b200.mmio import make_dense
    from paper_2307_14774_b200.workloads import stencil27
    yield "stencil16_f64", stencil27(16)
    yield "stencil12_f32", stencil27(12, "f32")
    yield "tridiag_f64", _banded(5000, (-1, 0, 1), np.float64, 1)
    yield "band9_f32", _banded(3000, tuple(range(-4, 5)), np.float32, 2)  # runs of 9: dense-row path
    yield "blocks3_f64", _banded(4096, (-300, -299, -298, -1, 0, 1, 700, 701, 702), np.float64, 3)
    yield "dense96_f64", make_dense(96)  # 16-bit runs, more than 4 slots per block row


@pytest.mark.parametrize("name,m", list(_cases()), ids=[n for n, _ in _cases()])
def test_run_plan_bitwise_equals_general_walk(spc5, name, m, monkeypatch):
    x = np.random.default_rng(11).uniform(-1, 1, m.num_cols).astype(m.values.dtype)
    vs_list = (8, 16) if m.values.dtype == np.float32 else (4, 8, 16)
    for r in (1, 2, 4, 8):
        for vs in vs_list:
            monkeypatch.delenv("SPC5_NO_RUN", raising=False)
            y_run = spc5.spmv(spc5.csr_to_spc5(m, r, vs), x)
            monkeypatch.setenv("SPC5_NO_RUN", "1")
            y_gen = spc5.spmv(spc5.csr_to_spc5(m, r, vs), x)
            assert y_run.tobytes() == y_gen.tobytes(), (name, r, vs)
            y_ref = np.zeros(m.num_rows, m.values.dtype)
            oracle.spmv_spc5_scalar(oracle.csr_to_spc5(m, r, vs), x, y_ref)
            assert_close(m, y_run, y_ref, x, f"run {name} {r},{vs}")


def test_non_run_masks_keep_the_general_walk(spc5):
    """Masks with holes (0b101) must not take the run path: a matrix mixing a
    band with every-other-column rows still matches the oracle."""
    m = _banded(4000, (-2, 0, 2, 5), np.float64, 4)
    x = np.random.default_rng(12).uniform(-1, 1, m.num_cols)
    for r in (1, 4, 8):
        y = spc5.spmv(spc5.csr_to_spc5(m, r, 8), x)
        y_ref = np.zeros(m.num_rows)
        oracle.spmv_spc5_scalar(oracle.csr_to_spc5(m, r, 8), x, y_ref)
        assert_close(m, y, y_ref, x, f"holes {r}")
