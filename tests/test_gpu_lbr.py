"""K2 lane-per-block-row mode (LBR, csrc/spmv_kernel.cuh lbr_chunk): parity of
the mode forced on every golden case (plan knob SPC5_LBR=1), where the plan
would otherwise pick it only for long-panel matrices with mostly empty block
rows (FEM beta(8,8)).

Same bar as tests/test_gpu_parity.py: conversion untouched (K1), y within the
oracle tolerance of kernels.py:121-143's sequential sums, repeatable bit for
bit, range products (spmv_parallel) bitwise equal to the full product, split
panels through the carry slots / fixup kernel, accumulate mode, empty panels.
"""
import numpy as np
import pytest

from golden_io import case_x, expected_small, fmt_keys, small_case, small_case_names
from oracle import oracle
from test_gpu_parity import assert_close, giant_row_matrix

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spc5(cuda_device):
    import paper_2307_14774_b200 as pkg
    return pkg


@pytest.fixture(autouse=True)
def force_lbr(monkeypatch):
    monkeypatch.setenv("SPC5_LBR", "1")


def _oracle_y(m, r, vs, x):
    y_ref = np.zeros(m.num_rows, m.values.dtype)
    oracle.spmv_spc5_scalar(oracle.csr_to_spc5(m, r, vs), x, y_ref)
    return y_ref


@pytest.mark.parametrize("name", small_case_names())
def test_lbr_small_vs_oracle(spc5, name):
    m = small_case(name)
    x = case_x(name, m)
    for r, vs, _ in fmt_keys(expected_small()["cases"][name]):
        s = spc5.csr_to_spc5(m, r, vs)
        y = spc5.spmv(s, x)
        assert_close(m, y, _oracle_y(m, r, vs, x), x, f"lbr {name} {r},{vs}")
        assert spc5.spmv(s, x).tobytes() == y.tobytes(), (name, r, vs)


@pytest.mark.parametrize("chunk", [None, "32", "64"])
def test_lbr_giant_panels_and_ranges(spc5, chunk, monkeypatch):
    """Panels far longer than a chunk (every chunk starts inside a panel: carry
    slots + fixup) and range products over them, at several chunk sizes."""
    if chunk:
        monkeypatch.setenv("SPC5_CB", chunk)
    for prec in ("f64", "f32"):
        m = giant_row_matrix(prec)
        x = np.random.default_rng(9).uniform(-1, 1, m.num_cols).astype(m.values.dtype)
        for r, vs in ((1, 4), (2, 8), (4, 16), (8, 8), (8, 16)):
            s = spc5.csr_to_spc5(m, r, vs)
            y = np.zeros(m.num_rows, m.values.dtype)
            spc5.spmv_spc5_scalar(s, x, y)
            assert_close(m, y, _oracle_y(m, r, vs, x), x, f"lbr giant {prec} {r},{vs}")
            for w in (2, 3, 5, 8):
                yp = np.zeros(m.num_rows, m.values.dtype)
                spc5.spmv_parallel(s, x, yp, spc5.KernelConfig(precision=prec), w)
                assert yp.tobytes() == y.tobytes(), (prec, r, vs, w)


def test_lbr_fem_and_powerlaw_slices(spc5):
    from paper_2307_14774_b200.workloads import fem_rows, powerlaw_rows
    cases = (("fem", fem_rows(3000, 4200), ((4, 8), (8, 8), (2, 8), (1, 8))),
             ("powerlaw", powerlaw_rows(1000, 2600, precision="f32"), ((1, 16), (2, 16), (4, 16))))
    for name, m, fmts in cases:
        x = np.random.default_rng(3).uniform(-1, 1, m.num_cols).astype(m.values.dtype)
        prec = "f32" if m.values.dtype == np.float32 else "f64"
        for r, vs in fmts:
            s = spc5.csr_to_spc5(m, r, vs)
            y = spc5.spmv(s, x)
            assert_close(m, y, _oracle_y(m, r, vs, x), x, f"lbr {name} {r},{vs}")
            for w in (1, 3, 8):
                yp = np.zeros(m.num_rows, m.values.dtype)
                spc5.spmv_parallel(s, x, yp, spc5.KernelConfig(precision=prec), w)
                assert yp.tobytes() == y.tobytes(), (name, r, vs, w)


def test_lbr_accumulate_and_empty_panels(spc5):
    """y += A.x keeps the rows of empty panels; y = A.x zeroes them (chunks
    holding empty panels fall back to lane-per-block windows)."""
    from paper_2307_14774_b200.mmio import CsrMatrix
    rng = np.random.default_rng(5)
    n = 700
    rows = []
    for i in range(n):
        k = 0 if (i // 8) % 3 == 1 else int(rng.integers(1, 40))
        rows.append(np.sort(rng.choice(n, size=k, replace=False)))
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(c) for c in rows])
    ci = np.concatenate(rows).astype(np.int32)
    m = CsrMatrix(n, n, rp, ci, rng.uniform(-1, 1, ci.size))
    x = rng.uniform(-1, 1, n)
    for r in (1, 2, 4, 8):
        s = spc5.csr_to_spc5(m, r, 8)
        y_ref = _oracle_y(m, r, 8, x)
        y = np.zeros(n)
        spc5.spmv_spc5_scalar(s, x, y)  # accumulates into y (kernels.py:121-143)
        once = y.copy()
        spc5.spmv_spc5_scalar(s, x, y)  # (split panels add their carries after y: not bitwise 2x)
        assert_close(m, y / 2, y_ref, x, f"lbr acc twice {r}")
        assert_close(m, once, y_ref, x, f"lbr acc {r}")
        keep = np.full(n, 7.0)
        spc5.spmv_spc5_scalar(s, x, keep)
        assert np.all(keep[rp[1:] == rp[:-1]] == 7.0)  # rows of empty panels untouched
        y2 = spc5.spmv(s, x)
        assert_close(m, y2, y_ref, x, f"lbr overwrite {r}")
        assert np.all(y2[rp[1:] == rp[:-1]] == 0.0)
