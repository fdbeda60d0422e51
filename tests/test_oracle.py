"""Pin the C oracle (oracle/spc5_oracle.c) against the reference's own outputs.

Golden vectors come from running the reference (tests/golden/make_golden.py):
the hand matrix of tests/test_blocks.py:23-36, the edge-block case of
tests/test_kernels.py:152-162, the adversarial cancellation of
tests/test_kernels.py:233-254, 30 ``random_csr`` matrices, config 1 and the
27-point stencil.  Only after these pass is the oracle trusted as the checker
of the CUDA path.
"""

import numpy as np
import pytest

from golden_io import (Csr, case_x, config1, digest, expected_small, fmt_keys, small_case,
                       small_case_names, stencil)
from oracle import oracle

CASES = small_case_names()


def test_hand_matrix_known_answers():
    # tests/test_blocks.py:23-36 (reference), restated
    m = small_case("hand")
    s = oracle.csr_to_spc5(m, 1, 4)
    assert s.block_rowptr.tolist() == [0, 2, 3, 3, 4]
    assert s.block_colidx.tolist() == [0, 6, 1, 6]
    assert s.block_masks.tolist() == [0b1101, 0b0001, 0b0001, 0b0011]
    assert s.values.tolist() == [1, 2, 3, 4, 5, 6, 7]
    s = oracle.csr_to_spc5(m, 2, 4)
    assert s.block_rowptr.tolist() == [0, 2, 3]
    assert s.block_colidx.tolist() == [0, 6, 6]
    assert s.block_masks.tolist() == [0b1101, 0b0010, 0b0001, 0, 0, 0b0011]
    assert s.values.tolist() == [1, 2, 3, 5, 4, 6, 7]
    y = np.zeros(4)
    oracle.spmv_spc5_scalar(s, np.ones(8), y)
    assert y.tolist() == [10, 5, 0, 13]


def test_edge_block_known_answer():
    m = small_case("edge")
    s = oracle.csr_to_spc5(m, 2, 8)
    y = np.zeros(2)
    oracle.spmv_spc5_scalar(s, np.array([9.0, 9, 9, 1, 2]), y)
    assert y.tolist() == [5.0, 6.0]


@pytest.mark.parametrize("name", CASES)
def test_conversion_and_scalar_bit_exact(name):
    m = small_case(name)
    rec = expected_small()["cases"][name]
    x = case_x(name, m)
    for r, vs, f in fmt_keys(rec):
        s = oracle.csr_to_spc5(m, r, vs)
        assert s.num_blocks == f["num_blocks"], (name, r, vs)
        assert digest(s.block_rowptr) == f["rowptr"], (name, r, vs)
        assert digest(s.block_colidx) == f["colidx"], (name, r, vs)
        assert digest(s.block_masks) == f["masks"], (name, r, vs)
        assert digest(s.values) == f["values"], (name, r, vs)
        y = np.zeros(m.num_rows, dtype=m.values.dtype)
        oracle.spmv_spc5_scalar(s, x, y)
        assert digest(y) == f["y_scalar"], (name, r, vs)
        for w, ranges in f["partition"].items():
            assert oracle.partition_by_nnz(s, int(w)) == [tuple(t) for t in ranges]
        if "values_list" in f:
            assert s.block_colidx.tolist() == f["colidx_list"]
            assert s.block_masks.tolist() == f["masks_list"]


@pytest.mark.parametrize("name", CASES)
def test_exact_reference(name):
    m = small_case(name)
    rec = expected_small()["cases"][name]
    y, a = oracle.csr_reference(m, case_x(name, m))
    assert digest(y) == rec["csr_reference_y"], name
    assert digest(a) == rec["csr_reference_abs"], name


def test_scalar_threads_bitwise():
    for name in ("tall", "longrows", "rand05", "dense16"):
        m = small_case(name)
        x = case_x(name, m)
        for r, vs in ((1, 8), (4, 16), (8, 4)):
            s = oracle.csr_to_spc5(m, r, vs)
            y1 = np.zeros(m.num_rows, m.values.dtype)
            oracle.spmv_spc5_scalar(s, x, y1, threads=1)
            for t in (2, 3, 8):
                yt = np.zeros(m.num_rows, m.values.dtype)
                oracle.spmv_spc5_scalar(s, x, yt, threads=t)
                assert yt.tobytes() == y1.tobytes()


def test_config1_matches_reference():
    from paper_2307_14774_b200.workloads import config1 as gen1, x_vector
    c1 = config1()
    m = gen1(c1["seed"])
    assert digest(m.row_ptr) == c1["row_ptr"]
    assert digest(m.col_idx) == c1["col_idx"]
    assert digest(m.values) == c1["values"]
    x = x_vector(8192, "f64", c1["x_seed"])
    y, _ = oracle.csr_reference(m, x)
    assert digest(y) == c1["csr_reference_y"]
    for r, vs, f in fmt_keys(c1):
        s = oracle.csr_to_spc5(m, r, vs)
        assert (digest(s.block_rowptr), digest(s.block_colidx), digest(s.block_masks),
                digest(s.values)) == (f["rowptr"], f["colidx"], f["masks"], f["values"])
        y = np.zeros(8192)
        oracle.spmv_spc5_scalar(s, x, y, threads=4)
        assert digest(y) == f["y_scalar"]
        for w, ranges in f["partition"].items():
            assert oracle.partition_by_nnz(s, int(w)) == [tuple(t) for t in ranges]


def test_stencil_matches_reference():
    from paper_2307_14774_b200.workloads import stencil27, x_vector
    for key, rec in stencil()["cases"].items():
        m = stencil27(rec["n"], rec["precision"])
        assert m.nnz == rec["nnz"] == (3 * rec["n"] - 2) ** 3
        assert digest(m.row_ptr) == rec["row_ptr"] and digest(m.col_idx) == rec["col_idx"]
        assert digest(m.values) == rec["values"]
        x = x_vector(m.num_cols, rec["precision"])
        for r, vs, f in fmt_keys(rec):
            s = oracle.csr_to_spc5(m, r, vs)
            assert s.num_blocks == f["num_blocks"]
            assert (digest(s.block_rowptr), digest(s.block_colidx), digest(s.block_masks),
                    digest(s.values)) == (f["rowptr"], f["colidx"], f["masks"], f["values"])
            y = np.zeros(m.num_rows, m.values.dtype)
            oracle.spmv_spc5_scalar(s, x, y)
            assert digest(y) == f["y_scalar"], (key, r, vs)


def test_stencil_block_count_formula():
    # nb(r, vs) = (n/r)(3n-2)^2 if r+2 <= vs else 2(n/r)(3n-2)^2
    from paper_2307_14774_b200.workloads import stencil27
    n = 16
    m = stencil27(n)
    for r in (1, 2, 4, 8):
        s = oracle.csr_to_spc5(m, r, 8)
        expect = (n // r) * (3 * n - 2) ** 2 * (1 if r + 2 <= 8 else 2)
        assert s.num_blocks == expect


def test_corruption_detected():
    m = small_case("tall")
    s = oracle.csr_to_spc5(m, 1, 8)
    s.block_masks = s.block_masks.copy()
    i = int(np.flatnonzero(s.block_masks != 0xFF)[0])
    mask = int(s.block_masks[i])
    unset = next(k for k in range(8) if not (mask >> k) & 1)
    s.block_masks[i] = mask | (1 << unset)
    with pytest.raises((RuntimeError, IndexError)):
        oracle.spmv_spc5_scalar(s, np.ones(m.num_cols), np.zeros(m.num_rows))


def test_unsorted_csr_rejected():
    bad = Csr(1, 8, np.array([0, 2], np.int64), np.array([5, 3], np.int32), np.ones(2))
    with pytest.raises(ValueError):
        oracle.csr_to_spc5(bad, 1, 8)


def test_offsets_and_popcounts_golden():
    """oracle.block_value_offsets and the package's host mask_popcounts against the
    reference's block_value_offsets / mask_popcounts (kernels.py:82-96), and the
    footprint comparison formula (blocks.py:192-198)."""
    import paper_2307_14774_b200 as spc5
    for name in small_case_names():
        m = small_case(name)
        for r, vs, f in fmt_keys(expected_small()["cases"][name]):
            s = oracle.csr_to_spc5(m, r, vs)
            assert digest(oracle.block_value_offsets(s)) == f["offsets"], (name, r, vs)
            assert digest(spc5.mask_popcounts(s.block_masks)) == f["popcounts"], (name, r, vs)
            vb = m.values.dtype.itemsize
            csr_bytes = (m.num_rows + 1) * 4 + m.nnz * 4 + m.nnz * vb
            spc5_bytes = (m.nnz * vb + s.num_blocks * 4 + s.num_blocks * r * (1 if vs <= 8 else 2)
                          + (s.num_panels + 1) * 4)
            assert [csr_bytes, spc5_bytes] == f["footprint_comparison"], (name, r, vs)
