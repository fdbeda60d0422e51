"""Host workload twins (CPU): the BASELINE config 3/4 generators have the
shapes and distributions BASELINE.json names.  The device generators are
checked against these twins bit for bit in tests/test_gpu_parity.py."""

import numpy as np

from paper_2307_14774_b200.workloads import (FEM_NBR, FEM_NODES, PL_N, fem_neighbours, fem_rows,
                                             powerlaw_len_table, powerlaw_rows)


def test_powerlaw_length_table():
    t = powerlaw_len_table()
    assert t.dtype == np.int32 and len(t) == 4096
    assert t.min() >= 1 and t.max() <= 8192
    assert np.all(np.diff(t) >= 0)  # quantiles ascend
    assert abs(float(t.mean()) - 16.0) < 0.5  # lognormal mean 16


def test_powerlaw_rows_shape():
    lo, hi = 100_000, 102_000
    m = powerlaw_rows(lo, hi)
    assert m.num_rows == hi - lo and m.num_cols == PL_N
    assert m.values.dtype == np.float32
    lens = np.diff(m.row_ptr)
    assert lens.min() >= 1
    assert 12 < lens.mean() < 20
    near = 0
    for i in range(m.num_rows):
        c = m.col_idx[m.row_ptr[i]:m.row_ptr[i + 1]].astype(np.int64)
        assert np.all(np.diff(c) > 0)  # sorted, distinct
        assert c.min() >= 0 and c.max() < PL_N
        near += int(np.sum(np.abs(c - (lo + i)) <= 4096))
    assert 0.75 < near / m.nnz < 0.9  # ~80 % within +-4096 of the diagonal
    assert np.all(np.abs(m.values) < 1.0)


def test_powerlaw_rows_are_slices():
    a = powerlaw_rows(5000, 5100)
    b = powerlaw_rows(5050, 5070)
    off = a.row_ptr[50]
    assert np.array_equal(b.col_idx, a.col_idx[off:off + b.nnz])
    assert b.values.tobytes() == a.values[off:off + b.nnz].tobytes()


def test_fem_rows_shape():
    for q in (0, 1, 5000, FEM_NODES - 1):
        nb = fem_neighbours(q)
        assert len(nb) == FEM_NBR and np.all(np.diff(nb) > 0)
        assert q not in nb and np.all(np.abs(nb - q) <= 2048)
        assert nb.min() >= 0 and nb.max() < FEM_NODES
    m = fem_rows(3 * 700, 3 * 710)
    assert np.all(np.diff(m.row_ptr) == 81)
    for i in range(m.num_rows):
        c = m.col_idx[m.row_ptr[i]:m.row_ptr[i + 1]]
        assert np.all(np.diff(c) > 0)
        assert np.array_equal(c.reshape(27, 3) % 3, np.tile(np.arange(3), (27, 1)))  # 3x3 blocks
    # the three dof rows of a node share the node pattern
    assert np.array_equal(m.col_idx[0:81], m.col_idx[81:162])
    v = fem_rows(0, 3000).values
    assert abs(float(v.mean())) < 0.02 and abs(float(v.std()) - 1.0) < 0.02


def test_stencil_box_twin():
    """n x n x nz box (weak scaling): nz = n is the cube; a slab's rows reach
    the neighbouring slabs and interior rows keep all 27 entries."""
    from paper_2307_14774_b200.workloads import stencil27_rows
    n = 6
    cube = stencil27_rows(n, 0, n ** 3)
    same = stencil27_rows(n, 0, n ** 3, nz=n)
    assert np.array_equal(cube.row_ptr, same.row_ptr)
    assert np.array_equal(cube.col_idx, same.col_idx)
    box = stencil27_rows(n, 0, 3 * n ** 3, nz=3 * n)
    assert box.num_cols == 3 * n ** 3
    # the first row of slab 1 (z = n) couples to z = n - 1 (slab 0) and z = n + 1
    i = n ** 3 + n * n + n + 1  # interior in x, y; z = n + 1
    c = box.col_idx[box.row_ptr[i]:box.row_ptr[i + 1]]
    assert len(c) == 27 and c.min() == i - n * n - n - 1 and c.max() == i + n * n + n + 1
    j = n ** 3 + n + 1  # z = n, slab edge
    c = box.col_idx[box.row_ptr[j]:box.row_ptr[j + 1]]
    assert len(c) == 27 and c.min() < n ** 3
