"""Seeded synthetic workloads for the five BASELINE.json configs.

No public matrix suite is used (SuiteSparse is absent offline); these
generators stand in with the shapes, sizes and value distributions that
BASELINE.json names.  Host versions (numpy) live here; the device versions
(``spc5_gen_stencil27`` in csrc/gen.cu) produce bit-identical CSR arrays so a
row slice generated on the host checks a slice of a device-generated matrix
(the sliced oracle).

Values are position keyed, ``v(i, j) = 2*u(i, j) - 1`` with
``u = (splitmix64((i << 32) ^ j ^ seedmix) >> 11) * 2**-53`` -- the scheme the
reference uses for ``make_dense`` (mmio.py:304-322) -- so any row range can be
regenerated without materialising the matrix.  The stencil diagonal is 27
(BASELINE config 2; config 5 leaves it open and uses the same choice).
"""

from __future__ import annotations

import numpy as np

from .mmio import CsrMatrix, dtype_for, make_random, mix64

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
MATRIX_SEED = 0
X_SEED = 1

# (dz, dy, dx) in lexicographic order => columns ascend within a row
STENCIL27 = [(dz, dy, dx) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]


def seed_mix(seed: int) -> np.uint64:
    with np.errstate(over="ignore"):
        return mix64(np.array([np.uint64(seed) + GOLDEN], dtype=np.uint64))[0]


def keyed_uniform(i: np.ndarray, j: np.ndarray, seed: int) -> np.ndarray:
    """U(-1, 1) in float64, a pure function of (i, j, seed)."""
    key = (np.asarray(i, np.uint64) << np.uint64(32)) ^ np.asarray(j, np.uint64) ^ seed_mix(seed)
    u = (mix64(key) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return 2.0 * u - 1.0


def stencil27_rows(n: int, lo: int, hi: int, precision: str = "f64", seed: int = MATRIX_SEED,
                   diag: float = 27.0) -> CsrMatrix:
    """Rows [lo, hi) of the 27-point stencil on an n^3 grid, row = (z*n + y)*n + x.

    Returned as a CSR with ``hi - lo`` rows and ``n**3`` columns; the full
    matrix is ``stencil27_rows(n, 0, n**3)``.
    """
    dtype = dtype_for(precision)
    N = n ** 3
    lo, hi = max(0, lo), min(N, hi)
    i = np.arange(lo, hi, dtype=np.int64)
    z, y, x = i // (n * n), (i // n) % n, i % n
    cols = np.empty((len(i), 27), dtype=np.int64)
    valid = np.empty((len(i), 27), dtype=bool)
    for k, (dz, dy, dx) in enumerate(STENCIL27):
        valid[:, k] = ((z + dz >= 0) & (z + dz < n) & (y + dy >= 0) & (y + dy < n)
                       & (x + dx >= 0) & (x + dx < n))
        cols[:, k] = i + dz * n * n + dy * n + dx
    counts = valid.sum(axis=1)
    row_ptr = np.zeros(len(i) + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    rows_flat = np.broadcast_to(i[:, None], cols.shape)[valid]
    cols_flat = cols[valid]
    vals = keyed_uniform(rows_flat, cols_flat, seed)
    vals[rows_flat == cols_flat] = diag
    return CsrMatrix(len(i), N, row_ptr, cols_flat.astype(np.int32), vals.astype(dtype))


def stencil27(n: int, precision: str = "f64", seed: int = MATRIX_SEED) -> CsrMatrix:
    return stencil27_rows(n, 0, n ** 3, precision, seed)


def stencil27_nnz(n: int) -> int:
    return (3 * n - 2) ** 3


def x_vector(num_cols: int, precision: str = "f64", seed: int = X_SEED) -> np.ndarray:
    """x ~ U(-1, 1) drawn like the reference harness does (bench.py:168-169)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=num_cols).astype(dtype_for(precision))


def config1(seed: int = MATRIX_SEED) -> CsrMatrix:
    """BASELINE config 1: make_random(8192, 8192, 16, 0.0, seed), f64 (use as-is)."""
    return make_random(8192, 8192, 16, 0.0, seed, "f64")


# Config descriptors used by bench.py and the tests.  ``formats`` are (r, vs).
CONFIGS = {
    1: dict(name="random8192_16perrow_f64", precision="f64", formats=[(1, 8)]),
    2: dict(name="stencil27_128cubed_f64", precision="f64", n=128,
            formats=[(1, 8), (2, 8), (4, 8), (8, 8)]),
    3: dict(name="powerlaw_4M_f32", precision="f32", formats=[(1, 16), (2, 16), (4, 16)]),
    4: dict(name="fem_786K_f64", precision="f64", formats=[(4, 8), (8, 8)]),
    5: dict(name="stencil27_400cubed", precision="f64", n=400,
            formats=[(1, 8), (2, 8), (4, 8), (8, 8)]),
}
