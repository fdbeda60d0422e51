"""Host-side matrix types and the reference's synthetic generators.

``CsrMatrix`` keeps the field names and contract of the reference type
(/root/reference/pkg/src/spc5/mmio.py:84-100): ``row_ptr`` int64[n+1],
``col_idx`` int32[nnz] strictly increasing per row, ``values`` f32/f64.

``make_random`` / ``make_dense`` / ``make_identity`` reproduce the reference
generators draw for draw (mmio.py:304-379) so that config 1 of BASELINE.json
(``make_random(8192, 8192, 16, 0.0, seed)``) is the same matrix here as in the
reference; tests/golden/config1.json pins that with digests taken from the
reference itself.  Matrix Market parsing and SuiteSparse fetching are out of
scope for this build ("Out of scope").
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

DTYPES = {"f32": np.float32, "f64": np.float64}

# mmio.py:41-43 -- value seed of the dense generator (value depends on (i, j) only)
DENSE_VALUE_SEED = np.uint64(0x5BC5C0DEB10C55ED)


def dtype_for(precision: str) -> np.dtype:
    try:
        return np.dtype(DTYPES[precision])
    except KeyError:
        raise ValueError(f"unknown precision {precision!r}; expected 'f32' or 'f64'") from None


@dataclass
class CsrMatrix:
    """Compressed sparse row matrix with sorted, unique column indices per row."""

    num_rows: int
    num_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return len(self.values)

    @property
    def precision(self) -> str:
        return "f32" if self.values.dtype == np.float32 else "f64"


def mix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def make_dense(n: int, precision: str = "f64") -> CsrMatrix:
    """Fully populated n x n matrix, value(i, j) from splitmix64 of (i, j) (mmio.py:304-322)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    dtype = dtype_for(precision)
    i = np.arange(n, dtype=np.uint64)
    key = (i[:, None] << np.uint64(32)) ^ i[None, :] ^ DENSE_VALUE_SEED
    unit = (mix64(key.ravel()) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return CsrMatrix(n, n, np.arange(0, n * n + 1, n, dtype=np.int64),
                     np.tile(np.arange(n, dtype=np.int32), n), unit.astype(dtype))


def make_identity(n: int, precision: str = "f64") -> CsrMatrix:
    if n < 1:
        raise ValueError("n must be >= 1")
    return CsrMatrix(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32),
                     np.ones(n, dtype=dtype_for(precision)))


def make_random(n_rows: int, n_cols: int, nnz_per_row: int, clustering: float,
                seed: int, precision: str = "f64") -> CsrMatrix:
    """Random CSR with a contiguous run of round(clustering*k) columns per row.

    Same generator stream as the reference (mmio.py:336-379): per row one
    ``integers`` draw for the run start (when the run is non-empty) and one
    ``choice(..., replace=False)`` for the scattered rest, then every value
    in a single ``uniform(-1, 1)`` draw after all rows.
    """
    dtype = dtype_for(precision)
    if n_rows < 0 or n_cols < 0:
        raise ValueError("dimensions must be non-negative")
    if nnz_per_row > n_cols:
        raise ValueError(f"nnz_per_row={nnz_per_row} infeasible for {n_cols} columns")
    if not 0.0 <= clustering <= 1.0:
        raise ValueError("clustering must be in [0, 1]")
    rng = np.random.default_rng(seed)
    k = nnz_per_row
    run_len = int(round(clustering * k))
    scattered = k - run_len
    rows = []
    for _ in range(n_rows):
        if k == 0:
            rows.append(np.empty(0, dtype=np.int64))
            continue
        start = int(rng.integers(0, n_cols - run_len + 1)) if run_len > 0 else 0
        run = np.arange(start, start + run_len, dtype=np.int64)
        if scattered > 0:
            # draw from the columns outside the run, then shift over it
            picks = rng.choice(n_cols - run_len, size=scattered, replace=False).astype(np.int64)
            picks[picks >= start] += run_len
            rows.append(np.sort(np.concatenate([run, picks])))
        else:
            rows.append(run)
    row_ptr = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum([len(c) for c in rows], out=row_ptr[1:])
    col_idx = (np.concatenate(rows) if rows else np.empty(0, np.int64)).astype(np.int32)
    values = rng.uniform(-1.0, 1.0, size=len(col_idx)).astype(dtype)
    return CsrMatrix(n_rows, n_cols, row_ptr, col_idx, values)
