"""ctypes front-end of the C oracle (oracle/spc5_oracle.c).

TEST INFRASTRUCTURE ONLY -- the checker, never the thing measured or shipped.
Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this module.  The product package (paper_2307_14774_b200) never does.

Each function restates one reference function (file:line in
/root/reference/pkg/src/spc5/) on numpy inputs:

  csr_to_spc5          blocks.py:96-143
  block_value_offsets  kernels.py:91-96
  spmv_spc5_scalar     kernels.py:121-143, 205-213 (incl. the cursor check)
  partition_by_nnz     parallel.py:31-52
  csr_reference        kernels.py:233-250
  scaled_error         kernels.py:284-312 (the VERIFY_FACTOR budget)
  spc5_to_csr          blocks.py:146-168 (numpy restatement, small inputs)

Parity of the restatement is pinned against tests/golden/ (made by importing
the reference, see tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"
SRC_PATH = HERE / "spc5_oracle.c"

VALID_R = (1, 2, 4, 8)
VALID_VS = (4, 8, 16)
VERIFY_FACTOR = 8.0
ABS_FLOOR = {"f32": 1e-30, "f64": 1e-300}

_i64p = ctypes.POINTER(ctypes.c_int64)
_lib = None


def build(force: bool = False) -> Path:
    """Compile the oracle with gcc (unfused arithmetic, OpenMP)."""
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < SRC_PATH.stat().st_mtime:
        tmp = LIB_PATH.with_suffix(f".{os.getpid()}.tmp")
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC",
                               "-shared", "-o", str(tmp), str(SRC_PATH)])
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(LIB_PATH))
        vp = ctypes.c_void_p
        L.oracle_convert_count.argtypes = [ctypes.c_int64, ctypes.c_int64, vp, vp,
                                           ctypes.c_int, ctypes.c_int, vp]
        L.oracle_convert_fill.argtypes = [ctypes.c_int64, ctypes.c_int64, vp, vp, vp,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_int, vp,
                                          vp, vp, vp]
        L.oracle_block_value_offsets.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                                 vp, vp]
        L.oracle_partition_by_nnz.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                              ctypes.c_int, vp, vp, ctypes.c_int, vp]
        for name in ("oracle_spmv_scalar_f64", "oracle_spmv_scalar_f32"):
            fn = getattr(L, name)
            fn.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp, vp,
                           vp, ctypes.c_int]
            fn.restype = ctypes.c_int64
        for name in ("oracle_csr_exact_f64", "oracle_csr_exact_f32"):
            getattr(L, name).argtypes = [ctypes.c_int64, vp, vp, vp, vp, vp, vp]
        L.oracle_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def mask_dtype(vs: int):
    return np.dtype(np.uint8) if vs <= 8 else np.dtype(np.uint16)


@dataclass
class OracleSpc5:
    """Plain holder with the reference Spc5Matrix field names (blocks.py:51-62)."""

    num_rows: int
    num_cols: int
    r: int
    vs: int
    block_rowptr: np.ndarray
    block_colidx: np.ndarray
    block_masks: np.ndarray
    values: np.ndarray

    @property
    def num_panels(self) -> int:
        return len(self.block_rowptr) - 1

    @property
    def num_blocks(self) -> int:
        return len(self.block_colidx)

    @property
    def nnz(self) -> int:
        return len(self.values)


def _csr_arrays(m):
    rp = np.ascontiguousarray(m.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(m.col_idx, dtype=np.int32)
    va = np.ascontiguousarray(m.values)
    return rp, ci, va


def csr_to_spc5(m, r: int, vs: int) -> OracleSpc5:
    """blocks.py:96-143 restated (see spc5_oracle.c)."""
    if r not in VALID_R or vs not in VALID_VS:
        raise ValueError(f"bad shape r={r} vs={vs}")
    rp, ci, va = _csr_arrays(m)
    n = int(m.num_rows)
    num_panels = (n + r - 1) // r
    counts = np.zeros(num_panels, dtype=np.int64)
    st = lib().oracle_convert_count(n, int(m.num_cols), _p(rp), _p(ci), r, vs, _p(counts))
    if st:
        raise ValueError(f"oracle conversion rejected the CSR input (status {st})")
    rowptr = np.zeros(num_panels + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    nb = int(rowptr[-1])
    colidx = np.zeros(nb, dtype=np.uint32)
    masks = np.zeros(nb * r, dtype=mask_dtype(vs))
    vals = np.empty_like(va)
    if nb:
        st = lib().oracle_convert_fill(n, int(m.num_cols), _p(rp), _p(ci), _p(va),
                                       va.dtype.itemsize, r, vs, _p(rowptr), _p(colidx),
                                       _p(masks), _p(vals))
        if st:
            raise ValueError(f"oracle conversion failed (status {st})")
    else:
        vals = va.copy()
    return OracleSpc5(n, int(m.num_cols), r, vs, rowptr, colidx, masks, vals)


def block_value_offsets(s) -> np.ndarray:
    masks = np.ascontiguousarray(s.block_masks)
    out = np.zeros(s.num_blocks + 1, dtype=np.int64)
    lib().oracle_block_value_offsets(s.num_blocks, s.r, s.vs, _p(masks), _p(out))
    return out


def spmv_spc5_scalar(s, x, y, threads: int = 1) -> None:
    """y[:num_rows] += A.x in the reference's scalar order (kernels.py:205-213)."""
    if len(x) < s.num_cols or len(y) < s.num_rows:
        raise ValueError("x/y too short")
    dt = s.values.dtype
    xv = np.ascontiguousarray(np.asarray(x, dtype=dt))
    offs = block_value_offsets(s)
    if offs[-1] > s.nnz:
        raise IndexError("value cursor runs past the value array")
    if s.num_blocks:
        # the highest column any set bit touches must exist in x (numpy would
        # raise IndexError inside the reference loop)
        orm = np.bitwise_or.reduce(s.block_masks.reshape(s.num_blocks, s.r).astype(np.int64),
                                   axis=1)
        hi_bit = np.full(s.num_blocks, -1, dtype=np.int64)
        for k in range(s.vs):
            hi_bit[((orm >> k) & 1) == 1] = k
        top = s.block_colidx.astype(np.int64) + hi_bit
        if np.any(top[hi_bit >= 0] >= len(xv)):
            raise IndexError("mask bit addresses x past its end")
    ypad = np.zeros(s.num_panels * s.r, dtype=dt)
    fn = lib().oracle_spmv_scalar_f64 if dt == np.float64 else lib().oracle_spmv_scalar_f32
    vals = np.ascontiguousarray(s.values)
    end = fn(s.num_panels, s.r, s.vs, _p(np.ascontiguousarray(s.block_rowptr, dtype=np.int64)),
             _p(np.ascontiguousarray(s.block_colidx)), _p(np.ascontiguousarray(s.block_masks)),
             _p(vals), _p(xv), _p(ypad), int(threads))
    if end != s.nnz:
        raise RuntimeError(f"value cursor ended at {end}, expected {s.nnz}")
    y[:s.num_rows] += ypad[:s.num_rows]


class ScalarRunner:
    """The C scalar kernel bound to one matrix/x, checks done once (CPU-baseline timing).

    run() is exactly oracle_spmv_scalar_* over all panels (kernels.py:121-143)
    into a preallocated ypad; it returns the value cursor.
    """

    def __init__(self, s, x, threads: int = 1):
        self.s = s
        dt = s.values.dtype
        self.x = np.ascontiguousarray(np.asarray(x, dtype=dt))
        self.rp = np.ascontiguousarray(s.block_rowptr, dtype=np.int64)
        self.ci = np.ascontiguousarray(s.block_colidx)
        self.mk = np.ascontiguousarray(s.block_masks)
        self.va = np.ascontiguousarray(s.values)
        self.ypad = np.zeros(s.num_panels * s.r, dtype=dt)
        self.threads = int(threads)
        self.fn = lib().oracle_spmv_scalar_f64 if dt == np.float64 else lib().oracle_spmv_scalar_f32
        if block_value_offsets(s)[-1] != s.nnz:
            raise RuntimeError("value cursor mismatch")

    def run(self) -> int:
        self.ypad[:] = 0
        return int(self.fn(self.s.num_panels, self.s.r, self.s.vs, _p(self.rp), _p(self.ci),
                           _p(self.mk), _p(self.va), _p(self.x), _p(self.ypad), self.threads))

    def y(self):
        return self.ypad[:self.s.num_rows]


def partition_by_nnz(s, workers: int) -> list[tuple[int, int]]:
    """parallel.py:31-52 restated; returns the list of (lo, hi) panel ranges."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    out = np.zeros(2 * workers, dtype=np.int64)
    st = lib().oracle_partition_by_nnz(s.num_panels, s.num_blocks, s.r, s.vs,
                                       _p(np.ascontiguousarray(s.block_rowptr, dtype=np.int64)),
                                       _p(np.ascontiguousarray(s.block_masks)), workers, _p(out))
    if st:
        raise ValueError("partition failed")
    return [(int(out[2 * k]), int(out[2 * k + 1])) for k in range(workers)]


def csr_reference(m, x) -> tuple[np.ndarray, np.ndarray]:
    """kernels.py:233-250: exactly summed products (in matrix precision) and sum|p|."""
    rp, ci, va = _csr_arrays(m)
    xv = np.ascontiguousarray(np.asarray(x, dtype=va.dtype))
    y = np.zeros(m.num_rows, dtype=np.float64)
    a = np.zeros(m.num_rows, dtype=np.float64)
    fn = lib().oracle_csr_exact_f64 if va.dtype == np.float64 else lib().oracle_csr_exact_f32
    fn(int(m.num_rows), _p(rp), _p(ci), _p(va), _p(xv), _p(y), _p(a))
    return y, a


def scaled_error(m, y, x) -> np.ndarray:
    """Per-row error in units of nnz_row*eps*sum|p| (+floor), kernels.py:284-306."""
    prec = "f32" if m.values.dtype == np.float32 else "f64"
    eps = float(np.finfo(m.values.dtype).eps)
    y_ref, abs_ref = csr_reference(m, x)
    nnz_row = np.maximum(np.diff(np.asarray(m.row_ptr, dtype=np.int64)), 1).astype(np.float64)
    budget = nnz_row * eps * abs_ref + ABS_FLOOR[prec]
    return np.abs(np.asarray(y[:m.num_rows], dtype=np.float64) - y_ref) / budget


def relative_error(y_gpu, y_ref, abs_ref) -> np.ndarray:
    """|y_gpu - y_ref| / sum_j |a_ij x_j| -- the north-star per-entry tolerance metric."""
    denom = np.where(abs_ref > 0, abs_ref, 1.0)
    return np.abs(np.asarray(y_gpu, np.float64) - np.asarray(y_ref, np.float64)) / denom


def spc5_to_csr(s):
    """blocks.py:146-168 restated in numpy: returns (row_ptr, col_idx, values)."""
    if s.num_blocks == 0:
        return (np.zeros(s.num_rows + 1, dtype=np.int64), np.empty(0, dtype=np.int32),
                s.values.copy())
    r, vs = s.r, s.vs
    bp = np.repeat(np.arange(s.num_panels, dtype=np.int64), np.diff(s.block_rowptr))
    slot_row = np.repeat(bp * r, r) + np.tile(np.arange(r, dtype=np.int64), s.num_blocks)
    slot_anchor = np.repeat(s.block_colidx.astype(np.int64), r)
    bits = (s.block_masks[:, None].astype(np.int64) >> np.arange(vs)) & 1
    si, bit = np.nonzero(bits)
    rows = slot_row[si]
    cols = (slot_anchor[si] + bit).astype(np.int32)
    order = np.argsort(rows, kind="stable")
    row_ptr = np.zeros(s.num_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=s.num_rows), out=row_ptr[1:])
    return row_ptr, cols[order], s.values[order]


def threads() -> int:
    return int(lib().oracle_threads())
