"""SpMV entry points of the reference ``spc5.kernels`` module, run on the GPU.

``spmv_spc5_scalar`` / ``spmv_spc5_vector`` (kernels.py:205-230) keep their
signatures, checks and exceptions; both launch K2 (csrc/spmv_kernel.cuh).  The
strategy / reduction / x_load toggles of :class:`KernelConfig` select CPU SIMD
idioms (expand vs compact, hsum vs multi-reduce) that have no counterpart on a
GPU warp; they are validated and recorded, and only ``precision`` changes what
runs (kernels.py:47-72, 219-223).

Numerics: products are formed in the matrix precision as in the reference and
row sums are kept in fp64; for f32 matrices in lane-per-panel-row chunks the
few products of one slot call (<= 27) are first summed with f32 FMAs and that
partial is added to the fp64 row sum.  Every sum is
reduced in an order fixed by the plan, so results are deterministic run to run
and across ``spmv_parallel`` worker counts; they differ from the reference's
strictly sequential order by rounding only (tolerance: |dy_i| <= 1e-12 (f64) /
1e-5 (f32) * sum_j |a_ij x_j|).

x / y may be numpy arrays (copied through the host-buffer C entry point) or
torch CUDA tensors (used in place, on torch's current stream).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .blocks import Spc5Matrix, as_spc5, csr_to_spc5, torch_stream
from .mmio import DTYPES

__all__ = ["KernelConfig", "SpmvResult", "VerifyReport", "spmv", "spmv_csr", "spmv_spc5_scalar",
           "spmv_spc5_vector", "csr_reference", "verify_against_oracle",
           "block_value_offsets", "mask_popcounts", "VERIFY_FACTOR"]

STRATEGIES = ("scalar", "expand", "compact")
REDUCTIONS = ("hsum", "multi")
X_LOADS = ("partial", "single")
VERIFY_FACTOR = 8.0
_ABS_FLOOR = {"f32": 1e-30, "f64": 1e-300}


@dataclass(frozen=True)
class KernelConfig:
    """Strategy selection for one SpMV run (kernels.py:47-72)."""

    strategy: str = "compact"
    reduction: str = "hsum"
    x_load: str = "partial"
    precision: str = "f64"

    def __post_init__(self):
        if self.strategy not in STRATEGIES:
            raise ValueError(f"strategy must be one of {STRATEGIES}")
        if self.reduction not in REDUCTIONS:
            raise ValueError(f"reduction must be one of {REDUCTIONS}")
        if self.x_load not in X_LOADS:
            raise ValueError(f"x_load must be one of {X_LOADS}")
        if self.precision not in DTYPES:
            raise ValueError("precision must be 'f32' or 'f64'")

    @property
    def dtype(self):
        return np.dtype(DTYPES[self.precision])


@dataclass
class SpmvResult:
    y: object
    flops: int
    elapsed: float


def mask_popcounts(masks: np.ndarray) -> np.ndarray:
    """Per-mask popcount (kernels.py:82-88)."""
    return np.bitwise_count(np.asarray(masks).astype(np.uint16)).astype(np.int64)


def block_value_offsets(s) -> np.ndarray:
    """Cumulative value offset per block, offsets[-1] == nnz (kernels.py:91-96), on the GPU."""
    import torch
    s = as_spc5(s)
    h = s.handle()
    out = torch.empty(h.info.num_blocks + 1, dtype=torch.int64, device="cuda")
    nat.check(nat.lib.spc5_block_value_offsets(h.ptr, out.data_ptr(), torch_stream()))
    return out.cpu().numpy()


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _check_xy(num_rows: int, num_cols: int, x, y) -> None:
    if len(x) < num_cols:
        raise ValueError(f"x has {len(x)} elements, matrix needs {num_cols}")
    if len(y) < num_rows:
        raise ValueError(f"y has {len(y)} elements, matrix needs {num_rows}")


def _run(s: Spc5Matrix, x, y, accumulate: bool) -> None:
    """Dispatch one product into y (numpy or torch CUDA), y[:num_rows] only."""
    st = torch_stream()
    h = s.handle(st)
    dt = s.dtype
    if _is_torch(x) or _is_torch(y):
        import torch
        tdt = torch.float64 if dt == np.float64 else torch.float32
        xd = x if _is_torch(x) else torch.from_numpy(np.ascontiguousarray(x, dtype=dt))
        xd = xd.to(device="cuda", dtype=tdt).contiguous()
        if _is_torch(y) and y.is_cuda and y.dtype == tdt and y.is_contiguous():
            nat.check(nat.lib.spc5_spmv(h.ptr, xd.data_ptr(), y.data_ptr(), int(accumulate), st))
            return
        tmp = torch.zeros(s.num_rows, dtype=tdt, device="cuda")
        nat.check(nat.lib.spc5_spmv(h.ptr, xd.data_ptr(), tmp.data_ptr(), 0, st))
        if accumulate:
            y[:s.num_rows] += tmp.to(y.device) if _is_torch(y) else tmp.cpu().numpy()
        else:
            y[:s.num_rows] = tmp.to(y.device) if _is_torch(y) else tmp.cpu().numpy()
        return
    xh = np.ascontiguousarray(np.asarray(x)[:s.num_cols], dtype=dt)
    if isinstance(y, np.ndarray) and y.dtype == dt and y.flags.c_contiguous and y.flags.writeable:
        nat.check(nat.lib.spc5_spmv_host(h.ptr, xh.ctypes.data, y.ctypes.data,
                                         int(accumulate), st))
        return
    tmp = np.zeros(s.num_rows, dtype=dt)
    nat.check(nat.lib.spc5_spmv_host(h.ptr, xh.ctypes.data, tmp.ctypes.data, 0, st))
    if accumulate:
        y[:s.num_rows] += tmp
    else:
        y[:s.num_rows] = tmp


def spmv_csr(m, x, y) -> None:
    """y[i] += row_i . x for a CsrMatrix (kernels.py:106-118, the reference's CSR
    comparison kernel).  On the GPU a CSR row is a beta(1, c) panel: the matrix
    goes through K1 into beta(1, 8|16) and the product through K2, so the sums
    agree with the sequential loop within the package tolerance."""
    _check_xy(m.num_rows, m.num_cols, x, y)
    from .blocks import csr_to_spc5
    s = csr_to_spc5(m, 1, 8 if m.values.dtype == np.float64 else 16)
    _run(s, x, y, accumulate=True)


def spmv_spc5_scalar(m, x, y) -> None:
    """y[:num_rows] += A.x (kernels.py:205-213); K2 on the GPU."""
    m = as_spc5(m)
    _check_xy(m.num_rows, m.num_cols, x, y)
    _run(m, x, y, accumulate=True)


def spmv_spc5_vector(m, x, y, cfg: KernelConfig) -> None:
    """y[:num_rows] += A.x with the config checks of kernels.py:216-230."""
    if cfg.strategy == "scalar":
        raise ValueError("vector kernel called with the scalar strategy")
    m = as_spc5(m)
    if m.dtype != cfg.dtype:
        raise ValueError(f"matrix is {m.precision} but config asks for {cfg.precision}")
    _check_xy(m.num_rows, m.num_cols, x, y)
    _run(m, x, y, accumulate=True)


def spmv(m, x, y=None):
    """y = A.x (north-star form); returns y (new zeros-initialised array if None)."""
    m = as_spc5(m)
    if y is None:
        if _is_torch(x):
            import torch
            y = torch.empty(m.num_rows, dtype=torch.float64 if m.dtype == np.float64
                            else torch.float32, device=x.device)
        else:
            y = np.empty(m.num_rows, dtype=m.dtype)
    _check_xy(m.num_rows, m.num_cols, x, y)
    _run(m, x, y, accumulate=False)
    return y


# ---- exact oracle + verification (kernels.py:233-317), on the GPU ------------

def csr_reference(m, x) -> tuple[np.ndarray, np.ndarray]:
    """Exactly summed row products (products in matrix precision) and sum |p|."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    rp = torch.from_numpy(np.ascontiguousarray(m.row_ptr, dtype=np.int64)).to(dev)
    ci = torch.from_numpy(np.ascontiguousarray(m.col_idx, dtype=np.int32)).to(dev)
    va = torch.from_numpy(np.ascontiguousarray(m.values)).to(dev)
    xd = torch.from_numpy(np.ascontiguousarray(x, dtype=m.values.dtype)).to(dev)
    y = torch.empty(m.num_rows, dtype=torch.float64, device=dev)
    a = torch.empty(m.num_rows, dtype=torch.float64, device=dev)
    prec = nat.F64 if m.values.dtype == np.float64 else nat.F32
    nat.check(nat.lib.spc5_csr_exact(m.num_rows, prec, rp.data_ptr(), ci.data_ptr(),
                                     va.data_ptr(), xd.data_ptr(), y.data_ptr(), a.data_ptr(),
                                     torch_stream()))
    return y.cpu().numpy(), a.cpu().numpy()


@dataclass
class VerifyReport:
    passed: bool
    max_scaled_error: float
    threshold: float
    worst_row: int
    worst_trial: int
    trials: int

    def __str__(self):
        status = "pass" if self.passed else "FAIL"
        return (f"{status}: max scaled error {self.max_scaled_error:.3g} "
                f"(threshold {self.threshold:g}, worst row {self.worst_row}, "
                f"trial {self.worst_trial}/{self.trials})")


def verify_against_oracle(m, r: int, vs: int, cfg: KernelConfig, trials: int = 3,
                          seed: int = 0, spc5=None) -> VerifyReport:
    """Run the GPU kernel on random x against the exact oracle (kernels.py:269-317)."""
    if m.values.dtype != cfg.dtype:
        raise ValueError(f"matrix is {m.precision} but config asks for {cfg.precision}")
    s = as_spc5(spc5) if spc5 is not None else csr_to_spc5(m, r, vs)
    eps = float(np.finfo(cfg.dtype).eps)
    floor = _ABS_FLOOR[cfg.precision]
    nnz_row = np.maximum(np.diff(np.asarray(m.row_ptr, dtype=np.int64)), 1).astype(np.float64)
    rng = np.random.default_rng(seed)
    worst, worst_row, worst_trial = 0.0, -1, -1
    for t in range(trials):
        x = rng.uniform(-1.0, 1.0, size=m.num_cols).astype(m.values.dtype)
        y = np.zeros(m.num_rows, dtype=m.values.dtype)
        try:
            if cfg.strategy == "scalar":
                spmv_spc5_scalar(s, x, y)
            else:
                spmv_spc5_vector(s, x, y, cfg)
        except (RuntimeError, IndexError, ValueError):
            return VerifyReport(False, float("inf"), VERIFY_FACTOR, -1, t, trials)
        y_ref, abs_ref = csr_reference(m, x)
        scaled = np.abs(y.astype(np.float64) - y_ref) / (nnz_row * eps * abs_ref + floor)
        idx = int(np.argmax(scaled)) if len(scaled) else 0
        if len(scaled) and scaled[idx] > worst:
            worst, worst_row, worst_trial = float(scaled[idx]), idx, t
    return VerifyReport(worst <= VERIFY_FACTOR, worst, VERIFY_FACTOR, worst_row, worst_trial,
                        trials)


def timed(fn, *args) -> float:
    t0 = time.perf_counter()
    fn(*args)
    return time.perf_counter() - t0
