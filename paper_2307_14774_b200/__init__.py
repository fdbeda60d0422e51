"""B200-native SPC5 beta(r, vs) sparse matrix/vector product (arXiv 2307.14774).

Drop-in for the hot path of the reference package ``spc5``
(/root/reference/pkg/src/spc5/__init__.py:11-21 names): CSR->SPC5 conversion,
the SpMV entry points, the nnz-balanced partition and the timing harness,
backed by hand-written sm_100a CUDA kernels in ``libspc5_b200.so`` (C ABI:
include/spc5_b200.h).  The library is loaded on the first device call
(``_native.load()``) and a missing library raises ImportError there; there is
no CPU fallback.
"""

from . import _native  # noqa: F401  (loads libspc5_b200.so on first use)
from .blocks import (VALID_R, VALID_VS, FillingStats, Spc5Matrix, csr_to_spc5,
                     csr_to_spc5_device, filling_stats, footprint_comparison, load_spc5,
                     load_spc5_shard, save_spc5_shard,
                     mask_dtype, save_spc5, spc5_to_csr, validate_spc5)
from .harness import (CSV_VERSION_LINE, BenchRecord, CostModelFit, InsufficientDataError,
                      ValidationError, fit_cost_model, read_records, run_bench, run_kernel,
                      spearman_rank_correlation, write_records, write_scatter)
from .kernels import (KernelConfig, SpmvResult, VerifyReport, block_value_offsets,
                      csr_reference, mask_popcounts, spmv, spmv_csr, spmv_spc5_scalar,
                      spmv_spc5_vector,
                      verify_against_oracle)
from .mmio import CsrMatrix, make_dense, make_identity, make_random
from .parallel import Partition, partition_by_nnz, spmv_parallel

__version__ = "0.1.0"

__all__ = [
    "CSV_VERSION_LINE", "CostModelFit", "InsufficientDataError", "fit_cost_model",
    "read_records", "spearman_rank_correlation", "write_records", "write_scatter",
    "BenchRecord", "CsrMatrix", "FillingStats", "KernelConfig", "Partition", "Spc5Matrix",
    "SpmvResult", "VALID_R", "VALID_VS", "ValidationError", "VerifyReport",
    "block_value_offsets", "csr_reference", "csr_to_spc5", "csr_to_spc5_device",
    "filling_stats", "footprint_comparison", "load_spc5", "load_spc5_shard", "save_spc5_shard", "make_dense", "make_identity",
    "make_random", "mask_dtype", "mask_popcounts", "partition_by_nnz", "run_bench",
    "run_kernel", "save_spc5", "spc5_to_csr", "spmv", "spmv_csr", "spmv_parallel",
    "spmv_spc5_scalar",
    "spmv_spc5_vector", "validate_spc5", "verify_against_oracle",
]
