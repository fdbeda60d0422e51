"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests:/root/repo \
        python tests/golden/make_golden.py

It imports the reference package ``spc5`` (pure Python + numpy) and its test
helper ``util.random_csr``, runs ``csr_to_spc5`` (blocks.py:96-143),
``spmv_spc5_scalar`` (kernels.py:205-213), ``partition_by_nnz``
(parallel.py:31-52), ``filling_stats`` (blocks.py:176-189) and
``csr_reference`` (kernels.py:233-250) on fixed inputs, and writes:

  inputs_small.npz     CSR inputs of the small cases (hand matrix
                       tests/test_blocks.py:13-19, edge blocks
                       tests/test_kernels.py:152-162, random_csr set, ...)
  expected_small.json  digests / exact arrays of the reference outputs
  config1.json         digests for BASELINE config 1 (make_random 8192^2)
  stencil.json         digests for the 27-point stencil at small n

Nothing at test time reads /root/reference; the tests only read these files.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

import spc5  # the reference package
from spc5.blocks import VALID_R, VALID_VS, csr_to_spc5, filling_stats, footprint_comparison
from spc5.kernels import block_value_offsets, csr_reference, mask_popcounts, spmv_spc5_scalar
from spc5.mmio import CsrMatrix, make_dense, make_identity, make_random
from spc5.parallel import partition_by_nnz
from util import random_csr  # reference tests/util.py:41-51

OUT = Path(__file__).resolve().parent
WORKERS = (1, 2, 3, 4, 7, 8)


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def canon(s):
    """Canonical dtypes of the four format arrays (blocks.py:55-62)."""
    return (s.block_rowptr.astype(np.int64), s.block_colidx.astype(np.uint32),
            s.block_masks, s.values)


def x_for(case_idx: int, m) -> np.ndarray:
    return np.random.default_rng(100 + case_idx).uniform(-1, 1, m.num_cols).astype(m.values.dtype)


def record(m, case_idx: int, full: bool, formats=None) -> dict:
    rec = {"num_rows": m.num_rows, "num_cols": m.num_cols, "nnz": m.nnz,
           "precision": m.precision, "formats": {}}
    x = x_for(case_idx, m)
    y_ref, abs_ref = csr_reference(m, x)
    rec["csr_reference_y"] = digest(y_ref)
    rec["csr_reference_abs"] = digest(abs_ref)
    if full:
        rec["csr_reference_y_list"] = y_ref.tolist()
    for r in VALID_R:
        for vs in VALID_VS:
            if formats is not None and (r, vs) not in formats:
                continue
            s = csr_to_spc5(m, r, vs)
            rp, ci, mk, va = canon(s)
            y = np.zeros(m.num_rows, dtype=m.values.dtype)
            spmv_spc5_scalar(s, x, y)
            st = filling_stats(s)
            f = {"num_blocks": s.num_blocks,
                 "rowptr": digest(rp), "colidx": digest(ci), "masks": digest(mk),
                 "values": digest(va), "y_scalar": digest(y),
                 "filling": st.filling, "footprint_bytes": st.footprint_bytes,
                 "partition": {str(w): partition_by_nnz(s, w).ranges for w in WORKERS},
                 # kernels.py:82-96 and blocks.py:192-198
                 "offsets": digest(block_value_offsets(s)),
                 "popcounts": digest(mask_popcounts(s.block_masks).astype(np.int64)),
                 "footprint_comparison": list(footprint_comparison(m, r, vs))}
            if full:
                f.update(rowptr_list=rp.tolist(), colidx_list=ci.tolist(),
                         masks_list=mk.tolist(), values_list=va.tolist(), y_list=y.tolist(),
                         offsets_list=block_value_offsets(s).tolist())
            rec["formats"][f"{r},{vs}"] = f
    return rec


def small_cases():
    cases = {}
    cases["hand"] = CsrMatrix(4, 8, np.array([0, 4, 5, 5, 7], np.int64),
                              np.array([0, 2, 3, 6, 1, 6, 7], np.int32),
                              np.array([1.0, 2, 3, 4, 5, 6, 7], np.float64))
    cases["edge"] = CsrMatrix(2, 5, np.array([0, 2, 3], np.int64), np.array([3, 4, 4], np.int32),
                              np.array([1.0, 2.0, 3.0], np.float64))
    cases["empty"] = CsrMatrix(3, 3, np.zeros(4, np.int64), np.empty(0, np.int32),
                               np.empty(0, np.float64))
    cases["lastpanel"] = make_random(5, 12, 3, 0.5, seed=8)
    cases["dense16"] = make_dense(16)
    cases["dense16_f32"] = make_dense(16, "f32")
    cases["identity32"] = make_identity(32)
    cases["cancel"] = CsrMatrix(1, 3, np.array([0, 3], np.int64), np.array([0, 1, 2], np.int32),
                                np.array([1e16, 1.0, -1e16], np.float64))
    n, vs = 16, 8
    cases["oneperblock"] = CsrMatrix(n, n * vs, np.arange(n + 1, dtype=np.int64),
                                     np.arange(n, dtype=np.int32) * vs, np.ones(n, np.float64))
    cases["longrows"] = make_random(9, 5000, 700, 0.25, seed=5)
    cases["longrows_f32"] = make_random(11, 3000, 1200, 0.5, seed=6, precision="f32")
    cases["tall"] = make_random(1000, 300, 5, 0.0, seed=7)
    rng = np.random.default_rng(2024)
    for i in range(30):
        prec = "f32" if rng.random() < 0.3 else "f64"
        cases[f"rand{i:02d}"] = random_csr(rng, max_dim=96, precision=prec)
    return cases


def main():
    cases = small_cases()
    arrays = {}
    expected = {"reference_version": spc5.__version__, "workers": list(WORKERS), "cases": {}}
    for idx, (name, m) in enumerate(cases.items()):
        arrays[f"{name}__row_ptr"] = m.row_ptr.astype(np.int64)
        arrays[f"{name}__col_idx"] = m.col_idx.astype(np.int32)
        arrays[f"{name}__values"] = m.values
        arrays[f"{name}__shape"] = np.array([m.num_rows, m.num_cols], np.int64)
        full = name in ("hand", "edge", "cancel", "lastpanel", "empty")
        rec = record(m, idx, full)
        rec["index"] = idx
        expected["cases"][name] = rec
        print(f"case {name}: {m.num_rows}x{m.num_cols} nnz={m.nnz}", file=sys.stderr)
    np.savez_compressed(OUT / "inputs_small.npz", **arrays)
    (OUT / "expected_small.json").write_text(json.dumps(expected, separators=(",", ":")))

    # BASELINE config 1: make_random(8192, 8192, 16, 0.0, seed=0), x seed 1
    m = make_random(8192, 8192, 16, 0.0, 0)
    x = np.random.default_rng(1).uniform(-1, 1, 8192).astype(np.float64)
    c1 = {"seed": 0, "x_seed": 1, "row_ptr": digest(m.row_ptr.astype(np.int64)),
          "col_idx": digest(m.col_idx.astype(np.int32)), "values": digest(m.values),
          "nnz": m.nnz, "formats": {}}
    y_ref, abs_ref = csr_reference(m, x)
    c1["csr_reference_y"] = digest(y_ref)
    for r in VALID_R:
        for vs in (8, 16):
            s = csr_to_spc5(m, r, vs)
            rp, ci, mk, va = canon(s)
            y = np.zeros(8192)
            spmv_spc5_scalar(s, x, y)
            c1["formats"][f"{r},{vs}"] = {
                "num_blocks": s.num_blocks, "rowptr": digest(rp), "colidx": digest(ci),
                "masks": digest(mk), "values": digest(va), "y_scalar": digest(y),
                "footprint_bytes": filling_stats(s).footprint_bytes,
                "offsets": digest(block_value_offsets(s)),
                "partition": {str(w): partition_by_nnz(s, w).ranges for w in (1, 2, 4, 8)}}
            print(f"config1 r={r} vs={vs} nb={s.num_blocks}", file=sys.stderr)
    (OUT / "config1.json").write_text(json.dumps(c1, indent=1))

    # 27-point stencil (generator: paper_2307_14774_b200.workloads, position-keyed values)
    from paper_2307_14774_b200.workloads import stencil27, x_vector
    st = {"cases": {}}
    for n, prec, vsv in ((12, "f64", 8), (12, "f32", 16), (20, "f64", 8)):
        m = stencil27(n, prec)
        m = CsrMatrix(m.num_rows, m.num_cols, m.row_ptr, m.col_idx, m.values)
        x = x_vector(m.num_cols, prec)
        rec = {"n": n, "precision": prec, "nnz": m.nnz, "row_ptr": digest(m.row_ptr),
               "col_idx": digest(m.col_idx), "values": digest(m.values), "formats": {}}
        for r in VALID_R:
            s = csr_to_spc5(m, r, vsv)
            rp, ci, mk, va = canon(s)
            y = np.zeros(m.num_rows, dtype=m.values.dtype)
            spmv_spc5_scalar(s, x, y)
            rec["formats"][f"{r},{vsv}"] = {
                "num_blocks": s.num_blocks, "rowptr": digest(rp), "colidx": digest(ci),
                "masks": digest(mk), "values": digest(va), "y_scalar": digest(y),
                "partition": {str(w): partition_by_nnz(s, w).ranges for w in (1, 2, 4, 8)}}
        st["cases"][f"n{n}_{prec}"] = rec
        print(f"stencil n={n} {prec} done", file=sys.stderr)
    (OUT / "stencil.json").write_text(json.dumps(st, indent=1))


if __name__ == "__main__":
    main()
