"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
K1 (conversion) and K2 (products, every chunk mode) over the golden small
cases, a giant-row matrix (split chunks, carry + fixup), power-law / FEM row
slices (flat value ranges), a 20^3 stencil (lane-per-panel-row), range
products and the host-buffer pipeline, each checked against the oracle so a
run that "passes" the tool also computed the right thing.

usage: compute-sanitizer --tool memcheck python tools/sanitize_small.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2307_14774_b200 as spc5  # noqa: E402
from golden_io import small_case, small_case_names  # noqa: E402
from oracle import oracle  # noqa: E402
from test_gpu_parity import giant_row_matrix  # noqa: E402
from paper_2307_14774_b200.workloads import fem_rows, powerlaw_rows, stencil27  # noqa: E402


def check(m, r, vs, label, workers=(1, 3)):
    x = np.random.default_rng(7).uniform(-1, 1, m.num_cols).astype(m.values.dtype)
    s = spc5.csr_to_spc5(m, r, vs)
    ref = oracle.csr_to_spc5(m, r, vs)
    for f in ("block_rowptr", "block_colidx", "block_masks", "values"):
        assert np.array_equal(getattr(s, f), getattr(ref, f)), (label, r, vs, f)
    y = spc5.spmv(s, x)
    yr = np.zeros(m.num_rows, dtype=m.values.dtype)
    oracle.spmv_spc5_scalar(ref, x, yr)
    _, a = oracle.csr_reference(m, x)
    tol = 1e-12 if m.values.dtype == np.float64 else 1e-5
    e = oracle.relative_error(y, yr, a)
    assert e.size == 0 or float(e.max()) <= tol, (label, r, vs, float(e.max()))
    prec = "f64" if m.values.dtype == np.float64 else "f32"
    for w in workers:
        yp = np.zeros(m.num_rows, dtype=m.values.dtype)
        spc5.spmv_parallel(s, x, yp, spc5.KernelConfig(precision=prec), w)
        assert yp.tobytes() == y.tobytes(), (label, r, vs, w)


def main():
    n = 0
    for name in small_case_names():
        m = small_case(name)
        for r in (1, 2, 4, 8):
            for vs in (4, 8, 16):
                check(m, r, vs, name, workers=(2,))
                n += 1
    for prec in ("f64", "f32"):
        m = giant_row_matrix(prec)
        for r, vs in ((1, 4), (2, 8), (4, 16)):
            check(m, r, vs, "giant", workers=(2, 5))
            n += 1
    for m, fmts in ((powerlaw_rows(1000, 1600, precision="f32"), ((1, 16), (2, 16), (4, 16))),
                    (fem_rows(3000, 3600), ((4, 8), (8, 8))),
                    (stencil27(20), ((1, 8), (2, 8), (4, 8), (8, 8)))):
        for r, vs in fmts:
            check(m, r, vs, "slice")
            n += 1
    print(f"sanitize workload ok: {n} conversions + products")


if __name__ == "__main__":
    main()
