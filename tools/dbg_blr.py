"""Debug helper: per-format bad rows of the small golden cases (GPU vs oracle)."""
import sys
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np
from golden_io import small_case, case_x, expected_small, fmt_keys
from oracle import oracle
import paper_2307_14774_b200 as spc5
names = sys.argv[1:] or ["longrows", "longrows_f32"]
for rep in range(3):
    for name in names:
        m = small_case(name)
        x = case_x(name, m)
        for r, vs, f in fmt_keys(expected_small()["cases"][name]):
            s = spc5.csr_to_spc5(m, r, vs)
            y = np.zeros(m.num_rows, m.values.dtype)
            spc5.spmv_spc5_scalar(s, x, y)
            ref = oracle.csr_to_spc5(m, r, vs)
            yr = np.zeros(m.num_rows, dtype=x.dtype); oracle.spmv_spc5_scalar(ref, x, yr)
            _, a = oracle.csr_reference(m, x)
            err = np.abs(y.astype(np.float64) - yr) / np.where(a > 0, a, 1)
            bad = np.nonzero(err > 1e-5)[0].tolist()
            if bad:
                print(rep, name, r, vs, "bad rows", bad, flush=True)
print("done")
