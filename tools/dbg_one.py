"""Debug helper: one small golden case, one format, several products (for compute-sanitizer)."""
import sys
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np
from golden_io import small_case, case_x
from oracle import oracle
import paper_2307_14774_b200 as spc5
name, r, vs = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
m = small_case(name)
x = case_x(name, m)
s = spc5.csr_to_spc5(m, r, vs)
ref = oracle.csr_to_spc5(m, r, vs)
yr = np.zeros(m.num_rows, dtype=x.dtype); oracle.spmv_spc5_scalar(ref, x, yr)
_, a = oracle.csr_reference(m, x)
for rep in range(4):
    y = np.zeros(m.num_rows, m.values.dtype)
    spc5.spmv_spc5_scalar(s, x, y)
    err = np.abs(y.astype(np.float64) - yr) / np.where(a > 0, a, 1)
    print(rep, "bad rows", np.nonzero(err > 1e-5)[0].tolist(), flush=True)
