"""Calibration: cuSPARSE CSR SpMV (torch.sparse) and a plain copy on the config-2 matrix."""
import sys, time, json
sys.path.insert(0, '.')
import torch
from paper_2307_14774_b200 import _native as nat
from paper_2307_14774_b200.workloads import x_vector

n = 128
N = n ** 3
rp = torch.empty(N + 1, dtype=torch.int64, device='cuda')
nat.check(nat.lib.spc5_gen_stencil27_rowptr(n, 0, N, rp.data_ptr(), 0))
nnz = int(rp[-1])
ci = torch.empty(nnz, dtype=torch.int32, device='cuda')
va = torch.empty(nnz, dtype=torch.float64, device='cuda')
nat.check(nat.lib.spc5_gen_stencil27_fill(n, 0, N, 1, 0, 27.0, rp.data_ptr(), ci.data_ptr(), va.data_ptr(), 0))
torch.cuda.synchronize()
A = torch.sparse_csr_tensor(rp, ci.to(torch.int64), va, size=(N, N))
x = torch.from_numpy(x_vector(N)).cuda()
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
us = t(lambda: torch.mv(A, x))
csr_bytes = nnz * 12 + (N + 1) * 8 + 2 * N * 8
print(json.dumps({"cusparse_csr_us": us, "gflops": 2 * nnz / us / 1e3, "csr_gbs": csr_bytes / us / 1e3}))
a = torch.empty(2**28, dtype=torch.float32, device='cuda'); b = torch.empty_like(a)
us = t(lambda: b.copy_(a))
print(json.dumps({"copy_1GiB_us": us, "gbs": 2 * a.numel() * 4 / us / 1e3}))
# gather-only: y[i] = sum_j x[col[j]] for CSR structure via torch index_select + segment sum (bandwidth probe)
us = t(lambda: torch.index_select(x, 0, ci.to(torch.int64)))
print(json.dumps({"index_select_us": us}))
