"""e2e probe (experiments): spc5_spmv_host wall time per call vs its parts."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_14774_b200 import _native as nat  # noqa: E402
from paper_2307_14774_b200.blocks import torch_stream  # noqa: E402
from paper_2307_14774_b200.workloads import x_vector  # noqa: E402

mats, nr, nc = bench.build_matrices(2, [(1, 8)])
s = mats[(1, 8)]
h = s.handle().ptr
xp = torch.empty(nc, dtype=torch.float64, pin_memory=True)
xp.numpy()[:] = x_vector(nc)
yp = torch.empty(nr, dtype=torch.float64, pin_memory=True)
st = torch_stream()
for _ in range(3):
    nat.check(nat.lib.spc5_spmv_host(h, xp.data_ptr(), yp.data_ptr(), 0, st))
reps = 50
t0 = time.perf_counter()
for _ in range(reps):
    nat.check(nat.lib.spc5_spmv_host(h, xp.data_ptr(), yp.data_ptr(), 0, st))
t1 = time.perf_counter()
print(f"spc5_spmv_host: {(t1 - t0) / reps * 1e3:.3f} ms per call")
xd = torch.empty(nc, dtype=torch.float64, device="cuda")
yd = torch.empty(nr, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    xd.copy_(xp, non_blocking=True)
    nat.check(nat.lib.spc5_spmv(h, xd.data_ptr(), yd.data_ptr(), 0, st))
    yp.copy_(yd, non_blocking=True)
    torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"serial copy+kernel+copy: {(t1 - t0) / reps * 1e3:.3f} ms per call")
# device-only: the 8 range products of the pipeline vs one full product
ranges = [tuple(r) for r in np.array_split(np.arange(s.num_panels), 8)]
bounds = [(int(r[0]), int(r[-1]) + 1) for r in ranges]
xd.copy_(xp)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    for lo, hi in bounds:
        nat.check(nat.lib.spc5_spmv_panels(h, lo, hi, xd.data_ptr(), yd.data_ptr(), 0, st))
e1.record()
torch.cuda.synchronize()
print(f"8 range products: {e0.elapsed_time(e1) / reps * 1e3:.1f} us per call")
e0.record()
for _ in range(reps):
    nat.check(nat.lib.spc5_spmv(h, xd.data_ptr(), yd.data_ptr(), 0, st))
e1.record()
torch.cuda.synchronize()
print(f"1 full product: {e0.elapsed_time(e1) / reps * 1e3:.1f} us per call")
