"""Host-side cost of one spc5_spmv call and launch-gap check (experiments)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_14774_b200 import _native as nat  # noqa: E402
from paper_2307_14774_b200.blocks import torch_stream  # noqa: E402
from paper_2307_14774_b200.workloads import x_vector  # noqa: E402

fmts = [(1, 8), (2, 8), (4, 8), (8, 8)]
mats, nr, nc = bench.build_matrices(2, fmts)
x = torch.from_numpy(x_vector(nc, "f64")).to("cuda")
ys = {f: torch.empty(nr, dtype=torch.float64, device="cuda") for f in fmts}
hs = {f: mats[f].handle().ptr for f in fmts}
st = torch_stream()
for _ in range(5):
    for f in fmts:
        nat.check(nat.lib.spc5_spmv(hs[f], x.data_ptr(), ys[f].data_ptr(), 0, st))
torch.cuda.synchronize()
# host cost per call: enqueue 400 calls, measure CPU time
t0 = time.perf_counter()
for _ in range(100):
    for f in fmts:
        nat.check(nat.lib.spc5_spmv(hs[f], x.data_ptr(), ys[f].data_ptr(), 0, st))
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue per call {(t1 - t0) / 400 * 1e6:.1f} us; wall per step {(t2 - t0) / 100 * 1e6:.1f} us")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(100):
    for f in fmts:
        nat.check(nat.lib.spc5_spmv(hs[f], x.data_ptr(), ys[f].data_ptr(), 0, st))
e1.record()
torch.cuda.synchronize()
print(f"device per step (no per-launch events) {e0.elapsed_time(e1) * 10:.1f} us")
