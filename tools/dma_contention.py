"""DMA contention probe (experiments): K2 device time alone and while H2D /
D2H copies run on other streams (config 2, beta(1,8), full and 1/8 range)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_14774_b200 import _native as nat  # noqa: E402
from paper_2307_14774_b200.workloads import x_vector  # noqa: E402

mats, nr, nc = bench.build_matrices(2, [(1, 8)])
s = mats[(1, 8)]
h = s.handle().ptr
x = torch.from_numpy(x_vector(nc)).to("cuda")
y = torch.empty(nr, dtype=torch.float64, device="cuda")
hp = torch.empty(64 << 20, dtype=torch.uint8, pin_memory=True)
dbuf = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
sk, sc = torch.cuda.Stream(), torch.cuda.Stream()
np_ = s.num_panels


def run(mode, rng):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(sc):
        for _ in range(8):
            if mode == "h2d":
                dbuf.copy_(hp, non_blocking=True)
            elif mode == "d2h":
                hp.copy_(dbuf, non_blocking=True)
    with torch.cuda.stream(sk):
        e0.record()
        for _ in range(20):
            if rng:
                nat.check(nat.lib.spc5_spmv(h, x.data_ptr(), y.data_ptr(), 0, sk.cuda_stream))
            else:
                nat.check(nat.lib.spc5_spmv(h, x.data_ptr(), y.data_ptr(), 0, sk.cuda_stream))
        e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 20 * 1e3


for mode in ("none", "h2d", "d2h", "none"):
    print(mode, f"{run(mode, False):.1f} us per full product")


def copy_time(mode, kernels):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(sk):
        for _ in range(kernels):
            nat.check(nat.lib.spc5_spmv(h, x.data_ptr(), y.data_ptr(), 0, sk.cuda_stream))
    with torch.cuda.stream(sc):
        e0.record()
        for _ in range(2):
            if mode == "h2d":
                dbuf[:16 << 20].copy_(hp[:16 << 20], non_blocking=True)
            else:
                hp[:16 << 20].copy_(dbuf[:16 << 20], non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    return 2 * (16 << 20) / (e0.elapsed_time(e1) * 1e-3) / 1e9


for mode in ("h2d", "d2h"):
    print(mode, f"alone {copy_time(mode, 0):.1f} GB/s, under K2 {copy_time(mode, 20):.1f} GB/s")
