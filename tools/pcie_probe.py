"""PCIe probe (experiments): pinned H2D / D2H bandwidth alone and concurrently."""
import time

import torch

n = 16 << 20
h = torch.empty(n // 8, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n // 8, dtype=torch.float64, pin_memory=True)
d = torch.empty(n // 8, dtype=torch.float64, device="cuda")
d2 = torch.empty(n // 8, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    d.copy_(h, non_blocking=True)
    h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()


def t(fn, reps=20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


a = t(lambda: d.copy_(h, non_blocking=True))
b = t(lambda: h2.copy_(d2, non_blocking=True))
c = t(both)
print(f"H2D 16MB {a*1e3:.3f} ms ({n/a/1e9:.1f} GB/s)  D2H {b*1e3:.3f} ms ({n/b/1e9:.1f} GB/s)  "
      f"both {c*1e3:.3f} ms")
