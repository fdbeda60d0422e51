"""e2e stage probe (experiments): a few spc5_spmv_host calls on config 2, for
an ncu launch list of the pipeline's range products."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_14774_b200 import _native as nat  # noqa: E402
from paper_2307_14774_b200.blocks import torch_stream  # noqa: E402
from paper_2307_14774_b200.workloads import x_vector  # noqa: E402

f = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1,8").split(","))
mats, nr, nc = bench.build_matrices(2, [f])
h = mats[f].handle().ptr
xp = torch.empty(nc, dtype=torch.float64, pin_memory=True)
xp.numpy()[:] = x_vector(nc)
yp = torch.empty(nr, dtype=torch.float64, pin_memory=True)
st = torch_stream()
for _ in range(4):
    nat.check(nat.lib.spc5_spmv_host(h, xp.data_ptr(), yp.data_ptr(), 0, st))
torch.cuda.synchronize()
