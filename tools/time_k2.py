"""K2 timing only (experiments; no validation): any config's formats, CUDA events.

usage: python tools/time_k2.py [formats e.g. "1,8;2,8"] [reps] [config]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_14774_b200 import _native as nat  # noqa: E402
from paper_2307_14774_b200.blocks import torch_stream  # noqa: E402
from paper_2307_14774_b200.workloads import CONFIGS  # noqa: E402

fmts = [tuple(int(v) for v in f.split(",")) for f in
        (sys.argv[1] if len(sys.argv) > 1 else "1,8;2,8;4,8;8,8").split(";")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
cfg = int(sys.argv[3]) if len(sys.argv) > 3 else 2
prec = CONFIGS[cfg]["precision"]
tdt = torch.float64 if prec == "f64" else torch.float32
mats, nr, nc, x, _, _, _ = bench.build_matrices(cfg, fmts, validate=False)
y = torch.empty(nr, dtype=tdt, device="cuda")
out = {}
for f in fmts:
    h = mats[f].handle().ptr
    st = torch_stream()
    for _ in range(5):
        nat.check(nat.lib.spc5_spmv(h, x.data_ptr(), y.data_ptr(), 0, st))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        nat.check(nat.lib.spc5_spmv(h, x.data_ptr(), y.data_ptr(), 0, st))
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    gbs = bench.alg_bytes(mats[f], 8 if prec == "f64" else 4) / us / 1e3
    out[f"c{cfg}b{f}"] = [round(us, 1), round(gbs / bench.peaks()[0], 3)]
print(json.dumps(out))
