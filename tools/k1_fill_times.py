"""K1 device times (count pass, fill pass) of a config's r > 1 formats.  usage: python tools/k1_probe.py CONFIG"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2307_14774_b200.blocks import csr_to_spc5_device
from paper_2307_14774_b200.workloads import CONFIGS, config_shape, device_rows
cfg = CONFIGS[int(sys.argv[1])]
N, C = config_shape(cfg)
rp, ci, va = device_rows(cfg, 0, N)
for (r, vs) in cfg["formats"]:
    if r == 1: continue
    s = csr_to_spc5_device(N, C, rp, ci, va, r, vs)
    t = s.handle().convert_timing()
    print(f"b({r},{vs}) count {t['k1_count_ms']:.2f} fill {t['k1_fill_ms']:.2f} ms", flush=True)
    del s
    torch.cuda.empty_cache()
