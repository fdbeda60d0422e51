"""Summarise an ncu --page source CSV: hottest lines by stall samples / instructions.

usage: python tools/ncu_top.py REPORT [kernel-substring] [cuda|sass] [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ksub = sys.argv[2] if len(sys.argv) > 2 else ""
mode = sys.argv[3] if len(sys.argv) > 3 else "cuda"
N = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", mode],
                     capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name",')
for blk in blocks[1:]:
    name, _, body = blk.partition("\n")
    if ksub and ksub not in name:
        continue
    rows = list(csv.reader(io.StringIO(body)))
    hdr = rows[0]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iI = hdr.index("Instructions Executed")
    src = hdr.index("Source")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    data = []
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        try:
            data.append((float(r[iS] or 0), float(r[iI] or 0), r[src].strip()[:110],
                         {hdr[i]: float(r[i] or 0) for i in stall_cols}))
        except ValueError:
            pass
    tot_s = sum(d[0] for d in data) or 1
    tot_i = sum(d[1] for d in data) or 1
    print(f"== {name[:100]}  samples={tot_s:.0f} inst={tot_i:.0f}")
    agg = {}
    for d in data:
        for k, v in d[3].items():
            agg[k] = agg.get(k, 0) + v
    print("   stalls:", ", ".join(f"{k[6:]}={v / tot_s:.0%}" for k, v in
                                 sorted(agg.items(), key=lambda t: -t[1])[:8]))
    for d in sorted(data, key=lambda t: -t[0])[:N]:
        top = sorted(d[3].items(), key=lambda t: -t[1])[:2]
        print(f"{d[0] / tot_s:6.1%} {d[1] / tot_i:6.1%}  {d[2]}   [{', '.join(k[6:] for k, v in top if v)}]")
