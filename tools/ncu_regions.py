"""Group a kernel's SASS into runs of equal execution count (basic-block-ish
regions) and print the heavy ones: instruction share and stall share.

usage: python tools/ncu_regions.py REP KERNEL_SUBSTRING [min_share]
"""
import csv
import io
import subprocess
import sys

rep, ksub = sys.argv[1], sys.argv[2]
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
for blk in out.split('"Kernel Name",')[1:]:
    name, _, body = blk.partition("\n")
    if ksub not in name:
        continue
    rows = list(csv.reader(io.StringIO(body)))
    h = rows[0]
    iS, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    groups = []
    for r in rows[1:]:
        try:
            a, e, s = int(r[0], 16), int(float(r[iE] or 0)), float(r[iS] or 0)
        except (ValueError, IndexError):
            continue
        if groups and groups[-1][2] == e:
            groups[-1][1] = a
            groups[-1][3] += 1
            groups[-1][4] += s
        else:
            groups.append([a, a, e, 1, s, r[1].strip()[:40]])
    tot = sum(g[2] * g[3] for g in groups) or 1
    st = sum(g[4] for g in groups) or 1
    print(name[:100], f"total inst {tot}")
    for g in groups:
        if g[2] * g[3] > thr * tot or g[4] > thr * st:
            print(f"{g[0] & 0xfffff:05x}-{g[1] & 0xfffff:05x} exec={g[2]:9d} n={g[3]:4d} "
                  f"inst={g[2] * g[3] / tot:6.1%} stall={g[4] / st:6.1%}  {g[5]}")
    break
