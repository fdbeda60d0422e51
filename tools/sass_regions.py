"""Regions of equal execution count in a K2 capture's SASS page
(gpurun_out/prof/*.sass.csv.gz from tools/prof_env.sh): instruction share,
stall share, first line.  usage: python tools/sass_regions.py FILE.sass.csv.gz [min_share] [--dump LO HI]"""
import csv, gzip, io, sys
f = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else 0.01
body = gzip.open(f, "rt").read()
name, _, body = body.partition("\n")
rows = list(csv.reader(io.StringIO(body)))
h = rows[0]
iS, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
if "--dump" in sys.argv:
    k = sys.argv.index("--dump")
    lo, hi = int(sys.argv[k + 1], 16), int(sys.argv[k + 2], 16)
    for r in rows[1:]:
        a = int(r[0], 16) & 0xfffff
        if lo <= a <= hi:
            print(f"{a:05x} {int(float(r[iE] or 0)):9d} {float(r[iS] or 0):7.0f}  {r[1].strip()}")
    sys.exit()
groups = []
for r in rows[1:]:
    try:
        a, e, s = int(r[0], 16), int(float(r[iE] or 0)), float(r[iS] or 0)
    except (ValueError, IndexError):
        continue
    if groups and groups[-1][2] == e:
        groups[-1][1] = a; groups[-1][3] += 1; groups[-1][4] += s
    else:
        groups.append([a, a, e, 1, s, r[1].strip()[:50]])
tot = sum(g[2] * g[3] for g in groups) or 1
st = sum(g[4] for g in groups) or 1
print(name[:120], f"total inst {tot}")
for g in groups:
    if g[2] * g[3] > thr * tot or g[4] > thr * st:
        print(f"{g[0] & 0xfffff:05x}-{g[1] & 0xfffff:05x} exec={g[2]:9d} n={g[3]:4d} inst={g[2] * g[3] / tot:6.1%} stall={g[4] / st:6.1%}  {g[5]}")
