"""Print SASS lines executed >= thresh times per unit, in address order."""
import csv
import io
import subprocess
import sys

rep, ksub, unit = sys.argv[1], sys.argv[2], float(sys.argv[3])
thresh = float(sys.argv[4]) if len(sys.argv) > 4 else 0.3
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
for blk in out.split('"Kernel Name",')[1:]:
    name, _, body = blk.partition("\n")
    if ksub not in name:
        continue
    rows = list(csv.reader(io.StringIO(body)))
    h = rows[0]
    iI, src = h.index("Instructions Executed"), h.index("Source")
    iS = h.index("Warp Stall Sampling (All Samples)")
    for r in rows[1:]:
        try:
            n = float(r[iI] or 0)
        except ValueError:
            continue
        if n / unit >= thresh:
            print(f"{n / unit:5.2f} {float(r[iS] or 0):6.0f}  {r[src].strip()[:100]}")
    break
