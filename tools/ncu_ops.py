"""Instruction mix per kernel from an ncu source page (per unit of `div`)."""
import collections
import csv
import io
import subprocess
import sys

rep, ksub, div = sys.argv[1], sys.argv[2], float(sys.argv[3])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
for blk in out.split('"Kernel Name",')[1:]:
    name, _, body = blk.partition("\n")
    if ksub not in name:
        continue
    rows = list(csv.reader(io.StringIO(body)))
    h = rows[0]
    iI, src = h.index("Instructions Executed"), h.index("Source")
    byop, tot = collections.Counter(), 0
    for r in rows[1:]:
        try:
            n = float(r[iI] or 0)
        except ValueError:
            continue
        toks = r[src].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        byop[op.split(".")[0]] += n
        tot += n
    print(name[:90], f"total/unit={tot / div:.1f}")
    print("  " + "  ".join(f"{op}:{n / div:.1f}" for op, n in byop.most_common(45)))
    break
