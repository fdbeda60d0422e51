"""Stall-reason totals and the top stalled SASS lines of one kernel in an ncu report.

usage: python tools/ncu_stalls.py REP KERNEL_SUBSTRING [TOP]
"""
import csv
import io
import subprocess
import sys

rep, ksub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
for blk in out.split('"Kernel Name",')[1:]:
    name, _, body = blk.partition("\n")
    if ksub not in name:
        continue
    rows = list(csv.reader(io.StringIO(body)))
    h = rows[0]
    cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    iS, iSrc, iA = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Address")
    tot = {h[i]: 0.0 for i in cols}
    lines = []
    for r in rows[1:]:
        try:
            s = float(r[iS] or 0)
        except (ValueError, IndexError):
            continue
        for i in cols:
            tot[h[i]] += float(r[i] or 0)
        lines.append((s, r))
    all_s = sum(tot.values()) or 1.0
    print(name[:110])
    print("  ".join(f"{k[6:]}={v / all_s:.1%}" for k, v in sorted(tot.items(), key=lambda t: -t[1])
                    if v / all_s > 0.01))
    for s, r in sorted(lines, key=lambda t: -t[0])[:top]:
        why = sorted(((float(r[i] or 0), h[i][6:]) for i in cols), reverse=True)[:2]
        print(f"{s / all_s:6.1%} {r[iA]:>6} {r[iSrc].strip()[:70]:70s} "
              + " ".join(f"{n}:{v / max(s, 1):.0%}" for v, n in why if v))
    break
