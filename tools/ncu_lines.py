"""Executed instructions and stall samples per CUDA source line of one kernel:
joins an ncu SASS source page (--page source --print-source sass --csv) with
the line info of the local build (nvdisasm -g of the same cubin).

usage: python tools/ncu_lines.py SASS_CSV[.gz] ALL_SASS(nvdisasm -g output) FUNC_SUBSTR SRC [TOP]
"""
import collections
import csv
import gzip
import io
import re
import sys

csvf, sassf, fsub, srcf = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
txt = (gzip.open(csvf, "rt") if csvf.endswith(".gz") else open(csvf)).read()
blk = txt.split('"Kernel Name",')[1]
rows = list(csv.reader(io.StringIO(blk.partition("\n")[2])))
h = rows[0]
iA, iE, iS = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
base = int(rows[1][iA], 16)
execd, samp = {}, {}
for r in rows[1:]:
    try:
        off = int(r[iA], 16) - base
        execd[off] = float(r[iE] or 0)
        samp[off] = float(r[iS] or 0)
    except (ValueError, IndexError):
        continue
# local line info
line_of, infn, cur = {}, False, None
for ln in open(sassf):
    if ".section\t.text." in ln:
        infn = fsub in ln
        continue
    if not infn:
        continue
    if "//##" in ln:
        m = re.search(r'File "([^"]+)", line (\d+)', ln)
        if m and srcf.split("/")[-1] in m.group(1):
            cur = int(m.group(2))
        elif m:
            cur = m.group(1).split("/")[-1] + ":" + m.group(2)
        else:
            cur = None
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+\S', ln)
    if m:
        line_of[int(m.group(1), 16)] = cur
src = open(srcf).read().splitlines()
E, S = collections.Counter(), collections.Counter()
for off, e in execd.items():
    ln = line_of.get(off)
    E[ln] += e
    S[ln] += samp.get(off, 0)
te, ts = sum(E.values()), sum(S.values()) or 1
print(f"total warp instructions executed {te:.4g}; unmapped {E[None]:.3g}")
for ln, e in E.most_common(top):
    s = src[ln - 1].strip()[:70] if isinstance(ln, int) else (ln or "?")
    print(f"{ln!s:>5} {e / te:6.1%} {S[ln] / ts:6.1%}  {s}")
