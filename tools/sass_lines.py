"""SASS instruction count per source line of one kernel (nvdisasm -g line info).

usage: python tools/sass_lines.py CUBIN FUNC_SUBSTRING SRC_FILE [first_line last_line]
"""
import collections
import re
import subprocess
import sys

cubin, fsub, srcf = sys.argv[1], sys.argv[2], sys.argv[3]
lo = int(sys.argv[4]) if len(sys.argv) > 4 else 0
hi = int(sys.argv[5]) if len(sys.argv) > 5 else 10 ** 9
out = open(cubin).read() if cubin.endswith(".sass") else subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout
src = open(srcf).read().splitlines()
cnt, ops = collections.Counter(), collections.defaultdict(collections.Counter)
infn, cur = False, None
for ln in out.splitlines():
    if ln.startswith("\t.text.") or ".section\t.text." in ln:
        infn = fsub in ln
        continue
    if not infn:
        continue
    m = re.search(r'line (\d+)', ln) if "//##" in ln else None
    if m and srcf.split("/")[-1] in ln:
        cur = int(m.group(1))
        continue
    m = re.match(r'\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)', ln)
    if m and cur is not None:
        cnt[cur] += 1
        ops[cur][m.group(2).split(".")[0]] += 1
tot = sum(v for k, v in cnt.items() if lo <= k <= hi)
print(f"instructions in lines [{lo}, {hi}]: {tot}")
for k in sorted(cnt):
    if lo <= k <= hi:
        top = " ".join(f"{o}:{n}" for o, n in ops[k].most_common(4))
        print(f"{k:5d} {cnt[k]:5d}  {src[k - 1].strip()[:60]:60s} {top}")
