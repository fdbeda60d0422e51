"""Summarise the ncu launch list and the full capture into profiles/ (round-tagged).

usage: python tools/summarize_profiles.py ROUND LAUNCH_CSV FULL_REP[,FULL_REP...]
Writes profiles/launches_<round>.csv (kernel, launches, total us, share),
profiles/ncu_<round>.csv (key counters per captured K2 launch) and
profiles/traffic.json (dram bytes per K2 launch, read by bench.py).
"""
import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

rnd, launch_csv, rep = sys.argv[1], sys.argv[2], sys.argv[3]
out = Path("profiles")
out.mkdir(exist_ok=True)
rows = [r for r in csv.reader(open(launch_csv)) if len(r) > 10 and r[0] != "ID"]
agg = collections.OrderedDict()
for r in rows:
    name = r[4].split("(")[0].replace("spc5::<unnamed>::", "")
    k = (name, r[7], r[8])
    n, t = agg.get(k, (0, 0.0))
    agg[k] = (n + 1, t + float(r[14]) / 1e3)
tot = sum(t for n, t in agg.values())
with open(out / f"launches_{rnd}.csv", "w") as f:
    w = csv.writer(f)
    w.writerow(["kernel", "block", "grid", "launches", "total_us", "mean_us", "share"])
    for (name, blk, grid), (n, t) in agg.items():
        w.writerow([name, blk, grid, n, f"{t:.1f}", f"{t / n:.1f}", f"{t / tot:.3f}"])
rr = []
for one in rep.split(","):  # one capture per format, rows concatenated
    raw = subprocess.run(["ncu", "-i", one, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    part = list(csv.reader(io.StringIO(raw)))
    if not rr:
        rr = part
    else:
        rr += part[2:]
hdr, units = rr[0], rr[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic"]
idx = [hdr.index(w) for w in want if w in hdr]
traffic = {}
with open(out / f"ncu_{rnd}.csv", "w") as f:
    w = csv.writer(f)
    w.writerow([hdr[i] + (f" [{units[i]}]" if units[i] else "") for i in idx])
    for r in rr[2:]:
        w.writerow([r[i] for i in idx])
        name = r[hdr.index("Kernel Name")]
        rd = float(r[hdr.index("dram__bytes_read.sum")])
        wr = float(r[hdr.index("dram__bytes_write.sum")])
        ur = units[hdr.index("dram__bytes_read.sum")]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(ur, 1)
        traffic[name] = (rd + wr) * scale
json.dump({"config2": {"per_launch_bytes": traffic,
                       "note": f"ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum "
                               f"per K2 launch ({rnd})"}},
          open(out / "traffic.json", "w"), indent=1)
print(open(out / f"launches_{rnd}.csv").read())
print(open(out / f"ncu_{rnd}.csv").read())
