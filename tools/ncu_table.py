"""Key counters of the K2 captures in gpurun_out/prof/*.raw.csv (tools/prof_configs.sh).

usage: python tools/ncu_table.py DIR [alg_bytes.json]
Prints one row per capture: duration, DRAM bytes (vs algorithmic when known),
DRAM throughput, warps active, issue active, instructions, x-gather sectors
per request and the L2 hit rate of the L1TEX (x-gather) reads.
"""
import csv
import glob
import io
import json
import os
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1,
         "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3, "s": 1e6, "": 1, "%": 1, "inst": 1, "sector": 1, "request": 1, "warp": 1,
         "register/thread": 1}


def val(hdr, units, row, name):
    if name not in hdr:
        return None
    i = hdr.index(name)
    try:
        v = float(row[i].replace(",", ""))
    except ValueError:
        return None
    return v * SCALE.get(units[i], 1)


d = sys.argv[1]
alg = json.load(open(sys.argv[2])) if len(sys.argv) > 2 else {}
print("| capture | us (ncu) | DRAM MB | alg MB | DRAM/alg | DRAM % peak | warps active % | issue active % | inst (M) | x sectors/req | x L2 hit % | L1 hit % | regs |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for f in sorted(glob.glob(os.path.join(d, "*.raw.csv"))):
    tag = os.path.basename(f)[:-8]
    rows = list(csv.reader(io.StringIO(open(f).read())))
    if len(rows) < 3:
        continue
    hdr, units, r = rows[0], rows[1], rows[2]
    g = lambda n: val(hdr, units, r, n)  # noqa: E731
    dram = (g("dram__bytes_read.sum") or 0) + (g("dram__bytes_write.sum") or 0)
    sec = g("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum")
    req = g("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum")
    hit = g("lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum")
    tot = g("lts__t_sectors_srcunit_tex_op_read.sum")
    a = alg.get(tag)
    print(f"| {tag} | {g('gpu__time_duration.sum'):.1f} | {dram / 1e6:.1f} | "
          f"{a / 1e6 if a else float('nan'):.1f} | {dram / a if a else float('nan'):.3f} | "
          f"{g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
          f"{g('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
          f"{g('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
          f"{g('smsp__inst_executed.sum') / 1e6:.1f} | "
          f"{sec / req if sec and req else float('nan'):.2f} | "
          f"{100 * hit / tot if hit is not None and tot else float('nan'):.1f} | "
          f"{g('l1tex__t_sector_hit_rate.pct'):.1f} | {g('launch__registers_per_thread'):.0f} |")
