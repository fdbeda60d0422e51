#!/bin/bash
# ncu --set full captures of one K2 launch per (config, format), plus the
# x-gather counters (LSU sectors/request, L2 hit rate of L1TEX reads).
# Each capture's command first runs plain (&&) so ncu only sees a command that
# exited 0 on this box.  The reports stay on the box (/tmp/prof, tens of MB
# each); their raw-metric CSV and stall summary come back in gpurun_out/prof.
# usage: bash tools/prof_configs.sh "3:1,16 3:4,16 4:8,8 5:1,8 5:8,8"
O=gpurun_out/prof
mkdir -p $O /tmp/prof
EXTRA="l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum"
for item in $1; do
  c=${item%%:*}
  f=${item#*:}
  tag=c${c}_b${f/,/_}
  timeout 900 python tools/time_k2.py "$f" 1 $c > $O/$tag.plain.log 2>&1 &&
  timeout 1200 ncu --set full --metrics $EXTRA --import-source on --clock-control none \
    -k regex:spmv_kernel -s 5 -c 1 -o /tmp/prof/$tag -f python tools/time_k2.py "$f" 1 $c \
    > $O/$tag.ncu.log 2>&1
  echo "$tag rc=$?"
  ncu -i /tmp/prof/$tag.ncu-rep --page raw --csv > $O/$tag.raw.csv 2>/dev/null
  python tools/ncu_stalls.py /tmp/prof/$tag.ncu-rep spmv_kernel 30 > $O/$tag.stalls.txt 2>&1
done
