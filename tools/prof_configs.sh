#!/bin/bash
# ncu --set full captures of one K2 launch per (config, format), plus the
# x-gather counters (LSU sectors/request, L2 hit rate of L1TEX reads).
# Each capture's command first runs plain (&&) so ncu only sees a command that
# exited 0 on this box.  Outputs: gpurun_out/prof/<tag>.ncu-rep + logs.
# usage: bash tools/prof_configs.sh "3:1,16 3:4,16 4:8,8 5:1,8 5:8,8"
O=gpurun_out/prof
mkdir -p $O
EXTRA="l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum"
for item in $1; do
  c=${item%%:*}
  f=${item#*:}
  tag=c${c}_b${f/,/_}
  timeout 900 python tools/time_k2.py "$f" 1 $c > $O/$tag.plain.log 2>&1 &&
  timeout 1200 ncu --set full --metrics $EXTRA --import-source on --clock-control none \
    -k regex:spmv_kernel -s 5 -c 1 -o $O/$tag -f python tools/time_k2.py "$f" 1 $c \
    > $O/$tag.ncu.log 2>&1
  echo "$tag rc=$?"
done
