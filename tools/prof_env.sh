#!/bin/bash
# ncu --set full of one K2 launch per (env, config, format); env entries like
# "SPC5_FVR=0" ("-" = none).  usage: bash tools/prof_env.sh "ENV:CFG:FMT ..."
O=gpurun_out/prof
mkdir -p $O /tmp/prof
for item in $1; do
  IFS=: read -r envs c f <<< "$item"
  [ "$envs" = "-" ] && envs=""
  tag=c${c}_b${f/,/_}${envs:+_${envs//[=,]/_}}
  env ${envs//,/ } timeout 900 python tools/time_k2.py "$f" 1 $c > $O/$tag.plain.log 2>&1 &&
  env ${envs//,/ } timeout 1200 ncu --set full --import-source on --clock-control none \
    -k regex:spmv_kernel -s 5 -c 1 -o /tmp/prof/$tag -f python tools/time_k2.py "$f" 1 $c \
    > $O/$tag.ncu.log 2>&1
  echo "$tag rc=$?"
  ncu -i /tmp/prof/$tag.ncu-rep --page raw --csv > $O/$tag.raw.csv 2>/dev/null
  python tools/ncu_stalls.py /tmp/prof/$tag.ncu-rep spmv_kernel 40 > $O/$tag.stalls.txt 2>&1
  ncu -i /tmp/prof/$tag.ncu-rep --page source --csv --print-source sass > $O/$tag.sass.csv 2>/dev/null
  gzip -f $O/$tag.sass.csv
done
