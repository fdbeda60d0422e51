#!/bin/bash
# K2 tuning sweep (experiments, no validation): variants x env settings, config 2.
# usage: bash tools/sweep_k2.sh "m2 m3" "SPC5_WPC=8,SPC5_TEAM=2 SPC5_WPC=4" [formats]
cp paper_2307_14774_b200/libspc5_b200.so /tmp/libspc5_b200.so.orig
for v in $1; do
  cp variants/$v/libspc5_b200.so paper_2307_14774_b200/libspc5_b200.so
  for cfg in $2; do
    echo "$v $cfg $(env ${cfg//,/ } timeout 300 python tools/time_k2.py $3 2>&1 | tail -1)"
  done
done
cp /tmp/libspc5_b200.so.orig paper_2307_14774_b200/libspc5_b200.so
