#!/bin/bash
# bench configs under env settings (experiments, no e2e / cpu legs)
# usage: bash tools/cfg_sweep.sh "1 2 3 4" "SPC5_WIN_KB=6 SPC5_WIN_KB=10"
for cfg in $2; do for c in $1; do
  echo "$cfg $(env ${cfg//,/ } python bench.py --config $c --steps 30 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); print(d["config"]["workload"], round(d["value"],1), {k:(round(v["us"],1), round(v["frac"],3)) for k,v in d["formats"].items()})
except Exception as e: print("FAIL", e)')"
done; done
