# K1 (conversion) device times per config and format, from the bench line
for c in ${1:-2 3 4 5 7}; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
for k,v in d['formats'].items():
    c=v['conversion']; print('c$c',k,'count %.3f fill %.3f ms  k1 %.0f GB/s frac %.3f plan %.1f ms'%(c['k1_count_ms'],c['k1_fill_ms'],c['k1_gbs'],c['k1_frac'],c['plan_ms']))
"
done
