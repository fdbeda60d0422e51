#!/bin/bash
# Round profile refresh on the GPU box (run under gpurun): GPU tests, the bench
# line, the ncu launch list, one ncu --set full capture per config-2 format,
# the summaries under profiles/, and the other configs' bench lines.
# usage: bash tools/refresh_profiles.sh ROUND   (outputs in gpurun_out/prof/)
R=${1:-r1}
O=gpurun_out/prof
mkdir -p $O /tmp/prof
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
  > $O/ncu_launches.log 2>&1
reps=""
for f in "1,8" "2,8" "4,8" "8,8"; do
  n=b${f/,/_}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:spmv_kernel \
    --launch-skip 3 --launch-count 1 -o /tmp/prof/$n -f python tools/time_k2.py "$f" 1 2 \
    > $O/ncu_$n.log 2>&1
  python tools/ncu_stalls.py /tmp/prof/$n.ncu-rep spmv_kernel 30 > $O/stalls_$n.txt 2>&1
  reps="$reps${reps:+,}/tmp/prof/$n.ncu-rep"
done
python tools/summarize_profiles.py $R $O/launches.csv $reps > $O/summary.txt 2>&1
cp profiles/launches_$R.csv profiles/ncu_$R.csv profiles/traffic.json $O/ 2>/dev/null
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
for c in 1 3 4 6; do
  timeout 900 python bench.py --config $c --steps 50 --warmup 5 --no-e2e > $O/bench_c$c.json 2>&1
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>&1
timeout 1500 python bench.py --config 5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
  > $O/bench_c5.json 2>&1
ls -la $O
