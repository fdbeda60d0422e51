# round-2 call 2: K1 timings in the bench line, launch list, remaining ncu
# captures, x persistence-window A/B, compute-sanitizer logs
set -x
O=gpurun_out/c3
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench rc=$?"
for c in 2 3 4 7; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench_c$c.json 2> $O/bench_c$c.err; echo "c$c rc=$?"; done
# x persistence window A/B
for w in 0 1; do
  for c in "5 1,8;2,8;4,8;8,8" "2 1,8;2,8;4,8;8,8" "3 1,16;4,16" "4 4,8;8,8"; do
    set -- $c
    echo "window=$w c$1 $(SPC5_X_WINDOW=$w SPC5_PLAN_DEBUG= timeout 600 python tools/time_k2.py "$2" 30 $1 2>&1 | tail -1)" | tee -a $O/window_ab.txt
  done
done
# launch list of the bench command (after it exited 0 above)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
  > $O/ncu_launches.log 2>&1; echo "launches rc=$?"
bash tools/prof_configs.sh "5:2,8 5:4,8 3:2,16 4:4,8 7:1,16 7:8,16"
# window on: DRAM bytes of config 5 beta(1,8)
SPC5_X_WINDOW=1 bash tools/prof_env.sh "SPC5_X_WINDOW=1:5:1,8"
# compute-sanitizer (the workload first runs plain)
timeout 600 python tools/sanitize_small.py > $O/sanitize_plain.log 2>&1; echo "sanitize plain rc=$?"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py > $O/sanitize_$tool.log 2>&1
  echo "sanitize $tool rc=$?"
done
du -sh gpurun_out
