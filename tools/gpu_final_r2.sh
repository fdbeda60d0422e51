# round-2 final measurement call: tests, checked build, bench lines, launch list, ncu captures
set -x
O=gpurun_out/final
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/gpu_tests.log
bash tools/checked_build.sh > $O/checked_build.log 2>&1; tail -5 $O/checked_build.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; cat $O/smoke.log | tail -1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
for c in 1 2 3 4 6 7; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench_c$c.json 2> $O/bench_c$c.err; echo "c$c rc=$?"; done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
  > $O/ncu_launches.log 2>&1; echo "launches rc=$?"
bash tools/prof_configs.sh "5:1,8 5:2,8 5:4,8 5:8,8 7:1,16 7:2,16 7:4,16 7:8,16"
# the N > 1 code path with one rank (this environment has one GPU per call)
for c in 2 5; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2951$c \
    bench.py --gpus 2 --config $c --steps 5 --warmup 3 --iters 10 > $O/bench_dist1_c$c.json 2> $O/bench_dist1_c$c.err; echo "dist1 c$c rc=$?"
done
du -sh gpurun_out
