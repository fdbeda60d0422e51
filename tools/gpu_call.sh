# round-2 measurement call: GPU tests, the bench lines of every config, ncu counters
set -x
O=gpurun_out/c1
mkdir -p $O
nvidia-smi --query-gpu=name,memory.total,clocks.sm --format=csv > $O/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --config 7 --steps 20 --warmup 5 --no-e2e > $O/bench_c7.json 2> $O/bench_c7.err; echo "c7 rc=$?"
for c in 2 3 4 6; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench_c$c.json 2> $O/bench_c$c.err; echo "c$c rc=$?"; done
bash tools/prof_configs.sh "${PROF:-3:1,16 3:4,16 4:8,8 5:1,8 5:8,8}"
du -sh gpurun_out
