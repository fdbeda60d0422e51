O=gpurun_out/ab9
mkdir -p $O
for c in "5 1,8;2,8;4,8;8,8" "7 1,16;2,16;4,16;8,16" "2 1,8;2,8;4,8;8,8" "6 1,16;2,16;4,16;8,16" "3 1,16;2,16;4,16" "4 4,8;8,8"; do
  set -- $c
  echo "c$1 $(timeout 600 python tools/time_k2.py "$2" 20 $1 2>&1 | tail -1)" | tee -a $O/summary.txt
done
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" | tee -a $O/summary.txt
timeout 600 python tools/sanitize_small.py > $O/sanitize_plain.log 2>&1 && timeout 1800 compute-sanitizer --tool memcheck --leak-check no python tools/sanitize_small.py > $O/memcheck.log 2>&1; echo "memcheck rc=$?" | tee -a $O/summary.txt
tail -5 $O/memcheck.log
