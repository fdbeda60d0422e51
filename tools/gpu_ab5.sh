O=gpurun_out/ab5
mkdir -p $O
for c in "3 1,16;2,16;4,16" "4 4,8;8,8" "2 1,8;2,8;4,8;8,8" "6 1,16;2,16;4,16;8,16"; do
  set -- $c
  echo "c$1 $(timeout 300 python tools/time_k2.py "$2" 50 $1 2>&1 | tail -1)" | tee -a $O/summary.txt
done
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" | tee -a $O/summary.txt
bash tools/prof_env.sh "-:3:4,16"
