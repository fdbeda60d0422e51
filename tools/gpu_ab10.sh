O=gpurun_out/ab10
mkdir -p $O
for c in "3 1,16;2,16;4,16" "4 4,8;8,8" "2 1,8;2,8;4,8;8,8"; do
  set -- $c
  echo "c$1 $(timeout 600 python tools/time_k2.py "$2" 40 $1 2>&1 | tail -1)" | tee -a $O/summary.txt
done
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" | tee -a $O/summary.txt
SPC5_FVR=3 timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests3.log 2>&1; echo "tests fvr3 rc=$?" | tee -a $O/summary.txt
tail -3 $O/gpu_tests.log $O/gpu_tests3.log
