# A/B of K2 modes: GPU tests with the default plan and with FVR forced, then
# K2 times per config and SPC5_FVR setting.  usage: bash tools/gpu_ab.sh
O=gpurun_out/ab
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" | tee -a $O/summary.txt
SPC5_FVR=2 timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests_fvr2.log 2>&1; echo "tests fvr2 rc=$?" | tee -a $O/summary.txt
for v in 0 1 2; do
  for c in "3 1,16;2,16;4,16" "4 4,8;8,8" "2 1,8;2,8;4,8;8,8" "6 1,16;2,16;4,16;8,16"; do
    set -- $c
    echo "FVR=$v c$1 $(SPC5_FVR=$v timeout 300 python tools/time_k2.py "$2" 50 $1 2>&1 | tail -1)" | tee -a $O/summary.txt
  done
done
