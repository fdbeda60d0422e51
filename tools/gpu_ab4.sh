O=gpurun_out/ab4
mkdir -p $O
for c in "3 1,16;2,16;4,16" "4 4,8;8,8"; do
  set -- $c
  echo "c$1 $(timeout 300 python tools/time_k2.py "$2" 50 $1 2>&1 | tail -1)" | tee -a $O/summary.txt
done
echo "FVR=2 c3 $(SPC5_FVR=2 timeout 300 python tools/time_k2.py "1,16" 50 3 2>&1 | tail -1)" | tee -a $O/summary.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" | tee -a $O/summary.txt
SPC5_FVR=3 timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests3.log 2>&1; echo "tests fvr3 rc=$?" | tee -a $O/summary.txt
bash tools/prof_env.sh "-:3:4,16 -:4:8,8"
