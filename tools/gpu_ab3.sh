O=gpurun_out/ab3
mkdir -p $O
for v in 0 1; do
  for c in "3 1,16;2,16;4,16" "4 4,8;8,8" "2 1,8;2,8;4,8;8,8" "6 1,16;2,16;4,16;8,16"; do
    set -- $c
    echo "FVR=$v c$1 $(SPC5_FVR=$v timeout 300 python tools/time_k2.py "$2" 50 $1 2>&1 | tail -1)" | tee -a $O/summary.txt
  done
done
for cb in 192 256 512 768 1024; do
  echo "FVR=1 CB=$cb c3 $(SPC5_CB=$cb timeout 300 python tools/time_k2.py "2,16;4,16" 50 3 2>&1 | tail -1)" | tee -a $O/summary.txt
done
echo "FVR=3 c4 $(SPC5_FVR=3 timeout 300 python tools/time_k2.py "4,8;8,8" 50 4 2>&1 | tail -1)" | tee -a $O/summary.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" | tee -a $O/summary.txt
