# FVR A/B round 2: times per SPC5_FVR setting for the sparse configs + stall profile of the FVR kernel
O=gpurun_out/ab2
mkdir -p $O
for v in 0 1; do
  for c in "3 1,16;2,16;4,16" "4 4,8;8,8"; do
    set -- $c
    echo "FVR=$v c$1 $(SPC5_FVR=$v timeout 300 python tools/time_k2.py "$2" 50 $1 2>&1 | tail -1)" | tee -a $O/summary.txt
  done
done
echo "FVR=1 nokernel c3 $(SPC5_NO_FVR_KERNEL=1 timeout 300 python tools/time_k2.py "1,16;4,16" 50 3 2>&1 | tail -1)" | tee -a $O/summary.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" | tee -a $O/summary.txt
bash tools/prof_env.sh "SPC5_FVR=1:3:1,16 SPC5_FVR=1:3:4,16"
