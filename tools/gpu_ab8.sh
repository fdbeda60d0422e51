O=gpurun_out/ab8
mkdir -p $O
for i in 1 2; do
echo "XPF=0 c5 $(SPC5_NO_XPREFETCH=1 timeout 600 python tools/time_k2.py "8,8" 40 5 2>&1 | tail -1)" | tee -a $O/summary.txt
echo "XPF=1 c5 $(timeout 600 python tools/time_k2.py "8,8" 40 5 2>&1 | tail -1)" | tee -a $O/summary.txt
done
bash tools/prof_env.sh "-:5:8,8 -:2:8,8"
