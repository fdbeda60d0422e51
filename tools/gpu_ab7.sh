O=gpurun_out/ab7
mkdir -p $O
for v in 0 1; do
  for c in "5 1,8;2,8;4,8;8,8" "2 1,8;2,8;4,8;8,8" "7 1,16;2,16;4,16;8,16" "3 1,16;4,16" "4 4,8;8,8"; do
    set -- $c
    if [ $v = 0 ]; then E="SPC5_NO_XPREFETCH=1"; else E="SPC5_DUMMY=1"; fi
    echo "XPF=$v c$1 $(env $E timeout 600 python tools/time_k2.py "$2" 20 $1 2>&1 | tail -1)" | tee -a $O/summary.txt
  done
done
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" | tee -a $O/summary.txt
