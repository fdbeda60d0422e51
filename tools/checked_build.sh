#!/bin/bash
# Memcheck substitute (compute-sanitizer is closed on the GPU pool): the library
# built with -DSPC5_CHECKED=1 (bounds checks on every shared-memory read of a
# slot, every x gather and every y store; a violation prints and traps) runs
# the small parity workload of tools/sanitize_small.py and the parity tests of
# every chunk mode; then the product build is put back.
# Build the checked library first, where nvcc has the cores:
#   python tools/build_variant.py checked -DSPC5_CHECKED=1 &&
#   cp variants/checked/libspc5_b200.so paper_2307_14774_b200/libspc5_b200_checked.so
# usage (on the GPU box): bash tools/checked_build.sh > gpurun_out/checked.log 2>&1
P=paper_2307_14774_b200
[ -f $P/libspc5_b200_checked.so ] || { echo "no checked library"; exit 1; }
cp $P/libspc5_b200.so /tmp/libspc5_product.so
cp $P/libspc5_b200_checked.so $P/libspc5_b200.so
# the checks are live: with a one-column x bound the first product must trap
SPC5_CHECKED_SELFTEST=1 timeout 300 python -c "
import numpy as np, paper_2307_14774_b200 as p
from paper_2307_14774_b200.workloads import config1, x_vector
m = config1(); s = p.csr_to_spc5(m, 1, 8)
try:
    p.spmv(s, x_vector(m.num_cols)); print('SELFTEST FAILED: no trap')
except Exception as e:
    print('selftest trapped as expected:', str(e)[:120])
" 2>&1 | grep -i "selftest\|violation" | head -4
timeout 900 python tools/sanitize_small.py; echo "checked sanitize_small rc=$?"
timeout 900 python -m pytest tests/test_gpu_lbr.py tests/test_gpu_parity.py tests/test_gpu_concurrency.py -q -x -m gpu -k "not slow and not full_size" 2>&1 | tail -3
cp /tmp/libspc5_product.so $P/libspc5_b200.so
