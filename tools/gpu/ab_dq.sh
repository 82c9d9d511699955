#!/bin/bash
# dQ A/B: kernel parity tests on the in-tree lib, then C2 / C3 layer bwd time + dQ per-CTA spans and
# C5 GQA keep 0.1, in-tree vs alt_lib/$1.so.
OUT=gpurun_out/${OUT:-ab_dq}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_kernels_fullsize_gpu.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc $?"; tail -n 2 $OUT/pytest.log
for r in 1 2; do for lib in default $1; do
  if [ $lib = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$lib.so; fi
  C2=1 timeout 300 python tools/c3_items.py 2>&1 | grep "^fwd\|^dq per" | grep -v sorted | sed "s/^/$lib C2 $r /"
  timeout 300 python tools/c3_items.py 2>&1 | grep "^fwd\|^dq per" | grep -v sorted | sed "s/^/$lib C3 $r /"
done; done
for lib in default $1; do
  if [ $lib = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$lib.so; fi
  timeout 600 python tools/sweep_c5.py --keeps 0.1 --reps 3 --kv-heads 8 2>&1 | grep '^{' | sed "s/^/$lib C5 /" | cut -c1-220
done
unset SB_LIB_PATH
