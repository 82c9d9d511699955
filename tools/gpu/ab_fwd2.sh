#!/bin/bash
# Forward A/B: fwd/full parity tests on the in-tree lib, then C2 / C3 layer fwd time + per-CTA spans,
# in-tree vs alt_lib/$1.so, twice.
OUT=gpurun_out/${OUT:-ab_fwd2}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_kernels_fullsize_gpu.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc $?"; tail -n 2 $OUT/pytest.log
for r in 1 2; do for lib in default $1; do
  if [ $lib = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$lib.so; fi
  C2=1 timeout 300 python tools/c3_items.py 2>&1 | grep "^fwd\|^dq per\|^dkv per-CTA (us)" | grep -v sorted | sed "s/^/$lib C2 $r /"
  timeout 300 python tools/c3_items.py 2>&1 | grep "^fwd\|^dq per\|^dkv per-CTA (us)" | grep -v sorted | sed "s/^/$lib C3 $r /"
done; done
