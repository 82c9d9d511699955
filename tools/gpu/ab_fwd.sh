#!/bin/bash
# Forward-epilogue A/B: C3-layer fwd time and per-CTA spans for the in-tree lib and alt libs, fwd
# parity tests on the first alt, CTA-0 timeline on the first alt.
OUT=gpurun_out/${OUT:-ab_fwd}; mkdir -p $OUT
setlib() { if [ $1 = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$1.so; fi; }
setlib $1
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_kernels_fullsize_gpu.py -m gpu -x -q -k "fwd or forward" > $OUT/pytest_$1.log 2>&1; echo "pytest $1 rc $?"; tail -n 2 $OUT/pytest_$1.log
C3K=5 ROWS=12 timeout 300 python tools/trace_fwd2.py 2>&1 | tail -36 | head -20
for r in 1 2; do for lib in default "$@"; do
  setlib $lib
  timeout 300 python tools/c3_items.py 2>&1 | grep "^fwd" | sed "s/^/$lib $r /"
done; done
unset SB_LIB_PATH
