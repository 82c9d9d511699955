#!/bin/bash
# The GPU test suite against the debug library (no compute-sanitizer on this pool): mbarrier wait
# timeouts + index-invariant traps; a trap or hang fails the run.
OUT=gpurun_out/debugsuite; mkdir -p $OUT
SB_LIB_PATH=$PWD/paper_2604_13847_b200/lib/libsparsebalance_b200_debug.so timeout 2400 python -m pytest tests -m gpu -q -rf \
  --timeout 900 > $OUT/pytest_gpu_debug.log 2>&1; echo "pytest(debug lib) rc $?"
tail -5 $OUT/pytest_gpu_debug.log
SB_LIB_PATH=$PWD/paper_2604_13847_b200/lib/libsparsebalance_b200_debug.so timeout 300 python tools/sanitize_case.py > $OUT/case.log 2>&1; echo "case rc $?"; tail -2 $OUT/case.log
