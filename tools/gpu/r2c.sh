#!/bin/bash
OUT=gpurun_out/r2c; mkdir -p $OUT
SB_LIB_PATH=$PWD/paper_2604_13847_b200/lib/libsparsebalance_b200_debug.so timeout 300 python tools/check_fused.py > $OUT/check_debug.log 2>&1; echo "check(debug) rc $?"
cat $OUT/check_debug.log | tail -30
timeout 300 python tools/check_fused.py > $OUT/check.log 2>&1; echo "check rc $?"
tail -5 $OUT/check.log
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_cpp_dropin.py -m gpu -q -rf --timeout 600 > $OUT/pytest_kernels.log 2>&1; echo "pytest rc $?"
tail -30 $OUT/pytest_kernels.log
