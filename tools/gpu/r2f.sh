#!/bin/bash
OUT=gpurun_out/r2f; mkdir -p $OUT
SB_LIB_PATH=$PWD/paper_2604_13847_b200/lib/libsparsebalance_b200_debug.so timeout 300 python tools/check_fused.py > $OUT/check_debug.log 2>&1; echo "check(debug) rc $?"
tail -25 $OUT/check_debug.log
timeout 300 python tools/time_kernels.py > $OUT/time_kernels.log 2>&1; echo "time rc $?"; grep -v Warn $OUT/time_kernels.log | head -8
