#!/bin/bash
OUT=gpurun_out/r2q; mkdir -p $OUT
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_cpp_dropin.py -m gpu -q -rf --timeout 600 > $OUT/pytest_kernels.log 2>&1; echo "pytest rc $?"; tail -3 $OUT/pytest_kernels.log
bash tools/gpu/perf.sh r2q_perf | head -12
C3K=4 ROWS=10 timeout 300 python tools/trace_fwd2.py > $OUT/trace_fwd_c3.log 2>&1; grep -E "median|epi" $OUT/trace_fwd_c3.log | head -24
