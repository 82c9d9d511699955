#!/bin/bash
OUT=gpurun_out/r2d; mkdir -p $OUT
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_cpp_dropin.py -m gpu -q -rf --timeout 600 > $OUT/pytest_kernels.log 2>&1; echo "pytest rc $?"
grep -E "AssertionError:|passed|failed" $OUT/pytest_kernels.log | tail -12
timeout 600 python tools/time_kernels.py > $OUT/time_kernels.log 2>&1; echo "time rc $?"; head -3 $OUT/time_kernels.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-sub --no-cpu-baseline > $OUT/bench.log 2>&1; echo "bench rc $?"
tail -c 2500 $OUT/bench.log
