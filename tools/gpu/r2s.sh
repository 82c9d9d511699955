#!/bin/bash
# Kernel parity tests + quick perf on the current build.
mkdir -p gpurun_out/r2s
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_kernels_fullsize_gpu.py -m gpu -x -q > gpurun_out/r2s/pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r2s/pytest.log
bash tools/gpu/perf.sh r2s
