#!/bin/bash
# dK/dV item split: kernel parity tests, C4 planted items, C3 perf.
mkdir -p gpurun_out/r2v
timeout 900 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q > gpurun_out/r2v/pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r2v/pytest.log
timeout 600 python tools/c4_items.py 2>&1 | grep -v Warn | tee gpurun_out/r2v/items.log
bash tools/gpu/perf.sh r2v
