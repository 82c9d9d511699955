#!/bin/bash
# Final validation on the final build: full GPU suite, smoke, full N=1 bench + reference arm,
# ncu launch list + DRAM traffic.
mkdir -p gpurun_out/final2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final2/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -n 2 gpurun_out/final2/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final2/smoke.log 2>&1; echo "smoke rc $?"; tail -n 1 gpurun_out/final2/smoke.log
bash tools/gpu/fullbench.sh fullbench_final2
bash tools/gpu/traffic.sh
bash tools/gpu/launches.sh launches_final2 ""
