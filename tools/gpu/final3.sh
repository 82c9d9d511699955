#!/bin/bash
# Final validation + measurement set on the current build (round 2, after dynamic claiming):
# GPU suite, smoke, full N=1 bench + reference arm, DRAM traffic launch list, C3 launch list,
# one ncu --set full capture of the dK/dV kernel.
T=${1:-final3}; mkdir -p gpurun_out/$T
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/$T/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -n 2 gpurun_out/$T/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$T/smoke.log 2>&1; echo "smoke rc $?"; tail -n 1 gpurun_out/$T/smoke.log
bash tools/gpu/fullbench.sh fullbench_$T
bash tools/gpu/traffic.sh
python tools/capture_traffic.py gpurun_out/traffic/launches.csv | head -30
bash tools/gpu/launches.sh launches_$T ""
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_bwd_dkv -s 2 -c 1 -o gpurun_out/$T/dkv_full python bench.py --profile-only > gpurun_out/$T/ncu_full.log 2>&1; echo "ncu full rc $?"
