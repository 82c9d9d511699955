#!/bin/bash
# Final N=1 measurement set: full bench line + reference arm, DRAM traffic launch list, launch list.
bash tools/gpu/fullbench.sh fullbench_final
bash tools/gpu/traffic.sh
python tools/capture_traffic.py gpurun_out/traffic/launches.csv | head -30
bash tools/gpu/launches.sh launches_final ""
