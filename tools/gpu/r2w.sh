#!/bin/bash
mkdir -p gpurun_out/r2w
timeout 900 python tools/table_repeat.py > gpurun_out/r2w/table_repeat.log 2>&1; echo "repeat rc $?"; grep -v Warn gpurun_out/r2w/table_repeat.log | tail -20
bash tools/gpu/ab_hint.sh
