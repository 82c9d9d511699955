#!/bin/bash
mkdir -p gpurun_out/tl
timeout 600 python tools/timeline_c3.py > gpurun_out/tl/timeline.log 2>&1; echo rc $?; grep -v Warn gpurun_out/tl/timeline.log | tail -40
