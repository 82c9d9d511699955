#!/bin/bash
OUT=gpurun_out/r2e; mkdir -p $OUT
LAYERS=8 timeout 600 python tools/timeline_c3.py > $OUT/timeline_c3.log 2>&1; echo "timeline rc $?"; head -40 $OUT/timeline_c3.log
REPS=3 timeout 300 python tools/time_kernels.py > $OUT/plain.log 2>&1 && \
REPS=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_fused -c 1 -o $OUT/fused python tools/time_kernels.py > $OUT/ncu.log 2>&1; echo "ncu rc $?"
tail -3 $OUT/ncu.log
