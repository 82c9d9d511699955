#!/bin/bash
OUT=gpurun_out/${1:-ncu_fused}; mkdir -p $OUT
REPS=3 timeout 300 python tools/time_kernels.py > $OUT/plain.log 2>&1 && \
REPS=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_fused -c 1 -o $OUT/fused python tools/time_kernels.py > $OUT/ncu.log 2>&1; echo "ncu rc $?"
tail -2 $OUT/ncu.log
