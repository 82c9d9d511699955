#!/bin/bash
# One compute-sanitizer tool per call (B200_PROFILING.md): tools/gpu/sanitize.sh memcheck|synccheck|racecheck
OUT=gpurun_out/sanitizer; mkdir -p $OUT; TOOL=$1
timeout 300 python tools/sanitize_case.py > $OUT/plain_$TOOL.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 50 python tools/sanitize_case.py > $OUT/$TOOL.log 2>&1; echo "$TOOL rc $?"
tail -8 $OUT/$TOOL.log
