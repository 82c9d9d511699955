#!/bin/bash
OUT=gpurun_out/r4b; mkdir -p $OUT
timeout 300 python tools/c3_items.py > $OUT/c3_items.log 2>&1; echo "c3_items rc $?"
cat $OUT/c3_items.log | cut -c1-3000
C3K=5 PLANTED=1 timeout 300 python tools/trace_dkv.py > $OUT/trace.log 2>&1; echo "trace rc $?"; cut -c1-1500 $OUT/trace.log
