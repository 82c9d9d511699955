#!/bin/bash
mkdir -p gpurun_out/c4i
timeout 600 python tools/c4_items.py 2>&1 | grep -v Warn | tee gpurun_out/c4i/items.log
HKV=32 timeout 600 python tools/c4_items.py 2>&1 | grep -v Warn | tee gpurun_out/c4i/items_mha.log
