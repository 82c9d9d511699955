#!/bin/bash
# The driver's round-end command (N=1): full bench line with sub-records and CPU baseline; plus
# the reference arm.
OUT=gpurun_out/${1:-fullbench}; mkdir -p $OUT
timeout 1200 python bench.py --steps 10 --warmup 3 > $OUT/bench.log 2>&1; echo "bench rc $?"
tail -c 6000 $OUT/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.log 2>&1; echo "ref rc $?"
tail -c 1500 $OUT/bench_ref.log
