#!/bin/bash
# Mix-aware cost tables (40 % 32K / 60 % 2K packed cells), MHA 32 and GQA 32/8.
OUT=gpurun_out/tables; mkdir -p $OUT
timeout 1200 python -m paper_2604_13847_b200.profiler --mix 40/60 --out $OUT/b200_cost_table_mix4060_h32_d128_b128 > $OUT/mha.log 2>&1; echo "mha rc $?"
timeout 1200 python -m paper_2604_13847_b200.profiler --mix 40/60 --kv-heads 8 --out $OUT/b200_cost_table_mix4060_h32kv8_d128_b128 > $OUT/gqa.log 2>&1; echo "gqa rc $?"
tail -4 $OUT/mha.log $OUT/gqa.log
C3K=4 ROWS=24 timeout 300 python tools/trace_fwd2.py > $OUT/trace_fwd_c3.log 2>&1; echo "trace rc $?"; tail -40 $OUT/trace_fwd_c3.log
