#!/bin/bash
# Mix-aware cost tables on a dense budget grid (align() returns table-grid budgets only, so the grid
# step sets DST's balance granularity) and extra length bins over the C3 / C4 micro-batch range.
OUT=gpurun_out/tables_dense; mkdir -p $OUT
GRID=1,2,3,4,5,6,7,8,9,10,11,12,13,14,15,16,18,20,22,24,28,32,40,48,56,64
BINS=256,512,1024,2048,4096,8192,16384,24576,32768,40960,49152,57344,65536,81920,98304,114688,131072,147456,163840,196608,229376,262144
timeout 2400 python -m paper_2604_13847_b200.profiler --mix 40/60 --passes 5 --grid $GRID --bins $BINS --out $OUT/b200_cost_table_mix4060dense_h32_d128_b128 > $OUT/mha.log 2>&1; echo "mha rc $?"
timeout 2400 python -m paper_2604_13847_b200.profiler --mix 40/60 --kv-heads 8 --passes 5 --grid $GRID --bins $BINS --out $OUT/b200_cost_table_mix4060dense_h32kv8_d128_b128 > $OUT/gqa.log 2>&1; echo "gqa rc $?"
tail -n 3 $OUT/mha.log $OUT/gqa.log
