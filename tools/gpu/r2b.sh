#!/bin/bash
OUT=gpurun_out/r2b; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -25 $OUT/pytest_gpu.log
timeout 900 python -m paper_2604_13847_b200.profiler --out $OUT/b200_cost_table_h32_d128_b128 > $OUT/profiler_mha.log 2>&1; echo "prof mha rc $?"
timeout 900 python -m paper_2604_13847_b200.profiler --kv-heads 8 --out $OUT/b200_cost_table_h32kv8_d128_b128 > $OUT/profiler_gqa.log 2>&1; echo "prof gqa rc $?"
tail -4 $OUT/profiler_mha.log $OUT/profiler_gqa.log
timeout 600 python bench.py --profile-only --no-sub > $OUT/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3.csv python bench.py --profile-only --no-sub > $OUT/ncu.log 2>&1; echo "ncu rc $?"
