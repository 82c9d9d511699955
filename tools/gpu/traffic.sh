#!/bin/bash
# Roofline traffic capture on HEAD: plain run, then the ncu launch list with DRAM bytes.
OUT=gpurun_out/traffic; mkdir -p $OUT
timeout 600 python bench.py --profile-only > $OUT/plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"attn_|bwd_prep|transpose_sel|scan_kernel|q_records|match_rounds|dkv_split" -c 14 --csv --log-file $OUT/launches.csv python bench.py --profile-only > $OUT/ncu.log 2>&1; echo "ncu rc $?"
