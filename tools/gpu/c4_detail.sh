#!/bin/bash
# C4 at N GPUs, dense table: per-(rank, mb) measured fwd / bwd / total next to the plan.
N=${1:-4}; OUT=gpurun_out/c4_detail; mkdir -p $OUT
T4=profiles/b200_cost_table_mix4060dense_h32kv8_d128_b128.csv
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port $((29600 + RANDOM % 200)) -m paper_2604_13847_b200.driver --strategy sab_dst --iters 4 \
  --layers 36 --dense-grid --gbs-per-rank 10 --mbs 10 --heads 32 --kv-heads 8 --table $T4 --out $OUT/sab_dst > $OUT/log 2>&1
echo "rc $?"; cat $OUT/sab_dst/iterations.csv
