#!/bin/bash
# C4 balance variants at N GPUs: DST anchor (dst.cpp select_anchor) and micro-batches per rank.
N=${1:-4}; ITERS=${2:-4}; OUT=gpurun_out/${3:-balance_c4}
mkdir -p $OUT
run() {  # tag strategy extra
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 200)) -m paper_2604_13847_b200.driver --strategy $2 --iters $ITERS \
    --layers 36 --dense-grid --varlen --heads 32 --kv-heads 8 \
    --table profiles/b200_cost_table_mix4060_h32kv8_d128_b128.csv $3 --out $OUT/$1/$2 > $OUT/$1.$2.log 2>&1
  echo "== $1 $2 rc=$?"; cat $OUT/$1/$2/iterations.csv
}
run c4_max sab_dst "--gbs-per-rank 10 --mbs 10 --anchor max"
run c4_mb2_mean sab_dst "--gbs-per-rank 20 --mbs 10 --anchor mean"
run c4_mb2 baseline "--gbs-per-rank 20 --mbs 10"
run c4_mb2_max sab_dst "--gbs-per-rank 20 --mbs 10 --anchor max"
