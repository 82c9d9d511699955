#!/bin/bash
# Balance at N GPUs, ITERS iterations: C3 and C4, baseline vs SAB + DST on the dense-grid mix
# cost tables (table cost, and the member-wise varlen cost).
N=${1:-4}; ITERS=${2:-8}; OUT=gpurun_out/${3:-balance_final}
mkdir -p $OUT
T3=profiles/b200_cost_table_mix4060dense_h32_d128_b128.csv
T4=profiles/b200_cost_table_mix4060dense_h32kv8_d128_b128.csv
run() {  # tag strategy extra
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 200)) -m paper_2604_13847_b200.driver --strategy $2 --iters $ITERS \
    --layers 36 --dense-grid $3 --out $OUT/$1/$2 > $OUT/$1.$2.log 2>&1
  echo "== $1 $2 rc=$?"; cat $OUT/$1/$2/iterations.csv
}
C3="--gbs-per-rank 5 --mbs 5 --table $T3"
C4="--gbs-per-rank 10 --mbs 10 --heads 32 --kv-heads 8 --table $T4"
run c3 baseline "$C3"
run c3 sab_dst "$C3"
run c3_varlen sab_dst "$C3 --varlen"
run c4 baseline "$C4"
run c4 sab_dst "$C4"
run c4_varlen sab_dst "$C4 --varlen"
