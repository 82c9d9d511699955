#!/bin/bash
# Balance at N GPUs with the dense-grid mix cost tables (align() picks table-grid budgets, so the
# table's k step is DST's balance granularity). C3 (MHA) and C4 (GQA 32/8), SAB + DST, with and
# without the member-wise (varlen) cost.
N=${1:-4}; ITERS=${2:-4}; OUT=gpurun_out/${3:-balance_dense}
mkdir -p $OUT
T3=profiles/b200_cost_table_mix4060dense_h32_d128_b128.csv
T4=profiles/b200_cost_table_mix4060dense_h32kv8_d128_b128.csv
run() {  # tag strategy extra
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 200)) -m paper_2604_13847_b200.driver --strategy $2 --iters $ITERS \
    --layers 36 --dense-grid $3 --out $OUT/$1/$2 > $OUT/$1.$2.log 2>&1
  echo "== $1 $2 rc=$?"; cat $OUT/$1/$2/iterations.csv
}
run c3_dense sab_dst "--gbs-per-rank 5 --mbs 5 --table $T3"
run c3_dense_varlen sab_dst "--gbs-per-rank 5 --mbs 5 --varlen --table $T3"
run c4_dense sab_dst "--gbs-per-rank 10 --mbs 10 --heads 32 --kv-heads 8 --table $T4"
run c4_dense_varlen sab_dst "--gbs-per-rank 10 --mbs 10 --heads 32 --kv-heads 8 --varlen --table $T4"
run c4_dense_max sab_dst "--gbs-per-rank 10 --mbs 10 --heads 32 --kv-heads 8 --anchor max --table $T4"
