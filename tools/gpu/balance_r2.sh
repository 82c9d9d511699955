#!/bin/bash
# Balance target runs: the measured DP step driver, closed loop on GPU profiles,
# dense 1..256 DST grid, GPU-measured fwd+bwd cost tables, N GPUs, ITERS iterations each.
#   C3 mix (40% 32K / 60% 2K, gbs = 5N, mbs = 5, MHA 32 heads) and C4 (gbs = 10N, mbs = 10, GQA 32/8).
N=${1:-4}; ITERS=${2:-3}; OUT=gpurun_out/${3:-balance_r2}; EXTRA=${4:-}
mkdir -p $OUT
run() {  # tag strategy extra
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 200)) -m paper_2604_13847_b200.driver --strategy $2 --iters $ITERS \
    --layers 36 --dense-grid $EXTRA $3 --out $OUT/$1_N$N/$2 > $OUT/$1_N$N.$2.log 2>&1
  echo "== $1 $2 rc=$?"; cat $OUT/$1_N$N/$2/iterations.csv
}
for s in baseline sab_dst; do run c3 $s "--gbs-per-rank 5 --mbs 5 --table profiles/b200_cost_table_mix4060_h32_d128_b128.csv"; done
for s in baseline sab_dst; do run c4 $s "--gbs-per-rank 10 --mbs 10 --heads 32 --kv-heads 8 --table profiles/b200_cost_table_mix4060_h32kv8_d128_b128.csv"; done
