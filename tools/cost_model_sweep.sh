#!/bin/bash
# SAB+DST on N GPUs with three cost models: the reference's synthetic table, the GPU-measured
# table (profiles/b200_cost_table_h32_d128_b128.csv), and the measured table with the opt-in
# varlen member-wise cost. Same iterations / seeds as tools/balance_sweep.sh.
N=${1:-4}; ITERS=${2:-4}
run() {
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 200)) -m paper_2604_13847_b200.driver --strategy sab_dst --iters $ITERS \
    --layers 36 --gbs-per-rank 5 --mbs 5 --out gpurun_out/cost_N$N/$1 "${@:2}" > gpurun_out/cost_N$N.$1.log 2>&1
  echo "== $1"; cat gpurun_out/cost_N$N/$1/iterations.csv
}
run synthetic
run measured --table profiles/b200_cost_table_h32_d128_b128.csv
run measured_varlen --table profiles/b200_cost_table_h32_d128_b128.csv --varlen
