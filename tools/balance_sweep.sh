#!/bin/bash
# Strategy sweep of the measured DP step driver on N GPUs: per strategy,
# ITERS iterations of the 40/60 32K/2K mix, gbs = 5N, mbs = 5 (one packed micro-batch per rank),
# 36 layers; writes gpurun_out/balance_N<N>/<strategy>/{iterations.csv,decisions_*.csv,plan_*.json}.
N=${1:-4}; ITERS=${2:-3}
for s in baseline sab dst sab_dst; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 200)) -m paper_2604_13847_b200.driver --strategy $s --iters $ITERS \
    --layers 36 --gbs-per-rank 5 --mbs 5 --out gpurun_out/balance_N$N/$s > gpurun_out/balance_N$N.$s.log 2>&1
  echo "== $s"; cat gpurun_out/balance_N$N/$s/iterations.csv
done
