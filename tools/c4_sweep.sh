#!/bin/bash
# BASELINE C4: sparsity-aware batching + bidirectional tuning over ~128K-token micro-batches,
# GQA 32q / 8kv heads (group-shared selection), on N GPUs. Per strategy, ITERS iterations of the
# 40/60 32K/2K mix with gbs = 10N, mbs = 10 (one packed micro-batch of ~10 samples, mean 140K
# tokens, per rank), 36 layers, measured by the DP step driver.
N=${1:-2}; ITERS=${2:-3}
for s in baseline sab_dst; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 200)) -m paper_2604_13847_b200.driver --strategy $s --iters $ITERS \
    --layers 36 --gbs-per-rank 10 --mbs 10 --heads 32 --kv-heads 8 --out gpurun_out/c4_N$N/$s \
    > gpurun_out/c4_N$N.$s.log 2>&1
  echo "== $s rc=$?"; cat gpurun_out/c4_N$N/$s/iterations.csv
done
