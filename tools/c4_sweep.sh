#!/bin/bash
# BASELINE C4: sparsity-aware batching + bidirectional tuning over ~128K-token micro-batches,
# GQA 32q / 8kv heads (group-shared selection), on N GPUs. Per strategy, ITERS iterations of the
# 40/60 32K/2K mix with gbs = 10N, mbs = 10 (one packed micro-batch of ~10 samples, mean 140K
# tokens, per rank), 36 layers, measured by the DP step driver.
# Optional third argument: a cost-table CSV (x,k,latency_ms) for SAB/DST, e.g. the GPU-measured
# profiles/b200_cost_table_h32_d128_b128.csv; outputs then go to gpurun_out/c4_N<N>_table/.
N=${1:-2}; ITERS=${2:-3}; TABLE=${3:-}
TAG=c4_N$N; EXTRA=""
if [ -n "$TABLE" ]; then TAG=${TAG}_table; EXTRA="--table $TABLE"; fi
for s in baseline sab_dst; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 200)) -m paper_2604_13847_b200.driver --strategy $s --iters $ITERS \
    --layers 36 --gbs-per-rank 10 --mbs 10 --heads 32 --kv-heads 8 $EXTRA --out gpurun_out/$TAG/$s \
    > gpurun_out/$TAG.$s.log 2>&1
  echo "== $s rc=$?"; cat gpurun_out/$TAG/$s/iterations.csv
done
