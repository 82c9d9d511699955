#!/bin/bash
# PP projection on N GPUs: the reference's default PP shape (dp = N, pp = 4,
# 9 layers per stage, gbs = 8 per rank, mbs = 2 -> 4 micro-batches per rank, default length mix);
# each strategy's measured per-layer kernel times go through the 1F1B model.
N=${1:-2}; ITERS=${2:-3}
for s in baseline sab dst sab_dst; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 200)) -m paper_2604_13847_b200.driver --strategy $s --iters $ITERS \
    --layers 36 --gbs-per-rank 8 --mbs 2 --mix default --project-pp 4 --out gpurun_out/pp_N$N/$s \
    > gpurun_out/pp_N$N.$s.log 2>&1
  echo "== $s (dp only)"; cat gpurun_out/pp_N$N/$s/iterations.csv
  echo "== $s (projected pp=4)"; cat gpurun_out/pp_N$N/$s/iterations_pp4.csv
done
