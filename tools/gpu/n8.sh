#!/bin/bash
bash tools/gpu/scale.sh r2n8 8
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29611 \
  -m paper_2604_13847_b200.driver --strategy sab_dst --iters 4 --layers 36 --dense-grid --gbs-per-rank 5 --mbs 5 \
  --table profiles/b200_cost_table_h32_d128_b128.csv --out gpurun_out/r2n8/c3_N8/sab_dst > gpurun_out/r2n8/c3_driver.log 2>&1
echo "driver rc $?"; cat gpurun_out/r2n8/c3_N8/sab_dst/iterations.csv
