#!/bin/bash
mkdir -p gpurun_out/gpu_speed
for r in 1 2; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 200)) tools/gpu_speed.py > gpurun_out/gpu_speed/run$r.log 2>&1; echo "rc $?"; grep "^{" gpurun_out/gpu_speed/run$r.log; done
nvidia-smi -q -d CLOCK,POWER | grep -E "GPU 0|Max|SM  |Power Limit|Current Power" | head -60 > gpurun_out/gpu_speed/smi.txt
