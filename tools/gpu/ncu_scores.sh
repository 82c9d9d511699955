#!/bin/bash
mkdir -p gpurun_out/ncu_scores
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"block_scores" -s 1 -c 1 -o gpurun_out/ncu_scores/scores python tools/scores_dump.py /tmp/x.npz > gpurun_out/ncu_scores/log 2>&1; echo "ncu rc $?"
