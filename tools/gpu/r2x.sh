#!/bin/bash
bash tools/gpu/balance_final.sh 4 8 balance_final2
for r in 1 2; do bash tools/gpu/scale.sh n4b_$r 4 "--no-sub --no-cpu-baseline"; done
