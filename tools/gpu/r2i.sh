#!/bin/bash
OUT=gpurun_out/r2i; mkdir -p $OUT
for bwd in fused two-pass; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-sub --no-cpu-baseline --bwd $bwd > $OUT/bench_$bwd.log 2>&1; echo "bench $bwd rc $?"
python -c "
import json,sys
l=json.loads(open('$OUT/bench_$bwd.log').read().strip().splitlines()[-1])
print('$bwd', 'value', round(l['value'],1), 'ms', round(l['ms_per_step'],2), l['breakdown_ms_rank0'], 'k', l['k_final_rank0'][:3], 'fwdTF', round(l['fwd_tflops_rank0'],1), 'bwdTF', round(l['bwd_tflops_rank0'],1), 'clk', l['clocks'])
"
done
