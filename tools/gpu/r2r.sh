#!/bin/bash
OUT=gpurun_out/r2r; mkdir -p $OUT
for i in 1 2 3; do
for mode in sampler nosampler; do
  if [ $mode = nosampler ]; then export SB_NO_CLOCK_SAMPLER=1; else unset SB_NO_CLOCK_SAMPLER; fi
  SB_OPS_TIMING=1 SB_PHASE_DUMP=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-sub --no-cpu-baseline > $OUT/bench_$mode$i.log 2>$OUT/phases_$mode$i.log
  python -c "
import json
l=[x for x in open('$OUT/bench_$mode$i.log').read().splitlines() if x.startswith('{')][-1]; l=json.loads(l)
print('$mode$i', round(l['ms_per_step'],2), {k: round(v,2) for k,v in l['breakdown_ms_rank0'].items()}, 'e2e', round(l['e2e']['ms_per_step'],2))
"
done; done
