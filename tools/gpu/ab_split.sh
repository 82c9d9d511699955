#!/bin/bash
# C3 bench A/B: dK/dV item split (in-tree lib, cap = total / (4 grid)) vs split1 (cap = total / grid)
# vs headmajor (no split). Three alternating runs each.
OUT=gpurun_out/ab_split; mkdir -p $OUT
for r in 1 2 3; do
  for lib in default split1 headmajor; do
    if [ $lib = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$lib.so; fi
    timeout 600 python bench.py --steps 5 --warmup 3 --no-sub --no-cpu-baseline > $OUT/bench_${lib}_$r.log 2>&1
    python - <<PY
import json
l=[x for x in open('$OUT/bench_${lib}_$r.log').read().splitlines() if x.startswith('{')][-1]; l=json.loads(l)
print('$lib', $r, round(l['ms_per_step'],2), {k: round(v,2) for k,v in l['breakdown_ms_rank0'].items()})
PY
  done
done
unset SB_LIB_PATH
