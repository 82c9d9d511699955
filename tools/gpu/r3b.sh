#!/bin/bash
mkdir -p gpurun_out/r3b
SB_LIB_PATH=alt_lib/pdl1.so timeout 300 python tools/scores_dump.py gpurun_out/r3b/old.npz 2>&1 | tail -1
timeout 300 python tools/scores_dump.py gpurun_out/r3b/new.npz 2>&1 | tail -1
python - <<'PY'
import numpy as np
a, b = np.load("gpurun_out/r3b/old.npz"), np.load("gpurun_out/r3b/new.npz")
for k in a.files:
    print(k, "bit-identical" if np.array_equal(a[k].view(np.uint32), b[k].view(np.uint32)) else f"DIFF max {np.abs(a[k]-b[k]).max()}")
PY
timeout 900 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k "scores or topk or coverage or edge" 2>&1 | tail -2
for lib in pdl1 default; do
  if [ $lib = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$lib.so; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"block_scores" -c 4 --csv python tools/scores_dump.py /tmp/x.npz 2>/dev/null | grep block_scores | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ' | sed "s/^/$lib /"; echo
done
unset SB_LIB_PATH
for r in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-sub --no-cpu-baseline > gpurun_out/r3b/bench_$r.log 2>&1; python - <<PY
import json
l=[x for x in open('gpurun_out/r3b/bench_$r.log').read().splitlines() if x.startswith('{')][-1]; l=json.loads(l)
print('C3', round(l['value'],1), round(l['ms_per_step'],2), {k: round(v,2) for k,v in l['breakdown_ms_rank0'].items()})
PY
done
