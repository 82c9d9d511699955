#!/bin/bash
# dK/dV epilogue warpgroup A/B: in-tree lib vs alt_lib/preepi.so.
OUT=gpurun_out/ab_epi; mkdir -p $OUT
timeout 700 python -m pytest tests/test_kernels_gpu.py tests/test_kernels_fullsize_gpu.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc $?"; tail -n 2 $OUT/pytest.log
C3K=5 PLANTED=1 timeout 300 python tools/trace_dkv.py 2>&1 | grep "item (pairs" | cut -c1-400
for r in 1 2; do
  for lib in default prerec; do
    if [ $lib = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$lib.so; fi
    timeout 300 python bench.py --steps 5 --warmup 3 --no-sub --no-cpu-baseline > $OUT/bench_${lib}_$r.log 2>&1
    python - <<PY
import json
l=[x for x in open('$OUT/bench_${lib}_$r.log').read().splitlines() if x.startswith('{')][-1]; l=json.loads(l)
print('$lib', $r, round(l['value'],1), round(l['ms_per_step'],2), {k: round(v,2) for k,v in l['breakdown_ms_rank0'].items()})
PY
  done
done
for lib in default prerec; do
  if [ $lib = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$lib.so; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_bwd_dkv" -c 3 --csv python tools/time_kernels.py 2>/dev/null | grep gpu__time | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ' | sed "s/^/$lib C2 dkv ns: /"; echo
  timeout 600 python tools/sweep_c5.py --keeps 0.1 --reps 5 --kv-heads 8 2>&1 | grep '^{' | sed "s/^/$lib C5 /" | cut -c1-220
done
unset SB_LIB_PATH
