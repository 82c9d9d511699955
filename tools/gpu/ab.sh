#!/bin/bash
# Same-box A/B: in-tree library vs alt_lib/<name>.so for each name (C3 bench x2 each, alternating,
# C5 GQA keep 0.1 once each) + bwd parity tests + the C3 dK/dV per-CTA timeline.
# Usage: OUT=dir ab.sh <alt name>...
OUT=gpurun_out/${OUT:-ab}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_kernels_fullsize_gpu.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc $?"; tail -n 2 $OUT/pytest.log
setlib() { if [ $1 = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$1.so; fi; }
for lib in default "$@"; do
  setlib $lib
  timeout 300 python tools/c3_items.py > $OUT/c3_items_$lib.log 2>&1; echo "c3_items $lib rc $?"; grep -v sorted $OUT/c3_items_$lib.log | grep "dkv\|fwd"
done
for r in 1 2; do
  for lib in default "$@"; do
    setlib $lib
    timeout 300 python bench.py --steps 5 --warmup 3 --no-sub --no-cpu-baseline > $OUT/bench_${lib}_$r.log 2>&1
    python - <<PY
import json
l=[x for x in open('$OUT/bench_${lib}_$r.log').read().splitlines() if x.startswith('{')][-1]; l=json.loads(l)
print('$lib', $r, round(l['value'],1), round(l['ms_per_step'],2), {k: round(v,2) for k,v in l['breakdown_ms_rank0'].items()}, l['clocks']['sm_mhz'])
PY
  done
done
for lib in default "$@"; do
  setlib $lib
  timeout 600 python tools/sweep_c5.py --keeps 0.1 --reps 3 --kv-heads 8 2>&1 | grep '^{' | sed "s/^/$lib C5 /" | cut -c1-260
done
unset SB_LIB_PATH
