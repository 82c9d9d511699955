#!/bin/bash
# Same-box A/B: in-tree library vs alt_lib/$1.so (C3 bench x2 each, alternating) + bwd parity tests
# + the C3 dK/dV per-CTA timeline. Usage: ab.sh <alt name> [out dir]
ALT=${1:-prev}; OUT=gpurun_out/${2:-ab}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_kernels_fullsize_gpu.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc $?"; tail -n 2 $OUT/pytest.log
timeout 300 python tools/c3_items.py > $OUT/c3_items.log 2>&1; echo "c3_items rc $?"; grep -v sorted $OUT/c3_items.log | grep "dkv\|fwd\|model" 
for r in 1 2; do
  for lib in default $ALT; do
    if [ $lib = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$lib.so; fi
    timeout 300 python bench.py --steps 5 --warmup 3 --no-sub --no-cpu-baseline > $OUT/bench_${lib}_$r.log 2>&1
    python - <<PY
import json
l=[x for x in open('$OUT/bench_${lib}_$r.log').read().splitlines() if x.startswith('{')][-1]; l=json.loads(l)
print('$lib', $r, round(l['value'],1), round(l['ms_per_step'],2), {k: round(v,2) for k,v in l['breakdown_ms_rank0'].items()}, l['clocks']['sm_mhz'])
PY
  done
done
unset SB_LIB_PATH
