#!/bin/bash
# Programmatic dependent launch A/B: full GPU test suite on the new lib, then C3 bench alternating
# with alt_lib/nopdl.so, and the timeline's kernel gaps.
OUT=gpurun_out/ab_pdl; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_kernels_gpu.py tests/test_kernels_fullsize_gpu.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc $?"; tail -n 3 $OUT/pytest.log
for r in 1 2; do
  for lib in default pdl1; do
    if [ $lib = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$lib.so; fi
    timeout 600 python bench.py --steps 5 --warmup 3 --no-sub --no-cpu-baseline > $OUT/bench_${lib}_$r.log 2>&1
    python - <<PY
import json
l=[x for x in open('$OUT/bench_${lib}_$r.log').read().splitlines() if x.startswith('{')][-1]; l=json.loads(l)
print('$lib', $r, round(l['value'],1), round(l['ms_per_step'],2), {k: round(v,2) for k,v in l['breakdown_ms_rank0'].items()})
PY
  done
done
unset SB_LIB_PATH
timeout 300 python tools/time_kernels.py 2>&1 | grep -E "^fwd" | sed "s/^/pdl C2 /"
SB_LIB_PATH=alt_lib/pdl1.so timeout 300 python tools/time_kernels.py 2>&1 | grep -E "^fwd" | sed "s/^/pdl1 C2 /"
