#!/bin/bash
# K4 profile A/B: bit-exact profile / DST tests, then the C3 bench (full e2e) in-tree vs alt_lib/$1.so.
OUT=gpurun_out/${OUT:-ab_prof}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_dst_device_gpu.py -m gpu -x -q -k "coverage or dst or profile" > $OUT/pytest.log 2>&1; echo "pytest rc $?"; tail -n 2 $OUT/pytest.log
for r in 1 2; do for lib in default $1; do
  if [ $lib = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$lib.so; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-sub --no-cpu-baseline > $OUT/bench_${lib}_$r.log 2>&1
  python - <<PY
import json
l=[x for x in open('$OUT/bench_${lib}_$r.log').read().splitlines() if x.startswith('{')][-1]; l=json.loads(l)
print('$lib', $r, round(l['value'],1), round(l['ms_per_step'],2), {k: round(v,2) for k,v in l['breakdown_ms_rank0'].items()}, 'e2e', round(l['e2e']['value'],1), round(l['e2e']['ms_per_step'],1), l['clocks']['sm_mhz'])
PY
done; done
unset SB_LIB_PATH
