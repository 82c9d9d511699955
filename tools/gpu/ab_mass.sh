#!/bin/bash
# K4 sorted-mass A/B: profile / DST / closed-loop tests, sorted-mass kernel times (ncu, C3), C3 bench.
OUT=gpurun_out/${OUT:-ab_mass}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -k "coverage or profile or dst or closed or driver" > $OUT/pytest.log 2>&1; echo "pytest rc $?"; tail -n 2 $OUT/pytest.log
for lib in default $1; do
  if [ $lib = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$lib.so; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"row_sorted_mass|profile_partial" -c 6 --csv python bench.py --profile-only 2>/dev/null | grep gpu__time | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ' | sed "s/^/$lib sorted_mass ns: /"; echo
done
for r in 1 2; do for lib in default $1; do
  if [ $lib = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$lib.so; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-sub --no-cpu-baseline > $OUT/bench_${lib}_$r.log 2>&1
  python - <<PY
import json
l=[x for x in open('$OUT/bench_${lib}_$r.log').read().splitlines() if x.startswith('{')][-1]; l=json.loads(l)
print('$lib', $r, round(l['value'],1), round(l['ms_per_step'],2), {k: round(v,2) for k,v in l['breakdown_ms_rank0'].items()}, 'e2e', round(l['e2e']['value'],1), l['clocks']['sm_mhz'])
PY
done; done
unset SB_LIB_PATH
