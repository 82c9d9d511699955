#!/bin/bash
# dK/dV pair walk A/B: in-tree lib (listing q blocks walked last-to-first) vs alt_lib/forward.so.
OUT=gpurun_out/ab_rev; mkdir -p $OUT
for r in 1 2; do
  for lib in default forward; do
    if [ $lib = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$lib.so; fi
    timeout 600 python bench.py --steps 5 --warmup 3 --no-sub --no-cpu-baseline > $OUT/bench_${lib}_$r.log 2>&1
    python - <<PY
import json
l=[x for x in open('$OUT/bench_${lib}_$r.log').read().splitlines() if x.startswith('{')][-1]; l=json.loads(l)
print('$lib', $r, round(l['value'],1), round(l['ms_per_step'],2), {k: round(v,2) for k,v in l['breakdown_ms_rank0'].items()})
PY
  done
done
for lib in default forward; do
  if [ $lib = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$lib.so; fi
  timeout 300 python tools/time_kernels.py 2>&1 | grep -E "attn_bwd_dkv" | sed "s/^/$lib C2 /"
  timeout 600 python tools/sweep_c5.py --keeps 0.1 --reps 5 --kv-heads 8 2>&1 | grep '^{' | sed "s/^/$lib C5 /" | cut -c1-200
  timeout 300 python tools/c4_items.py 2>&1 | grep planted | sed "s/^/$lib C4 /" | cut -c1-40,150-260
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none \
    -k regex:"attn_bwd_dkv" -c 1 --csv --log-file $OUT/ncu_$lib.csv python bench.py --profile-only > $OUT/ncu_$lib.log 2>&1; echo "ncu $lib rc $?"
done
unset SB_LIB_PATH
python - <<'PY'
import csv
for lib in ("default", "forward"):
    rows = list(csv.reader(open(f"gpurun_out/ab_rev/ncu_{lib}.csv")))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]; h = rows[hi]
    mi, vi = h.index("Metric Name"), h.index("Metric Value")
    print(lib, {r[mi]: r[vi] for r in rows[hi + 1:] if len(r) > vi})
PY
