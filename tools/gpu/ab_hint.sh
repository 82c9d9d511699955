#!/bin/bash
# L2 eviction-hint A/B (in-tree lib vs alt_lib/nohint.so): C3 bench x3 alternating, C2 kernel times,
# and the dK/dV DRAM bytes of the C3 step (ncu launch list, layer 0).
OUT=gpurun_out/ab_hint; mkdir -p $OUT
for r in 1 2 3; do
  for lib in default nohint; do
    if [ $lib = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$lib.so; fi
    timeout 600 python bench.py --steps 5 --warmup 3 --no-sub --no-cpu-baseline > $OUT/bench_${lib}_$r.log 2>&1
    python - <<PY
import json
l=[x for x in open('$OUT/bench_${lib}_$r.log').read().splitlines() if x.startswith('{')][-1]; l=json.loads(l)
print('$lib', $r, round(l['ms_per_step'],2), {k: round(v,2) for k,v in l['breakdown_ms_rank0'].items()})
PY
  done
done
for lib in default nohint; do
  if [ $lib = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=alt_lib/$lib.so; fi
  timeout 300 python tools/time_kernels.py 2>&1 | grep -E "attn_bwd|fwd " | sed "s/^/$lib C2 /"
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none \
    -k regex:"attn_bwd_dkv|attn_bwd_dq" -c 2 --csv --log-file $OUT/ncu_$lib.csv python bench.py --profile-only > $OUT/ncu_$lib.log 2>&1; echo "ncu $lib rc $?"
done
unset SB_LIB_PATH
python - <<'PY'
import csv, collections, re
for lib in ("default", "nohint"):
    rows = list(csv.reader(open(f"gpurun_out/ab_hint/ncu_{lib}.csv")))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]; h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    L = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi: continue
        n = re.search(r"([A-Za-z_0-9]+)(<[^>]*>)?\(", r[ki]).group(1)
        d = L.setdefault(int(r[ii]), {"name": n}); d[r[mi]] = float(r[vi].replace(",", ""))
    for d in L.values():
        print(lib, d["name"], "us %.1f" % (d["gpu__time_duration.sum"] / 1e3), "rd MB %.0f" % (d["dram__bytes_read.sum"] / 1e6),
              "wr MB %.0f" % (d["dram__bytes_write.sum"] / 1e6), "L2 hit %.1f" % d["lts__t_sector_hit_rate.pct"])
PY
