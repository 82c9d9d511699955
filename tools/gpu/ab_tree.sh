#!/bin/bash
# A/B against a whole previous tree (alt_lib/head_tree: its own python + lib), for ABI-changing
# builds: parity tests on the in-tree build, then C3 layer fwd/bwd and the C3 bench, alternating.
OUT=$PWD/gpurun_out/${OUT:-ab_tree}; mkdir -p $OUT
ROOT=$PWD
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_kernels_fullsize_gpu.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc $?"; tail -n 3 $OUT/pytest.log
for r in 1 2; do for t in new old; do
  if [ $t = new ]; then cd $ROOT; else cd $ROOT/alt_lib/head_tree; fi
  timeout 300 python tools/c3_items.py 2>&1 | grep "^fwd" | head -1 | sed "s/^/$t C3 $r /"
  C2=1 timeout 300 python tools/c3_items.py 2>&1 | grep "^fwd" | head -1 | sed "s/^/$t C2 $r /"
  timeout 300 python bench.py --steps 5 --warmup 3 --no-sub --no-cpu-baseline > $OUT/bench_${t}_$r.log 2>&1
  python - <<PY
import json
l=[x for x in open('$OUT/bench_${t}_$r.log').read().splitlines() if x.startswith('{')][-1]; l=json.loads(l)
print('$t', $r, round(l['value'],1), round(l['ms_per_step'],2), {k: round(v,2) for k,v in l['breakdown_ms_rank0'].items()}, l['clocks']['sm_mhz'])
PY
done; done
cd $ROOT
