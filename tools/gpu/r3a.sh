#!/bin/bash
mkdir -p gpurun_out/r3a
timeout 900 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k "split or deterministic or bwd" > gpurun_out/r3a/pytest.log 2>&1; echo "pytest rc $?"; tail -n 2 gpurun_out/r3a/pytest.log
timeout 600 python tools/c4_items.py 2>&1 | grep -v Warn
for r in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-sub --no-cpu-baseline > gpurun_out/r3a/bench_$r.log 2>&1; python - <<PY
import json
l=[x for x in open('gpurun_out/r3a/bench_$r.log').read().splitlines() if x.startswith('{')][-1]; l=json.loads(l)
print('C3', round(l['value'],1), round(l['ms_per_step'],2), {k: round(v,2) for k,v in l['breakdown_ms_rank0'].items()}, l['k_final_rank0'][:3], l['clocks']['sm_mhz'])
PY
done
