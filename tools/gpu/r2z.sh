#!/bin/bash
mkdir -p gpurun_out/r2z
timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_kernels_fullsize_gpu.py -m gpu -x -q > gpurun_out/r2z/pytest.log 2>&1; echo "pytest rc $?"; tail -n 3 gpurun_out/r2z/pytest.log
timeout 600 python tools/timeline_c3.py > gpurun_out/r2z/timeline.log 2>&1; echo "tl rc $?"; grep -v Warn gpurun_out/r2z/timeline.log | head -24
for r in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-sub --no-cpu-baseline > gpurun_out/r2z/bench_$r.log 2>&1; python - <<PY
import json
l=[x for x in open('gpurun_out/r2z/bench_$r.log').read().splitlines() if x.startswith('{')][-1]; l=json.loads(l)
print('C3', round(l['value'],1), round(l['ms_per_step'],2), {k: round(v,2) for k,v in l['breakdown_ms_rank0'].items()}, l['k_final_rank0'][:3], l['clocks']['sm_mhz'])
PY
done
