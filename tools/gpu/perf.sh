#!/bin/bash
# Quick perf check: C3 bench (no sub-records), C2 kernel times, dK/dV trace at C3 (k = 4).
OUT=gpurun_out/${1:-perf}; mkdir -p $OUT
timeout 600 python bench.py --steps 5 --warmup 3 --no-sub --no-cpu-baseline > $OUT/bench.log 2>&1; echo "bench rc $?"
python - <<PY
import json
l=[x for x in open('$OUT/bench.log').read().splitlines() if x.startswith('{')][-1]; l=json.loads(l)
print('C3 value', round(l['value'],1), 'ms', round(l['ms_per_step'],2), {k: round(v,2) for k,v in l['breakdown_ms_rank0'].items()}, 'k', l['k_final_rank0'][:3], 'fwdTF', round(l['fwd_tflops_rank0'],1), 'bwdTF', round(l['bwd_tflops_rank0'],1), 'clk', l['clocks']['sm_mhz'])
PY
timeout 300 python tools/time_kernels.py > $OUT/time_kernels.log 2>&1; echo "time rc $?"; grep -v Warn $OUT/time_kernels.log | head -6
C3K=4 timeout 300 python tools/trace_dkv.py > $OUT/trace_dkv_c3.log 2>&1; echo "trace rc $?"; cat $OUT/trace_dkv_c3.log | tail -32
