#!/bin/bash
# Multi-GPU bench: tools/gpu/scale.sh OUTDIR N "<extra bench args>"
OUT=gpurun_out/$1; mkdir -p $OUT; N=$2
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus $N --steps 5 --warmup 3 $3 > $OUT/bench_N$N.log 2>&1; echo "bench N=$N rc $?"
python - <<PY
import json
l=[x for x in open('$OUT/bench_N$N.log').read().splitlines() if x.startswith('{')][-1]
l=json.loads(l)
print('N', l['n_gpus'], 'value', round(l['value'],1), 'ms', round(l['ms_per_step'],2), 'busy', [round(x,1) for x in l['busy_ms_per_rank']],
      'max/mean', round(l['max_over_mean'],4), 'worst step', round(l['max_over_mean_worst_step'],4), 'k0', l['k_final_rank0'][:4], 'tokens', l['config']['tokens_per_rank'],
      'clk', l['clocks'], 'gradAR', (l.get('grad_allreduce') or {}).get('ms_per_step_with_allreduce'))
PY
