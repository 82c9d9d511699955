#!/bin/bash
# N consecutive 4-GPU bench runs (release library), each under its own timeout,
# SB_HANG_DUMP armed (Python stacks of every rank if one stalls), NCCL_DEBUG=WARN (bench default);
# then DBG runs with the debug library (mbarrier wait timeouts + index traps).
RUNS=${1:-20}; DBG=${2:-3}; OUT=gpurun_out/n4_repeat; mkdir -p $OUT
one() {  # tag libpath
  if [ -n "$2" ]; then export SB_LIB_PATH=$2; else unset SB_LIB_PATH; fi
  SB_HANG_DUMP=240 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 300)) bench.py --gpus 4 --steps 3 --warmup 3 --no-sub --no-cpu-baseline \
    > $OUT/$1.log 2>&1
  rc=$?
  python - "$OUT/$1.log" "$1" "$rc" <<'PY'
import json, sys
path, tag, rc = sys.argv[1], sys.argv[2], sys.argv[3]
lines = [x for x in open(path).read().splitlines() if x.startswith('{')]
if not lines:
    print(tag, 'rc', rc, 'NO JSON LINE'); sys.exit()
l = json.loads(lines[-1])
print(tag, 'rc', rc, 'value', round(l['value'], 1), 'ms', round(l['ms_per_step'], 2), 'max/mean', round(l['max_over_mean'], 4),
      'worst step', round(l['max_over_mean_worst_step'], 4), 'clk', l['clocks'].get('sm_mhz'), l['clocks'].get('reasons'))
PY
}
for i in $(seq 1 $RUNS); do one rel_$i ""; done
for i in $(seq 1 $DBG); do one dbg_$i paper_2604_13847_b200/lib/libsparsebalance_b200_debug.so; done
unset SB_LIB_PATH
