"""Debug (not product): GPU timeline of one C3 step (bench.py's N=1 workload) under torch.profiler.

Prints per-kernel totals (steady state, warm) and the idle gaps between consecutive kernels on
the compute stream, to separate kernel time from launch / host-side gaps in the bench's phases."""
import collections
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import bench
from paper_2604_13847_b200 import dp, ops, synth

layers = int(os.environ.get("LAYERS", "36"))
lengths_all, routing_all = bench.c3_global_batch(1, 42, layers, sorted_=False)
table, _ = bench.cost_table()
bins = dp.assign_rank_batches(lengths_all, 1, 5, "sab", table=table)
ids = list(bins[0][0])
mine = [int(lengths_all[i]) for i in ids]
cu = np.concatenate([[0], np.cumsum(mine)]).astype(np.int32)
lay = ops.VarlenLayout.build(cu, 128)
q, k, v, do = synth.planted_qkv(mine, [routing_all[i][0] for i in ids], 32, 32, 128, 128, seed=42, device="cuda")
cfg = dp.DstSettings()
cfg.budget_grid = list(range(1, 257))
runner = dp.DPStep(dp.RankBatch(np.asarray(mine), ids, lay), q, k, v, do, synth.layer_scales(layers, 42), table, cfg)
for _ in range(3):
    runner.run()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    runner.run()
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
agg = collections.defaultdict(float)
cnt = collections.Counter()
gaps = []
for a, b in zip(ev, ev[1:]):
    gaps.append(b.time_range.start - a.time_range.end)
for e in ev:
    import re as _re
    m_ = _re.search(r"([A-Za-z_0-9]+)(<[^>]*>)?\(", e.name)
    n = (m_.group(1) + (m_.group(2) or "")) if m_ else e.name[:48]
    agg[n] += e.time_range.end - e.time_range.start
    cnt[n] += 1
span = ev[-1].time_range.end - ev[0].time_range.start
busy = sum(agg.values())
print(f"step span {span / 1e3:.2f} ms, kernel busy {busy / 1e3:.2f} ms, gaps {sum(g for g in gaps if g > 0) / 1e3:.2f} ms "
      f"({len(ev)} kernels), k_final {runner.last['k_final'][0].tolist()[:4]}...")
for n, t in sorted(agg.items(), key=lambda x: -x[1])[:25]:
    print(f"  {n:48s} n={cnt[n]:4d} total {t / 1e3:8.3f} ms  mean {t / cnt[n]:8.1f} us")
big = sorted(((g, i) for i, g in enumerate(gaps)), reverse=True)[:10]
for g, i in big:
    print(f"  gap {g:8.1f} us after {ev[i].name[:60]} -> {ev[i + 1].name[:40]}")
