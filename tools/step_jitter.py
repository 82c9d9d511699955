"""Debug (not product): per-step device time of 20 consecutive C3 steps (bench's N=1 workload)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2604_13847_b200 import dp, ops, synth

lengths_all, routing_all = bench.c3_global_batch(1, 42, 36, sorted_=False)
table, _ = bench.cost_table()
bins = dp.assign_rank_batches(lengths_all, 1, 5, "sab", table=table)
ids = list(bins[0][0]); mine = [int(lengths_all[i]) for i in ids]
cu = np.concatenate([[0], np.cumsum(mine)]).astype(np.int32)
lay = ops.VarlenLayout.build(cu, 128)
q, k, v, do = synth.planted_qkv(mine, [routing_all[i][0] for i in ids], 32, 32, 128, 128, seed=42, device="cuda")
cfg = dp.DstSettings(); cfg.budget_grid = list(range(1, 257))
runner = dp.DPStep(dp.RankBatch(np.asarray(mine), ids, lay), q, k, v, do, synth.layer_scales(36, 42), table, cfg)
for _ in range(3):
    runner.run()
torch.cuda.synchronize()
out = []
for i in range(int(os.environ.get("N", "20"))):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    a.record(); runner.run(); b.record()
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    out.append((a.elapsed_time(b), (h1 - h0) * 1e3, sum(x.elapsed_time(y) for x, y in runner.last["busy"])))
for r in out:
    print("step ms %.2f  host-enqueue ms %.2f  busy ms %.2f" % r)

# Back to back (no sync between steps), per-step phase marks as bench.py records them.
marks = []
for i in range(int(os.environ.get("N", "20"))):
    m = bench.Marker(torch, torch.cuda.current_stream())
    m("start")
    runner.run(mark=m)
    marks.append(m)
torch.cuda.synchronize()
for m in marks:
    d = m.durations()
    fwd_ev = [b.elapsed_time(a) for (ta, a), (tb, b) in zip(m.marks, m.marks[1:]) if ta == "bwd" and tb == "fwd"]
    print("b2b step: decided %.2f fwd %.2f bwd %.2f  max fwd-layer %.2f" % (d.get("decided", 0), d.get("fwd", 0),
                                                                            d.get("bwd", 0), -min(fwd_ev or [0])))
