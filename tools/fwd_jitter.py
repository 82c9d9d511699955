"""Debug (not product): distribution of single-call device times of the forward / backward at C3 (k = 4)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2604_13847_b200 import ops, synth

lens = [2048, 2048, 2048, 32768, 2048]
lengths_all, routing_all = bench.c3_global_batch(1, 42, 36, sorted_=False)
cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
lay = ops.VarlenLayout.build(cu, 128)
q, k, v, do = synth.planted_qkv([int(x) for x in lengths_all], [r[0] for r in routing_all], 32, 32, 128, 128, 42,
                                device="cuda")
S = ops.block_scores(q, k, lay)
kseq = torch.full((5,), 4, dtype=torch.int32, device="cuda")
idx, cnt = ops.topk_select(S, lay, kseq, 4)
o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt)
for name, fn in (("fwd", lambda: ops.sparse_attn_fwd(q, k, v, lay, idx, cnt)),
                 ("fwd_nores", lambda: ops.sparse_attn_fwd(q, k, v, lay, idx, cnt, residual=False)),
                 ("topk", lambda: ops.topk_select(S, lay, kseq, 4)),
                 ("bwd", lambda: ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt))):
    ts = []
    for i in range(int(os.environ.get("N", "200"))):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts = np.array(ts)
    print(f"{name:10s} median {np.median(ts):.3f} p90 {np.percentile(ts, 90):.3f} max {ts.max():.3f} n>1.5x {(ts > 1.5 * np.median(ts)).sum()}")
