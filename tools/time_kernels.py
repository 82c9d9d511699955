"""Debug: median device time of the C2 layer's fwd and bwd (dkv + dq) over many reps (not product)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_13847_b200 import ops
import bench
cu, k_seq = bench.workload(0)
T = int(cu[-1]); H, D, B = 32, 128, 128
lay = ops.VarlenLayout.build(cu, B)
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, do = (torch.randn((T, H, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
S = ops.block_scores(q, k, lay)
idx, cnt = ops.topk_select(S, lay, torch.from_numpy(k_seq).cuda(), int(k_seq.max()))
o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt)
reps = int(os.environ.get("REPS", "30"))
def timeit(fn):
    ts = []
    for _ in range(reps + 3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts[3:]))
tf = timeit(lambda: ops.sparse_attn_fwd(q, k, v, lay, idx, cnt))
tb = timeit(lambda: ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt))
print(f"fwd {tf:.4f} ms  bwd {tb:.4f} ms")
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(10):
        ops.sparse_attn_fwd(q, k, v, lay, idx, cnt)
        ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt)
        ops.coverage_profile(S, lay)
        ops.block_scores(q, k, lay)
    torch.cuda.synchronize()
agg = {}
for e in prof.events():
    if e.device_type.name == "CUDA":
        import re
        m = re.search(r"(attn_\w+|block_\w+|topk_\w+|bwd_prep\w*|transpose\w*|scan\w*|\w+_kernel)", e.name)
        n = m.group(1) if m else e.name[:40]
        agg.setdefault(n, []).append(e.device_time if hasattr(e, "device_time") else e.cuda_time)
for n, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{n:42s} n={len(v):3d} median {np.median(v) / 1000:.4f} ms")
