"""Debug: per-kernel device time of one C3 rank's 36-layer step (world of 2, rank 0) (not product)."""
import os, re, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
import bench
from paper_2604_13847_b200 import dp, ops
from paper_2604_13847_b200.host import api
world, rank, L, B, H, D = 2, 0, 36, 128, 32, 128
lengths_all, profiles_all = bench.c3_global_batch(world, bench.CFG["seed"], L)
table = api().synthesize_table(block_size=B)
bins = dp.assign_rank_batches(lengths_all, world, 5, "sab", table=table)
mine = [int(lengths_all[i]) for i in bins[rank][0]]
print("rank-0 micro-batch lengths", mine)
cu = np.concatenate([[0], np.cumsum(mine)]).astype(np.int32)
lay = ops.VarlenLayout.build(cu, B, device="cuda")
T = int(cu[-1])
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, do = (torch.randn((T, H, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
rng = np.random.default_rng(bench.CFG["seed"])
layer_scales = np.exp(rng.uniform(-0.5, 1.0, size=L))
routing = [[profiles_all[i][l] for i in bins[rank][0]] for l in range(L)]
# all ranks' estimates are needed for the pooled DST: emulate the allgather by building both ranks' inputs
pooled = []
for rr in range(world):
    m = [int(lengths_all[i]) for i in bins[rr][0]]
    prof = [[profiles_all[i][l] for l in range(L)] for i in bins[rr][0]]
    pooled.append((np.asarray(m), prof))
k_final, decisions, k_base, xs = dp.decide_budgets(pooled, table, dp.DstSettings(), L)
print("k_final rank0 per layer:", k_final[0].tolist())
nb = lay.nb_per_seq
scale = 1.0 / np.sqrt(D)
def step():
    S = ops.block_scores(q, k, lay, scale)
    for l in range(L):
        kk = np.minimum(k_final[0][l], nb).astype(np.int32)
        idx, cnt = ops.topk_select(S, lay, torch.from_numpy(kk).cuda(), int(max(1, kk.max())))
        o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt, scale)
        ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt, scale)
step(); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step(); torch.cuda.synchronize()
agg = {}
for e in prof.events():
    if e.device_type.name == "CUDA":
        mm = re.search(r"(attn_\w+|block_\w+|topk_\w+|bwd_prep\w*|transpose\w*|scan\w*|\w+_kernel)", e.name)
        n = mm.group(1) if mm else e.name[:40]
        agg.setdefault(n, []).append(e.device_time if hasattr(e, "device_time") else e.cuda_time)
for n, vv in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{n:42s} n={len(vv):4d} total {sum(vv) / 1000:.3f} ms  median {np.median(vv) / 1000:.4f} ms")
