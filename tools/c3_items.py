"""Debug (not product): dK/dV work structure of one C3 layer (rank 0's micro-batch [2048 x3, 32768,
2048], 32 heads MHA, planted routing, k = 5): item pair-count histogram, the split order the
kernel builds (head-major, longest-first, chunks of <= cap pairs), and the modelled per-CTA load
of the static snake assignment (cost = c_item + c_pair * pairs per entry)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2604_13847_b200 import ops, synth
from paper_2604_13847_b200.host import api

H, D, B = 32, 128, 128
K = int(os.environ.get("KK", "5"))
lens = [2048, 2048, 2048, 32768, 2048]
_, routing = api().generate_samples(len(lens), 1, B, seed=7, sorted=False, dist=bench.C3_DIST)
nbs = [(L + B - 1) // B for L in lens]
rout = [np.resize(routing[s][0], nbs[s]) for s in range(len(lens))]
cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
lay = ops.VarlenLayout.build(cu, B)
q, k, v, do = synth.planted_qkv(lens, rout, H, H, D, B, seed=3, device="cuda")
k_seq = torch.from_numpy(np.minimum(K, np.asarray(nbs)).astype(np.int32)).cuda()
if os.environ.get("C2"):  # the C2 layer instead (bench.c2_workload: packed 32K, keep U[0.05, 0.5]), random inputs
    cu, ks = bench.c2_workload(0)
    lens = np.diff(cu).tolist()
    nbs = [(L + B - 1) // B for L in lens]
    K = int(ks.max())
    lay = ops.VarlenLayout.build(cu, B)
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v, do = (torch.randn((int(cu[-1]), H, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
    k_seq = torch.from_numpy(np.asarray(ks, np.int32)).cuda()
S = ops.block_scores(q, k, lay)
idx, cnt = ops.topk_select(S, lay, k_seq, K)
ic, cc = idx.cpu().numpy(), cnt.cpu().numpy()
nbt = int(lay.nb_total)
blk_off = np.concatenate([[0], np.cumsum(nbs)])
seq_of = np.searchsorted(blk_off, np.arange(nbt), side="right") - 1
items = np.zeros((H, nbt), np.int64)
for h in range(H):
    for gi in range(nbt):
        for j in ic[h, gi, :cc[h, gi]]:
            items[h, blk_off[seq_of[gi]] + j] += 1
pairs = items.ravel()
tot = int(pairs.sum())
print("pairs", tot, "items", pairs.size, "non-empty", int((pairs > 0).sum()))
vals, counts = np.unique(pairs, return_counts=True)
print("pair-count histogram:", dict(zip(vals.tolist(), counts.tolist())))
grid = 148
cap = max(16, -(-tot // (4 * grid)))
order = []
for h in range(H):
    its = sorted(range(nbt), key=lambda j: -items[h, j])
    for j in its:
        p = int(items[h, j])
        nc = min(15, -(-p // cap)) if p > cap else 1
        for c in range(nc):
            lo, hi = p * c // nc, p * (c + 1) // nc
            order.append((h, j, c, nc, hi - lo))
c_item, c_pair = float(os.environ.get("CI", "3400")), float(os.environ.get("CP", "2606"))
load = np.zeros(grid)
npairs = np.zeros(grid)
for t, e in enumerate(order):
    rnd, pos = divmod(t, grid)
    c = pos if rnd % 2 == 0 else grid - 1 - pos
    load[c] += c_item + c_pair * e[4]
    npairs[c] += e[4]
print(f"cap {cap}, entries {len(order)}, rounds {-(-len(order) // grid)}")
print(f"modelled cycles/CTA: mean {load.mean():.0f} max {load.max():.0f} (x{load.max() / load.mean():.3f}); "
      f"pairs/CTA mean {npairs.mean():.0f} max {npairs.max():.0f}")
print(f"  at 1.635 GHz: mean {load.mean() / 1.635e3:.0f} us, max {load.max() / 1.635e3:.0f} us")
o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt)


def timeit(fn, reps=10):
    ts = []
    for _ in range(reps + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts[2:]))


print(f"fwd {timeit(lambda: ops.sparse_attn_fwd(q, k, v, lay, idx, cnt)):.3f} ms, "
      f"bwd {timeit(lambda: ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt)):.3f} ms")

import ctypes
lib = ops._lib()
for nm in ("sb_debug_set_trace_bwd", "sb_debug_set_trace_dq", "sb_debug_set_trace"):
    getattr(lib, nm).argtypes = [ctypes.c_void_p]


def spans(setter, fn, label):
    """Per-CTA busy spans (globaltimer stamps at trace[8192 + 2 cta + {0, 1}]) of one launch."""
    buf = torch.zeros(8192 + 2 * 256, dtype=torch.int64, device="cuda")
    getattr(lib, setter)(ctypes.c_void_p(buf.data_ptr()))
    fn()
    torch.cuda.synchronize()
    getattr(lib, setter)(ctypes.c_void_p(0))
    st = buf.cpu().numpy()[8192:8192 + 2 * 256].reshape(256, 2).astype(np.int64)
    st = st[st[:, 0] > 0]
    t0 = st[:, 0].min()
    dur = (st[:, 1] - st[:, 0]) / 1e3
    end = (st[:, 1] - t0) / 1e3
    beg = (st[:, 0] - t0) / 1e3
    print(f"{label} per-CTA (us), {len(st)} CTAs: start max {beg.max():.1f}; busy min {dur.min():.0f} median "
          f"{np.median(dur):.0f} max {dur.max():.0f}; span {end.max():.0f}; mean busy / span {dur.mean() / end.max():.3f}")
    print(f"{label} per-CTA busy sorted (us):", np.sort(dur).astype(int).tolist())
    return dur


bwd = lambda: ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt)
spans("sb_debug_set_trace_bwd", bwd, "dkv")
spans("sb_debug_set_trace_dq", bwd, "dq")
spans("sb_debug_set_trace", lambda: ops.sparse_attn_fwd(q, k, v, lay, idx, cnt), "fwd")
