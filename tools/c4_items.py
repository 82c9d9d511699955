"""Debug (not product): dK/dV item sizes under planted (column-concentrated) routing vs random
inputs, for one C4 micro-batch (3 x 32K + 7 x 2K, GQA 32/8, k = 5): per-item pair counts, the
snake-LPT makespan in pairs, and the kernel times of the backward on both inputs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2604_13847_b200 import ops, synth
from paper_2604_13847_b200.host import api

HQ, HKV, D, B = 32, int(os.environ.get("HKV", "8")), 128, 128
K = int(os.environ.get("KK", "5"))
lens = [32768, 2048, 2048, 32768, 2048, 2048, 2048, 2048, 32768, 2048]
h = api()
_, routing = h.generate_samples(len(lens), 1, B, seed=7, sorted=False,
                                dist=dict(short_weight=0.6, short_log_mean=float(np.log(2048)), short_log_sigma=0.0,
                                          long_log_mean=float(np.log(32768)), long_log_sigma=0.0))
nbs = [(L + B - 1) // B for L in lens]
rout = [np.resize(routing[s][0], nbs[s]) for s in range(len(lens))]
cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
lay = ops.VarlenLayout.build(cu, B)
g = torch.Generator(device="cuda").manual_seed(0)
T = int(cu[-1])
inputs = {
    "planted": synth.planted_qkv(lens, rout, HQ, HKV, D, B, seed=3, device="cuda"),
    "random": tuple(torch.randn((T, hh, D), generator=g, device="cuda").to(torch.bfloat16) for hh in (HQ, HKV, HKV, HQ)),
}
k_seq = torch.from_numpy(np.minimum(K, np.asarray(nbs)).astype(np.int32)).cuda()
grid = 148


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


for name, (q, k, v, do) in inputs.items():
    S = ops.block_scores(q, k, lay)
    idx, cnt = ops.topk_select(S, lay, k_seq, K, group=HQ // HKV)
    o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt)
    ic, cc = idx.cpu().numpy(), cnt.cpu().numpy()
    nbt = int(lay.nb_total)
    blk_off = lay.blk_off_host
    # transposed counts: item (selection row r, global key block) -> listing q blocks
    rows = ic.shape[0]
    ic3, cc2 = ic, cc
    seq_of = np.searchsorted(blk_off, np.arange(nbt), side="right") - 1
    items = np.zeros((rows, nbt), np.int64)
    for r in range(rows):
        for gi in range(nbt):
            for j in ic3[r, gi, :cc2[r, gi]]:
                items[r, blk_off[seq_of[gi]] + j] += 1
    sg = HQ // rows
    pairs = (items * sg).ravel()
    tot = pairs.sum()
    srt = np.sort(pairs)[::-1]
    load = np.zeros(grid)
    for t, p in enumerate(srt):  # snake LPT
        rnd, pos = divmod(t, grid)
        c = pos if rnd % 2 == 0 else grid - 1 - pos
        load[c] += p
    tb = timeit(lambda: ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt))
    tf = timeit(lambda: ops.sparse_attn_fwd(q, k, v, lay, idx, cnt))
    print(f"{name}: pairs {tot}, items>0 {int((pairs > 0).sum())}, max item {pairs.max()}, "
          f"top10 {srt[:10].tolist()}, per-CTA mean {tot / grid:.0f}, snake-LPT makespan {load.max():.0f} "
          f"(x{load.max() / (tot / grid):.2f}), fwd {tf:.3f} ms, bwd {tb:.3f} ms")
