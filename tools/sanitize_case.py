"""Small end-to-end case for compute-sanitizer (not product): every kernel family once --
scorer (K1 + K2), profile (K4), selector (K3), on-device DST (K8), forward (K5, with the O
residual), backward two-pass and fused (K6 + K7), block size 256 expansion, GQA group selection,
a partial last block and a zero-length sequence."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2604_13847_b200 import ops


def run(cu, hq, hkv, d, B, keep, seed):
    T = cu[-1]
    g = torch.Generator(device="cuda").manual_seed(seed)
    r = lambda h: torch.randn((T, h, d), generator=g, device="cuda").to(torch.bfloat16)  # noqa: E731
    q, k, v, do = r(hq), r(hkv), r(hkv), r(hq)
    lay = ops.VarlenLayout.build(cu, B)
    scale = 1.0 / math.sqrt(d)
    S = ops.block_scores(q, k, lay, scale)
    prof = ops.coverage_profile(S, lay)
    grid = torch.tensor([1, 2, 4, 8], dtype=torch.int32, device="cuda")
    ops.coverage_at_grid(prof, lay, grid)
    if B != 256:
        mb = torch.tensor([0, lay.nseq], dtype=torch.int32, device="cuda")
        one = lambda x: torch.tensor([x], dtype=torch.int32, device="cuda")  # noqa: E731
        ops.dst_decide(prof, lay, mb, one(4), one(2), one(1), grid, 0.1)
    k_seq = torch.tensor(np.maximum(1, np.ceil(keep * np.maximum(lay.nb_per_seq, 1))).astype(np.int32), device="cuda")
    group = hq // hkv
    idx, cnt = ops.topk_select(S, lay, k_seq, int(k_seq.max()), group=group)
    o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt, scale)
    ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt, scale)
    if d == 128 and B in (128, 256):
        ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt, scale, fused=True)
    torch.cuda.synchronize()


for case in (([0, 300, 300, 1000], 4, 2, 128, 128, 0.5, 1), ([0, 700, 1500], 2, 2, 64, 64, 0.6, 2),
             ([0, 1100, 1600], 4, 2, 128, 256, 0.6, 3)):
    run(*case)
    print("case ok", case[:5], flush=True)
print("sanitize case done")
