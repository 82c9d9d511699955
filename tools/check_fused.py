"""Debug: the fused backward on a few small cases vs the fp64 oracle and vs the two-pass (not product)."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_13847_b200 import ops
from oracle import device as orc
from tests.tolerance import check_bf16

def bits(t):
    return t.cpu().contiguous().view(torch.int16).numpy().view(np.uint16)

def run(cu, hq, hkv, keep, seed):
    T = cu[-1]; D = B = 128
    g = torch.Generator(device="cuda").manual_seed(seed)
    r = lambda h: torch.randn((T, h, D), generator=g, device="cuda").to(torch.bfloat16)
    q, k, v, do = r(hq), r(hkv), r(hkv), r(hq)
    lay = ops.VarlenLayout.build(cu, B)
    S = ops.block_scores(q, k, lay)
    nb = lay.nb_per_seq
    kseq = torch.tensor(np.maximum(1, np.ceil(keep * nb)).astype(np.int32), device="cuda")
    idx, cnt = ops.topk_select(S, lay, kseq, int(kseq.max()), group=hq // hkv)
    scale = 1 / math.sqrt(D)
    o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt, scale)
    torch.cuda.synchronize()
    t0 = time.time()
    dq, dk, dv = ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt, scale, fused=True)
    torch.cuda.synchronize()
    print(f"fused bwd done in {time.time() - t0:.3f}s", flush=True)
    dq2, dk2, dv2 = ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt, scale)
    torch.cuda.synchronize()
    ic, cc = idx.cpu().numpy(), cnt.cpu().numpy()
    ro, rlse = orc.sparse_attn_fwd(bits(q), bits(k), bits(v), cu, B, ic, cc, scale)
    rdq, rdk, rdv = orc.sparse_attn_bwd(bits(q), bits(k), bits(v), ro, bits(do), rlse, cu, B, ic, cc, scale)
    for name, got, ref in (("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv), ("dq2", dq2, rdq), ("dk2", dk2, rdk), ("dv2", dv2, rdv)):
        try:
            e = check_bf16(got, ref, name)
            print(f"  {name}: max err {e[0]:.3e} worst row {e[1]:.3e} fro {e[2]:.3e}")
        except AssertionError as ex:
            print(f"  {name}: FAIL {ex}")

for case in (([0, 128], 1, 1, 1.0, 1), ([0, 1000, 3000], 2, 2, 0.5, 2), ([0, 1000, 1100, 2900, 6000], 8, 2, 0.4, 3)):
    print(case, flush=True)
    run(*case)
print("done")
