"""Debug: dump block scores (C2 and a GQA / D=64 / B=64 case) to an .npz, for bit-identity
checks between two builds (SB_LIB_PATH) -- not product."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_13847_b200 import ops
import bench
out = []
for cu, hq, hkv, d, B in ((None, 32, 32, 128, 128), ([0, 1000, 1100, 2900, 9000], 8, 2, 64, 64)):
    if cu is None:
        cu, _ = bench.workload(0)
    T = int(cu[-1])
    lay = ops.VarlenLayout.build(cu, B)
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn((T, hq, d), generator=g, device="cuda").to(torch.bfloat16)
    k = torch.randn((T, hkv, d), generator=g, device="cuda").to(torch.bfloat16)
    out.append(ops.block_scores(q, k, lay).cpu().numpy())
torch.cuda.synchronize()
np.savez(sys.argv[1], *out)
