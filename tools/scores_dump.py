"""Debug (not product): dump K2 block scores for fixed inputs (C2 layout, MHA and GQA) to compare
two library builds bit for bit: SB_LIB_PATH=... python tools/scores_dump.py out.npz"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2604_13847_b200 import ops

cu, _ = bench.workload(0)
T = int(cu[-1])
out = {}
for hkv, d in ((32, 128), (8, 128), (8, 64)):
    g = torch.Generator(device="cuda").manual_seed(1)
    q = torch.randn((T, 32, d), generator=g, device="cuda").to(torch.bfloat16)
    k = torch.randn((T, hkv, d), generator=g, device="cuda").to(torch.bfloat16)
    for B in (64, 128):
        lay = ops.VarlenLayout.build(cu, B)
        out[f"h{hkv}_d{d}_b{B}"] = ops.block_scores(q, k, lay, 0.3).cpu().numpy()
np.savez(sys.argv[1], **out)
print("dumped", {k: v.shape for k, v in out.items()})
