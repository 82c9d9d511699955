"""Debug (not product): repeatability of profiler cells. Measures the mix cells x in XS at k = 2..9
three times (interleaved passes) and prints fwd + bwd per pass, to separate measurement noise
from real structure in k."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2604_13847_b200 import ops, profiler

XS = [40960, 65536]
KS = list(range(2, 10))
H, D, B = 32, 128, 128
T = max(XS)
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, do = (torch.randn((T, H, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
res = {}
for p in range(3):
    for x in XS:
        lens = profiler.mix_lengths(x)
        lay = ops.VarlenLayout.build(np.concatenate([[0], np.cumsum(lens)]).astype(np.int32), B)
        for kk in KS:
            f, b = profiler.measure_cell(q[:x], k[:x], v[:x], do[:x], lay, kk, 3, 1 / math.sqrt(D), 1)
            res.setdefault((x, kk), []).append((f, b))
for (x, kk), v_ in sorted(res.items()):
    print(x, kk, "fwd", [round(a, 3) for a, _ in v_], "bwd", [round(b, 3) for _, b in v_], "tot", [round(a + b, 3) for a, b in v_])
