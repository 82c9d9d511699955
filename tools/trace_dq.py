"""Debug: phase timeline of CTA 0 of the dQ pass on the C2 workload (not product)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_13847_b200 import ops
import bench
lib = ops._lib()
lib.sb_debug_set_trace_dq.argtypes = [ctypes.c_void_p]
cu, k_seq = bench.workload(0)
T = int(cu[-1]); H, D, B = 32, 128, 128
lay = ops.VarlenLayout.build(cu, B)
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, do = (torch.randn((T, H, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
S = ops.block_scores(q, k, lay)
idx, cnt = ops.topk_select(S, lay, torch.from_numpy(k_seq).cuda(), int(k_seq.max()))
o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt)
buf = torch.zeros(256 * 16, dtype=torch.int64, device="cuda")
for it in range(3):
    lib.sb_debug_set_trace_dq(ctypes.c_void_p(buf.data_ptr() if it == 2 else 0))
    ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt)
torch.cuda.synchronize()
t = buf.cpu().numpy().reshape(256, 16).astype(np.int64)
n = int((t[:, 1] > 0).sum())
a, b = 2, n - 2
r = slice(a, b)
nx = slice(a + 1, b + 1)
med = lambda x: float(np.median(x))
print("blocks traced", n)
print("period (ds wait start -> next):", med(np.diff(t[a:b + 1, 0])))
print("UMMA ds_full wait:", med(t[r, 1] - t[r, 0]))
print("UMMA k_full wait (issue_s):", med(t[r, 3] - t[r, 2]))
print("UMMA issue_s start (after s_free) - prev dQ issued:", med(t[r, 2] - t[r, 6]))
print("UMMA v_full wait (issue_dp):", med(t[r, 5] - t[r, 4]))
print("UMMA dQ issue (ds seen -> after commit):", med(t[r, 6] - t[r, 1]))
print("math: s seen -> P done:", med(t[r, 9] - t[r, 8]))
print("math: dp wait:", med(t[r, 10] - t[r, 9]))
print("math: dp seen -> ds stored:", med(t[r, 11] - t[r, 10]))
print("math: ds stored -> next s seen:", med(t[nx, 8] - t[r, 11]))
print("producer k_empty wait:", med(t[r, 13] - t[r, 12]), " v_empty wait:", med(t[r, 15] - t[r, 14]))
print("V lead (v arrive issue -> dp issue wait start):", med(t[r, 4] - t[r, 15]))
