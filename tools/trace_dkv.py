"""Debug: phase timeline of CTA 0 of the dK/dV pass on the C2 workload (not product)."""
import ctypes, math, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_13847_b200 import ops
import bench
lib = ops._lib()
lib.sb_debug_set_trace_bwd.argtypes = [ctypes.c_void_p]
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
    lib.sb_debug_set_trace_bwd(ctypes.c_void_p(buf.data_ptr() if it == 2 else 0))
    ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt)
torch.cuda.synchronize()
t = buf.cpu().numpy().reshape(256, 16).astype(np.int64)
n = int((t[:, 0] > 0).sum())
r = slice(2, n - 2)
print("pairs traced", n)
print("median period (pt wait start -> next):", np.median(np.diff(t[r, 0])))
print("median pt_full wait (MMA):", np.median(t[r, 1] - t[r, 0]))
print("median dV issue + St issue (pt seen -> before dst wait):", np.median(t[r, 2] - t[r, 1]))
print("median dst_full wait (MMA):", np.median(t[r, 3] - t[r, 2]))
print("median dK issue + dPt issue (dst seen -> next pt wait):", np.median(t[3:n-1, 0] - t[2:n-2, 3]))
print("softmax: st seen -> P stored:", np.median(t[r, 5] - t[r, 4]))
print("softmax: P stored -> dpt seen:", np.median(t[r, 6] - t[r, 5]))
print("softmax: dpt seen -> dS stored:", np.median(t[r, 7] - t[r, 6]))
print("softmax: dS stored -> next st seen:", np.median(t[3:n-1, 4] - t[2:n-2, 7]))
print("UMMA: q_full wait in issue_st:", np.median(t[3:n-1, 9] - t[3:n-1, 8]))
print("UMMA: dV issue (pt seen -> issue_st start):", np.median(t[3:n-1, 8] - t[2:n-2, 1]))
print("UMMA: dK issue (dst seen -> after q_empty commit):", np.median(t[r, 10] - t[r, 3]))
print("producer: q_empty wait:", np.median(t[r, 12] - t[r, 11]))
print("producer: lead of q_full arrive over its use:", np.median(t[3:n-1, 8] - t[3:n-1, 13]))
print("producer: TMA+vec issue time:", np.median(t[r, 13] - t[r, 12]))
