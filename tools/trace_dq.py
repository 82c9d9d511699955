"""Debug: phase timeline of CTA 0 of the dQ pass on the C2 workload (not product)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_13847_b200 import ops
import bench
lib = ops._lib()
lib.sb_debug_set_trace_dq.argtypes = [ctypes.c_void_p]
if os.environ.get("C3K"):  # C3 rank micro-batch [2048 x3, 32768, 2048] at a fixed keep count
    lens = [2048, 2048, 2048, 32768, 2048]
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    k_seq = np.minimum(int(os.environ["C3K"]), (np.array(lens) + 127) // 128).astype(np.int32)
else:
    cu, k_seq = bench.workload(0)
T = int(cu[-1]); H, D, B = 32, 128, 128
lay = ops.VarlenLayout.build(cu, B)
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, do = (torch.randn((T, H, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
S = ops.block_scores(q, k, lay)
idx, cnt = ops.topk_select(S, lay, torch.from_numpy(k_seq).cuda(), int(k_seq.max()))
o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt)
buf = torch.zeros(8192 + 2 * 256, dtype=torch.int64, device="cuda")
for it in range(3):
    lib.sb_debug_set_trace_dq(ctypes.c_void_p(buf.data_ptr() if it == 2 else 0))
    ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt)
torch.cuda.synchronize()
allb = buf.cpu().numpy().astype(np.int64)
t = allb[:4096].reshape(256, 16)
ti = allb[4096:4352].reshape(64, 4)
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
d = np.diff(t[2:n - 1, 0])
print("period percentiles 10/50/90/99:", [float(np.percentile(d, q)) for q in (10, 50, 90, 99)])
big = d > 2 * np.median(d)
print("blocks with > 2x median period:", int(big.sum()), "of", len(d), "; their excess:", float((d[big] - np.median(d)).sum()), "; total:", float(d.sum()))
nq = int((ti[:, 0] > 0).sum())
print("items", nq, "; math dq_done -> epilogue stores done:", med(ti[1:nq, 1] - ti[1:nq, 0]))
print("issuer stage_full wait (Q/dO staging for the next item):", med(ti[2:nq, 3] - ti[2:nq, 2]))
print("issuer load_qdo start - math dq_done of the previous item:", med(ti[2:nq, 2] - ti[1:nq - 1, 0]))
if os.environ.get("ROWS"):  # raw per-block stamps relative to block 0's ds-wait start
    names = {0: "ds wait", 1: "ds seen", 2: "iss_s start", 3: "k_full seen", 4: "v wait", 5: "v seen", 6: "dQ issued",
             8: "math s seen", 9: "P done", 10: "dp seen", 11: "ds stored"}
    base = t[0, 0]
    for gg in range(int(os.environ["ROWS"])):
        print(gg, "  ".join(f"{nm}={int(t[gg, sl] - base)}" for sl, nm in names.items()))
    for qq in range(min(nq, 8)):
        print("item", qq, [int(ti[qq, j] - base) for j in range(4)])
