"""Debug: phase timeline of CTA 0 of the dK/dV pass on the C2 workload (not product)."""
import ctypes, math, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_13847_b200 import ops
import bench
lib = ops._lib()
lib.sb_debug_set_trace_bwd.argtypes = [ctypes.c_void_p]
if os.environ.get("C3K"):  # C3 rank micro-batch [2048 x3, 32768, 2048] at a fixed keep count
    lens = [2048, 2048, 2048, 32768, 2048]
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    k_seq = np.minimum(int(os.environ["C3K"]), (np.array(lens) + 127) // 128).astype(np.int32)
else:
    cu, k_seq = bench.workload(0)
T = int(cu[-1]); H, D, B = 32, 128, 128
lay = ops.VarlenLayout.build(cu, B)
g = torch.Generator(device="cuda").manual_seed(0)
if os.environ.get("PLANTED"):  # planted column-concentrated routing (synth.py), as the bench's C3 step
    from paper_2604_13847_b200 import synth
    from paper_2604_13847_b200.host import api
    lens_p = np.diff(cu).tolist()
    _, routing = api().generate_samples(len(lens_p), 1, B, seed=7, sorted=False, dist=bench.C3_DIST)
    rout = [np.resize(routing[s_][0], (L + B - 1) // B) for s_, L in enumerate(lens_p)]
    q, k, v, do = synth.planted_qkv(lens_p, rout, H, H, D, B, seed=3, device="cuda")
else:
    q, k, v, do = (torch.randn((T, H, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
S = ops.block_scores(q, k, lay)
idx, cnt = ops.topk_select(S, lay, torch.from_numpy(k_seq).cuda(), int(k_seq.max()))
o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt)
buf = torch.zeros(8192 + 2 * 256, dtype=torch.int64, device="cuda")
for it in range(3):
    lib.sb_debug_set_trace_bwd(ctypes.c_void_p(buf.data_ptr() if it == 2 else 0))
    ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt)
torch.cuda.synchronize()
allb = buf.cpu().numpy().astype(np.int64)
t = allb[:4096].reshape(256, 16)
ti = allb[4096:4608].reshape(64, 8)
n = int((t[:, 0] > 0).sum())
r = slice(2, n - 2)
print("pairs traced", n)
med = lambda x: float(np.median(x))
nx = slice(3, n - 1)
print("period (pds wait start -> next):", med(np.diff(t[2:n - 1, 0])))
print("UMMA: pds wait:", med(t[r, 1] - t[r, 0]))
print("UMMA: dV + dK issue:", med(t[r, 10] - t[r, 1]))
print("UMMA: q_full wait in issue_st:", med(t[r, 9] - t[r, 8]))
print("math: st seen -> P done:", med(t[r, 5] - t[r, 4]))
print("math: dpt wait:", med(t[r, 6] - t[r, 5]))
print("math: dpt seen -> pds arrive:", med(t[r, 7] - t[r, 6]))
print("math: pds arrive -> next st seen:", med(t[nx, 4] - t[r, 7]))
print("producer: q_empty wait:", med(t[r, 12] - t[r, 11]))
print("producer: lead of q_full arrive over its use:", med(t[r, 8] - t[r, 13]))
print("producer: Q TMA issue -> landed:", med(t[r, 14] - t[r, 12]))
print("producer: Q landed -> St issue start:", med(t[r, 8] - t[r, 14]))
print("UMMA: issue_st start -> St issued (incl. waits):", med(t[r, 9] - t[r, 8]))

nt = int((ti[:, 0] > 0).sum())
print("items traced", nt)
print("t  KV issued | issuer kv wait start | kv_full seen | (wait) | prev acc_done seen | prev epi done")
for tt in range(1, min(nt, 14)):
    print(tt, int(ti[tt, 0] - ti[tt, 0]), int(ti[tt, 1] - ti[tt, 0]), int(ti[tt, 2] - ti[tt, 0]), int(ti[tt, 2] - ti[tt, 1]),
          int(ti[tt - 1, 3] - ti[tt, 0]), int(ti[tt - 1, 4] - ti[tt, 0]))
print("item (pairs: period K/V issue -> next K/V issue), items 1..:", [f"{int(ti[tt, 5])}:{int(ti[tt + 1, 0] - ti[tt, 0])}" for tt in range(1, min(nt - 1, 40))])
print("median K/V latency (issued -> seen):", float(np.median(ti[1:nt, 2] - ti[1:nt, 0])))
print("median issuer wait on kv_full:", float(np.median(ti[1:nt, 2] - ti[1:nt, 1])))
if os.environ.get("PAIRS"):  # per-pair event times (cycles) relative to the producer's pair start, pairs 1..12
    names = {11: "prod start", 12: "q_empty ok", 13: "aug written", 14: "Q landed", 8: "iss st start", 9: "q_full seen",
             4: "math st seen", 5: "P done", 6: "dpt seen", 7: "pds arrive", 1: "iss pds seen", 10: "dV issued"}
    for gg in range(1, 13):
        base = t[gg, 11]
        print(gg, "  ".join(f"{names[s_]}={int(t[gg, s_] - base)}" for s_ in (12, 13, 14, 8, 9, 4, 5, 6, 7, 1, 10)))

