"""Debug: phase timeline of CTA 0 of the forward kernel on the C2 workload (not product)."""
import ctypes, math, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_13847_b200 import ops
import bench
lib = ops._lib()
lib.sb_debug_set_trace.argtypes = [ctypes.c_void_p]
cu, k_seq = bench.workload(0)
T = int(cu[-1]); H, D, B = 32, 128, 128
lay = ops.VarlenLayout.build(cu, B)
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((T, H, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
S = ops.block_scores(q, k, lay)
idx, cnt = ops.topk_select(S, lay, torch.from_numpy(k_seq).cuda(), int(k_seq.max()))
buf = torch.zeros(256 * 32, dtype=torch.int64, device="cuda")
for it in range(3):
    lib.sb_debug_set_trace(ctypes.c_void_p(buf.data_ptr() if it == 2 else 0))
    ops.sparse_attn_fwd(q, k, v, lay, idx, cnt)
torch.cuda.synchronize()
allb = buf.cpu().numpy().astype(np.int64)
t = allb[:2048].reshape(256, 8)
pw = allb[2048:3072].reshape(256, 4)
ps = allb[3072:4096].reshape(256, 4)
ep = allb[4096:5120].reshape(256, 4)
in4 = allb[5120:6144].reshape(256, 4)
base = t[0, 0]
names = ["mma:before k_full", "mma:k ready/QK issue", "mma:PV v ready", "mma:PV p_full seen", "smx:S ready", "smx:P done", "smx:o_done seen"]
print("g  " + " | ".join(f"{n:>20s}" for n in names))
for gg in range(0, 60):
    row = t[gg]
    print(f"{gg:3d} " + " | ".join(f"{(x - base) if x else -1:20d}" for x in row[:7]))
d = np.diff(t[1:60, 1])
print("median cycles between QK issues:", np.median(d))
print("median softmax busy (P done - S ready):", np.median(t[1:60, 5] - t[1:60, 4]))
print("median S ready -> next S ready:", np.median(np.diff(t[1:60, 4])))
r = slice(2, 58)
print("median k_full wait:", np.median(t[r, 1] - t[r, 0]))
print("median QK issue -> v_full seen (prev PV):", np.median(t[r, 2] - t[r, 1]))
print("median v_full -> p_full seen:", np.median(t[r, 3] - t[r, 2]))
print("median p_full seen -> next before-k_full:", np.median(t[3:59, 0] - t[2:58, 3]))
print("median S ready after QK issue:", np.median(t[r, 4] - t[r, 1]))
print("median o_done wait (P done -> o_done seen):", np.median(t[r, 6] - t[r, 5]))
print("per-warp arrival relative to warp 2 (warps 2..5), median over blocks:", [float(np.median(pw[4:40, w] - pw[4:40, 0])) for w in range(4)])
print("per-warp S seen relative to warp 2:", [float(np.median(ps[4:40, w] - ps[4:40, 0])) for w in range(4)])
print("per-warp busy (arrive - S seen):", [float(np.median(pw[4:40, w] - ps[4:40, w])) for w in range(4)])
d = np.diff(t[1:200, 1])
d = d[d > 0]
print("QK-issue period percentiles 10/50/90/99:", [float(np.percentile(d, q)) for q in (10, 50, 90, 99)])
big = d > 2 * np.median(d)
print("blocks with > 2x median period:", int(big.sum()), "of", len(d), "; their excess:", float((d[big] - np.median(d)).sum()), "; total:", float(d.sum()))
print("per-warp period (S seen -> next S seen):", [float(np.median(np.diff(ps[4:40, w]))) for w in range(4)])
print("per-warp gap (arrive -> next S seen):", [float(np.median(ps[5:41, w] - pw[4:40, w])) for w in range(4)])
print("warp-5 S seen minus QK issue of same g:", float(np.median(ps[4:40, 3] - t[4:40, 1])))
print("warp-2 S seen minus QK issue of same g:", float(np.median(ps[4:40, 0] - t[4:40, 1])))
print("PV p_full seen minus warp-5 arrive:", float(np.median(t[4:40, 3] - pw[4:40, 3])))
# Item boundaries: blocks whose S-seen (warp 2) follows the previous one by > 2x the median.
sp = ps[:200, 0]
dd = np.diff(sp)
med = np.median(dd)
for gb in [i + 1 for i in range(len(dd)) if dd[i] > 2 * med][:4]:
    print(f"--- boundary before g={gb}")
    for gg in range(gb - 2, gb + 2):
        print(f"g={gg:3d} QKissue={t[gg,1]-base:8d} PVv={t[gg,2]-base:8d} PVp={t[gg,3]-base:8d} "
              f"inner(ld,max,h0,h1)={[int(x - base) for x in in4[gg]]} smx_done={t[gg,7]-base:8d} Sseen(w2..5)={[int(x - base) for x in ps[gg]]} arrive(w2..5)={[int(x - base) for x in pw[gg]]}")
print("epilogue stamps (rel. base): wait start, o_done seen, O read + o_free, stores done")
for qq in range(1, 5):
    print(qq, [int(x - base) for x in ep[qq]])
print("median epilogue: o_done wait", float(np.median(ep[1:20, 1] - ep[1:20, 0])), "read", float(np.median(ep[1:20, 2] - ep[1:20, 1])),
      "store", float(np.median(ep[1:20, 3] - ep[1:20, 2])))
