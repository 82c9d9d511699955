"""Debug: per-stream timeline of CTA 0 of the two-stream forward kernel on C2 (not product)."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_13847_b200 import ops
import bench
lib = ops._lib()
lib.sb_debug_set_trace.argtypes = [ctypes.c_void_p]
if os.environ.get("C3K"):  # C3 rank micro-batch [2048 x3, 32768, 2048] at a fixed keep count
    lens = [2048, 2048, 2048, 32768, 2048]
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    k_seq = np.minimum(int(os.environ["C3K"]), (np.array(lens) + 127) // 128).astype(np.int32)
else:
    cu, k_seq = bench.workload(0)
T = int(cu[-1]); H, D, B = 32, 128, 128
lay = ops.VarlenLayout.build(cu, B)
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn((T, H, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
S = ops.block_scores(q, k, lay)
idx, cnt = ops.topk_select(S, lay, torch.from_numpy(k_seq).cuda(), int(k_seq.max()))
buf = torch.zeros(8192 + 2 * 256, dtype=torch.int64, device="cuda")
for it in range(3):
    lib.sb_debug_set_trace(ctypes.c_void_p(buf.data_ptr() if it == 2 else 0))
    ops.sparse_attn_fwd(q, k, v, lay, idx, cnt)
torch.cuda.synchronize()
t = buf.cpu().numpy().astype(np.int64)[:4096].reshape(2, 256, 8)
base = min(t[0, 0, 0], t[1, 0, 0])
names = ["QK issued", "PV issued", "S seen", "P arrive", "epi start", "epi end"]
for s in range(2):
    print(f"stream {s}")
    for gg in range(0, int(os.environ.get("ROWS", "40"))):
        print(f"  g={gg:3d} " + " ".join(f"{n}={int(t[s, gg, i] - base) if t[s, gg, i] else -1:8d}" for i, n in enumerate(names)))
    r = slice(2, 150)
    d = np.diff(t[s, :150, 2]); d = d[d > 0]
    print("  median period (S seen -> next):", np.median(d))
    print("  median softmax (S seen -> P arrive):", np.median((t[s, r, 3] - t[s, r, 2])))
    print("  median P arrive -> PV issued:", np.median(t[s, r, 1] - t[s, r, 3]))
    print("  median QK issued -> S seen:", np.median(t[s, r, 2] - t[s, r, 0]))
    nx = t[s, 3:151, 0] - t[s, 2:150, 1]
    print("  median PV issued -> next QK issued:", np.median(nx))
    print("  median PV issued -> next k_full seen:", np.median(t[s, 3:151, 6] - t[s, 2:150, 1]))
