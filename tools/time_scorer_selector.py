"""Achieved HBM GB/s of the scorer (K1 pool, K2 block scores) and selector (K3) on C2 and C5
(north-star measurement item). Each kernel timed alone with CUDA events on the launching stream,
median of 20 after warm-up; algorithmic bytes as in DESIGN.md section 3 (not product)."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2604_13847_b200 import ops


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def run(name, cu, Hq, Hkv, k_seq_np, D=128, B=128):
    lay = ops.VarlenLayout.build(cu, B)
    T = int(cu[-1]); group = Hq // Hkv
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn((T, Hq, D), generator=g, device="cuda").to(torch.bfloat16)
    k = torch.randn((T, Hkv, D), generator=g, device="cuda").to(torch.bfloat16)
    qbar, kbar = ops.block_pool(q, lay), ops.block_pool(k, lay)
    S = ops.block_scores(q, k, lay, qbar=qbar, kbar=kbar)
    k_seq = torch.from_numpy(np.asarray(k_seq_np, np.int32)).cuda()
    k_max = int(max(k_seq_np))
    t_pq = timeit(lambda: ops.block_pool(q, lay))
    t_pk = timeit(lambda: ops.block_pool(k, lay))
    t_s = timeit(lambda: ops.block_scores(q, k, lay, qbar=qbar, kbar=kbar))
    t_sel = timeit(lambda: ops.topk_select(S, lay, k_seq, k_max, group=group))
    NB, TRI, hsel = lay.nb_total, lay.tri_total, Hq // group
    b_pq = T * Hq * D * 2 + NB * Hq * D * 4
    b_pk = T * Hkv * D * 2 + NB * Hkv * D * 4
    b_s = NB * (Hq + Hkv) * D * 4 + Hq * TRI * 4
    b_sel = Hq * TRI * 4 + hsel * NB * (k_max + 1) * 4
    gbs = lambda b, t: round(b / (t * 1e-3) / 1e9, 1)  # noqa: E731
    r = dict(workload=name, pool_q_us=round(t_pq * 1e3, 1), pool_q_gbs=gbs(b_pq, t_pq), pool_k_us=round(t_pk * 1e3, 1),
             pool_k_gbs=gbs(b_pk, t_pk), scores_us=round(t_s * 1e3, 1), scores_gbs=gbs(b_s, t_s),
             select_us=round(t_sel * 1e3, 1), select_gbs=gbs(b_sel, t_sel), select_bytes=b_sel, k_max=k_max)
    print(json.dumps(r), flush=True)
    return r


if __name__ == "__main__":
    cu, k_seq = bench.workload(0)
    out = [run("C2 32K packed, 32/32 heads", np.asarray(cu), 32, 32, k_seq)]
    for hkv in (32, 8):
        out.append(run(f"C5 131072 single, 32/{hkv} heads, k=103", np.array([0, 131072]), 32, hkv, [103]))
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/scorer_selector_gbs.json", "w"), indent=1)
