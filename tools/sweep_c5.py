"""C5 roofline sweep (BASELINE.json configs[4]): one 131072-token sequence, keep ratio swept over
0.05-0.5, scorer + selector + fwd + bwd on one B200, each phase timed with CUDA events on the
launching stream (median of --reps after warm-up).

Useful FLOPs follow bench.useful_flops: 4*d*sum(e_ij) fwd and
10*d*sum(e_ij) bwd per q head; with GQA group selection (--kv-heads < --heads, one index set per
kv group, reference routing shared by the group) every q head of the group does the same work, so
the per-selection-head sum is multiplied by the group size. The fraction is against the measured
burst bf16 peak in MEASURED_PEAKS.json (bench.peaks()).

    python tools/sweep_c5.py --out gpurun_out/c5_sweep.json
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import bench
from paper_2604_13847_b200 import ops


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=131072)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--kv-heads", type=int, default=8)
    ap.add_argument("--head-dim", type=int, default=128)
    ap.add_argument("--block", type=int, default=128)
    ap.add_argument("--keeps", default="0.05,0.1,0.2,0.3,0.5")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()

    T, Hq, Hkv, D, B = a.tokens, a.heads, a.kv_heads, a.head_dim, a.block
    group = Hq // Hkv
    peak_tf, _, _, _, peak_kind = bench.peaks()  # burst bf16 peak
    cu = np.array([0, T], np.int64)
    lay = ops.VarlenLayout.build(cu, B)
    nb = int(lay.nb_max)
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn((T, Hq, D), generator=g, device="cuda").to(torch.bfloat16)
    k = torch.randn((T, Hkv, D), generator=g, device="cuda").to(torch.bfloat16)
    v = torch.randn((T, Hkv, D), generator=g, device="cuda").to(torch.bfloat16)
    do = torch.randn((T, Hq, D), generator=g, device="cuda").to(torch.bfloat16)

    rows = []
    for keep in [float(x) for x in a.keeps.split(",")]:
        kk = max(1, int(math.ceil(keep * nb)))
        k_seq = torch.full((1,), kk, dtype=torch.int32, device="cuda")
        S = ops.block_scores(q, k, lay)
        idx, cnt = ops.topk_select(S, lay, k_seq, kk, group=group)
        o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt)
        t_sc = timeit(lambda: ops.block_scores(q, k, lay), a.reps)
        t_sel = timeit(lambda: ops.topk_select(S, lay, k_seq, kk, group=group), a.reps)
        t_f = timeit(lambda: ops.sparse_attn_fwd(q, k, v, lay, idx, cnt), a.reps)
        t_b = timeit(lambda: ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt), a.reps)
        ff, fb = bench.useful_flops(cu, B, idx.cpu().numpy(), cnt.cpu().numpy(), D)
        ff, fb = ff * group, fb * group
        tf_f, tf_b = ff / (t_f * 1e-3) / 1e12, fb / (t_b * 1e-3) / 1e12
        step = t_sc + t_sel + t_f + t_b
        r = dict(keep=keep, k=kk, scorer_ms=round(t_sc, 4), select_ms=round(t_sel, 4), fwd_ms=round(t_f, 4),
                 bwd_ms=round(t_b, 4), step_ms=round(step, 4), fwd_tflops=round(tf_f, 1), bwd_tflops=round(tf_b, 1),
                 step_tflops=round((ff + fb) / (step * 1e-3) / 1e12, 1), fwd_frac=round(tf_f / peak_tf, 3),
                 bwd_frac=round(tf_b / peak_tf, 3))
        print(json.dumps(r), flush=True)
        rows.append(r)
        del S, idx, cnt, o, lse
    res = dict(workload=f"C5: 1 x {T} tokens, {Hq}q/{Hkv}kv heads{" (GQA group selection)" if group > 1 else ""}, d={D}, B={B}",
               peak_tflops=peak_tf, peak_kind=peak_kind, device=torch.cuda.get_device_name(), rows=rows)
    if a.out:
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
