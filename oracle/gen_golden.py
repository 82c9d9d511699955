"""Generate tests/golden/* from the compiled, unmodified reference (oracle/_ref/libsbref.so).

Run here (needs /root/reference to have built the oracle): python oracle/gen_golden.py
The fixtures are committed so the parity tests also run on the GPU box.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def routing_scores(r):
    """Reference routing-score vectors before and after the reference's sort, and the
    reference coverage() on the sorted profile at the default budget grid."""
    rows = {}
    n = 0
    grid = [1, 2, 3, 4, 6, 8, 10, 12, 16, 20, 24, 32, 40, 48, 56, 64, 100, 200]
    for seed, kind, bsz in ((42, "bimodal", 256), (7, "bimodal", 64), (3, "long_tail", 128)):
        L_s, P_s = r.generate_samples(6, 3, bsz, seed=seed, kind=kind, sorted=True)
        L_u, P_u = r.generate_samples(6, 3, bsz, seed=seed, kind=kind, sorted=False)
        for s in range(6):
            for l in range(3):
                pre, srt = P_u[s][l], P_s[s][l]
                assert np.array_equal(np.sort(pre)[::-1], srt)
                if len(pre) < 4 or len(pre) > 4096:
                    continue
                ks = np.array([k for k in grid if k <= len(pre) + 2], np.int32)
                rows[f"row{n}"] = pre
                rows[f"sorted{n}"] = srt
                rows[f"ks{n}"] = ks
                rows[f"cov{n}"] = np.array([r.coverage(srt, int(k)) for k in ks])
                n += 1
    np.savez_compressed(os.path.join(OUT, "routing_scores.npz"), n=n, **rows)
    return n


def host_decisions(r):
    doc = {}
    t = r.synthesize_table(noise_sigma=0.3, seed=5, block_size=128)
    doc["table"] = dict(length_bins=t.length_bins.tolist(), budget_grid=t.budget_grid.tolist(),
                        latency_ms=t.latency_ms.ravel().tolist())
    rng = np.random.default_rng(99)
    q = []
    for _ in range(300):
        x, k = int(rng.integers(1, 300000)), int(rng.integers(0, 80))
        target = float(rng.uniform(0, t.latency_ms.max()))
        ms, ex = r.predict(t, x, k)
        b, inf = r.align(t, x, target)
        q.append([x, k, target, ms.hex(), ex, b, inf])
    doc["predict_align"] = q
    # plan_step runs (C3-like shape and the reference defaults), 3 iterations each.
    runs = []
    dist = dict(short_weight=0.6, short_log_mean=float(np.log(2048)), short_log_sigma=0.0,
                long_log_mean=float(np.log(32768)), long_log_sigma=0.0)
    for name, gbs, mbs, dp, nl, strat, anchor, scope, mode, d in (
            ("c3_sab_dst_mean", 40, 5, 8, 12, "sab_dst", "mean", "global", "coverage", dist),
            ("default_sab_dst_min", 16, 2, 2, 9, "sab_dst", "min", "global", "coverage", None),
            ("default_lbb_dst_rank", 16, 2, 2, 9, "lbb_dst", "max", "rank", "fixed", None),
            ("default_dst_mean", 16, 2, 2, 9, "dst", "mean", "global", "coverage", None)):
        est = r.make_estimator(r.default_bin_edges(65536))
        its = []
        for it in range(3):
            L, P = r.generate_samples(gbs, nl, 128, seed=500 + it, dist=d)
            res = r.plan_step(strat, np.arange(gbs), L, P, gbs=gbs, mbs=mbs, dp=dp, num_layers=nl, table=t, est=est,
                              iter_index=it, anchor=anchor, dst_scope=scope, base_mode=mode, threshold_p=0.1)
            its.append(dict(seed=500 + it, budgets=res["budgets"].tolist(), bins=res["micro_batch_bins"],
                            decisions=[[d_.micro_batch_id, d_.layer_id, d_.k_base, d_.k_anchor, d_.k_final,
                                        d_.direction, d_.coverage_drop.hex(), d_.predicted_ms_base.hex(),
                                        d_.predicted_ms_final.hex()] for d_ in res["decisions"]],
                            ema=[v.hex() for v in est.ema_budget]))
        runs.append(dict(name=name, gbs=gbs, mbs=mbs, dp=dp, num_layers=nl, strategy=strat, anchor=anchor,
                         scope=scope, base_mode=mode, dist=d, iterations=its))
    doc["plan_step"] = runs
    with open(os.path.join(OUT, "host_decisions.json"), "w") as f:
        json.dump(doc, f)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    r = ref.api()
    print("routing rows:", routing_scores(r))
    host_decisions(r)
    print("wrote", OUT)
