"""Bit-exact parity of the host decision layer against the compiled, unmodified reference
(oracle/_ref/libsbref.so built from /root/reference/proj/core/src by oracle/Makefile).

Every comparison is exact (==), including doubles: the decisions compare doubles with <=,
so any reordering of a sum would eventually flip a k_final. CPU only. Skipped where the
reference library is unavailable (the GPU box); tests/test_host_golden.py covers the same
surface from committed fixtures there.
"""
import json
import re

import numpy as np
import pytest

from paper_2604_13847_b200.host import DEFAULT_BUDGET_GRID, ProfileTable

RNG = np.random.default_rng(20260418)


def rand_profile(rng, m):
    a = rng.gamma(rng.uniform(0.05, 2.0), size=m)
    a = a / a.sum()
    return np.sort(a)[::-1].copy()


def rand_table(api, rng, noisy):
    grid = np.unique(rng.integers(1, 200, size=rng.integers(2, 20)))
    if len(grid) < 2:
        grid = np.array([1, 2])
    bins = np.unique(rng.integers(64, 300000, size=rng.integers(2, 16)))
    if len(bins) < 2:
        bins = np.array([256, 512])
    return api.synthesize_table(bins, grid, noise_sigma=0.4 if noisy else 0.0, block_size=int(rng.integers(32, 300)),
                                seed=int(rng.integers(1 << 30)))


def test_predict_align_parity(host, ref):
    rng = np.random.default_rng(1)
    for ti in range(40):
        t = rand_table(host, rng, noisy=ti % 2 == 0)
        tr = rand_table(ref, np.random.default_rng(1 + 0), noisy=False)  # exercise ref synthesize too
        del tr
        xs = rng.integers(1, 400000, size=200)
        ks = rng.integers(0, 260, size=200)
        for x, k in zip(xs, ks):
            assert host.predict(t, int(x), int(k)) == ref.predict(t, int(x), int(k))
        for x in xs[:100]:
            target = float(rng.uniform(0.0, t.latency_ms.max() * 1.2))
            assert host.align(t, int(x), target) == ref.align(t, int(x), target)


def test_synthesize_table_parity(host, ref):
    rng = np.random.default_rng(2)
    for _ in range(20):
        bins = np.unique(rng.integers(64, 300000, size=10))
        grid = np.unique(rng.integers(1, 100, size=8))
        kw = dict(c_lin=float(rng.uniform(0, 1e-5)), c_attn=float(rng.uniform(0, 1e-7)), c_fixed=float(rng.uniform(0.01, 1)),
                  noise_sigma=float(rng.choice([0.0, 0.2])), block_size=int(rng.integers(16, 512)), seed=int(rng.integers(1 << 40)))
        a = host.synthesize_table(bins, grid, **kw)
        b = ref.synthesize_table(bins, grid, **kw)
        assert np.array_equal(a.latency_ms, b.latency_ms)


def test_table_io_parity(host, ref, tmp_path):
    t = host.synthesize_table(noise_sigma=0.5, seed=11)
    p1, p2 = str(tmp_path / "a.csv"), str(tmp_path / "b.csv")
    host.save_table(t, p1)
    ref.save_table(t, p2)
    assert open(p1).read() == open(p2).read()
    (a, ra), (b, rb) = host.load_table(p1), ref.load_table(p1)
    assert ra == rb and np.array_equal(a.latency_ms, b.latency_ms)


def test_coverage_and_budgets_parity(host, ref):
    rng = np.random.default_rng(3)
    for _ in range(300):
        p = rand_profile(rng, int(rng.integers(1, 300)))
        for k in rng.integers(-1, 320, size=8):
            assert host.coverage(p, int(k)) == ref.coverage(p, int(k))
        tgt = float(rng.uniform(0, 1))
        assert host.coverage_budget(p, tgt) == ref.coverage_budget(p, tgt)
    for _ in range(100):
        profs = [rand_profile(rng, int(rng.integers(1, 100))) for _ in range(int(rng.integers(1, 12)))]
        grid = np.unique(rng.integers(1, 80, size=6))
        tgt = float(rng.uniform(0.3, 1.0))
        assert host.intrinsic_budget(profs, grid, tgt) == ref.intrinsic_budget(profs, grid, tgt)


def brute_force_k_final(t_api, table, x, k_base, lat_list, prof, p, anchor, grid):
    """Eqs. 6-7 with the empty-F extension, evaluated exhaustively."""
    arr = np.array(lat_list)
    t_anchor = {"min": arr.min(), "max": arr.max(), "mean": sum(lat_list) / len(lat_list)}[anchor]
    if anchor == "mean":
        s = 0.0
        for v in lat_list:
            s += v
        t_anchor = s / len(lat_list)
    cov = lambda k: t_api.coverage(prof, k)
    feasible_lat = [k for k in table.budget_grid if t_api.predict(table, x, int(k))[0] <= t_anchor]
    k_anchor = int(max(feasible_lat)) if feasible_lat else int(table.budget_grid[0])
    base_ms = t_api.predict(table, x, k_base)[0]
    if base_ms <= t_anchor:
        return k_anchor
    if cov(k_base) - cov(k_anchor) <= p:
        return k_anchor
    safe = [int(k) for k in grid if cov(k_base) - cov(int(k)) <= p]
    return min(safe) if safe else int(grid[-1])


def test_tune_global_batch_parity_and_bruteforce(host, ref):
    """Acceptance criterion 1: >= 10^4 seeded decisions, exact."""
    rng = np.random.default_rng(4)
    n_dec = 0
    while n_dec < 10000:
        grid = np.unique(rng.integers(1, 130, size=rng.integers(2, 64)))
        if len(grid) < 2:
            continue
        bins = np.unique(rng.integers(256, 200000, size=rng.integers(2, 10)))
        if len(bins) < 2:
            continue
        t = host.synthesize_table(bins, grid, noise_sigma=0.0, block_size=int(rng.integers(32, 300)), seed=int(rng.integers(1 << 30)))
        n = int(rng.integers(1, 24))
        xs = rng.integers(128, 250000, size=n)
        kb = rng.choice(grid, size=n)
        profs = [rand_profile(rng, int(rng.integers(1, 200))) for _ in range(n)]
        p = float(rng.choice([0.0, 0.05, 0.1, 0.2, 0.3, 1.0, rng.uniform(0, 1)]))
        anchor = ["min", "mean", "max"][int(rng.integers(3))]
        a = host.tune_global_batch(t, xs, kb, profs, threshold_p=p, anchor=anchor, budget_grid=grid)
        b = ref.tune_global_batch(t, xs, kb, profs, threshold_p=p, anchor=anchor, budget_grid=grid)
        assert a == b
        if n_dec < 2000:  # brute force on a subset (it is slow in Python)
            lat = [host.predict(t, int(x), int(k))[0] for x, k in zip(xs, kb)]
            for i, d in enumerate(a):
                assert d.k_final == brute_force_k_final(host, t, int(xs[i]), int(kb[i]), lat, profs[i], p, anchor, grid)
                if d.k_base in set(grid.tolist()):
                    assert d.coverage_drop <= p + 1e-12
        n_dec += n


def test_make_micro_batch_parity(host, ref):
    rng = np.random.default_rng(5)
    for _ in range(200):
        ns, nl = int(rng.integers(1, 9)), int(rng.integers(1, 5))
        lengths = rng.integers(1, 70000, size=ns)
        profs = [[rand_profile(rng, int(rng.integers(1, 300))) for _ in range(nl)] for _ in range(ns)]
        la, ma = host.make_micro_batch(lengths, profs)
        lb, mb = ref.make_micro_batch(lengths, profs)
        assert la == lb
        assert all(np.array_equal(x, y) for x, y in zip(ma, mb))


@pytest.mark.parametrize("kind", ["bimodal", "long_tail", "fixed"])
def test_generate_samples_parity(host, ref, kind):
    for seed in (0, 42, 123456789):
        for sorted_ in (True, False):
            la, pa = host.generate_samples(16, 6, 128, seed=seed, kind=kind, sorted=sorted_)
            lb, pb = ref.generate_samples(16, 6, 128, seed=seed, kind=kind, sorted=sorted_)
            assert np.array_equal(la, lb)
            assert all(np.array_equal(x, y) for s, r in zip(pa, pb) for x, y in zip(s, r))
    # The unsorted vectors ARE the reference's scores before its sort (workload.cpp:58).
    ls, ps = ref.generate_samples(16, 6, 128, seed=42, kind=kind, sorted=True)
    lu, pu = ref.generate_samples(16, 6, 128, seed=42, kind=kind, sorted=False)
    for s, u in zip(ps, pu):
        for x, y in zip(s, u):
            assert np.array_equal(x, np.sort(y)[::-1])


def test_estimator_parity(host, ref):
    rng = np.random.default_rng(6)
    for _ in range(100):
        edges = host.default_bin_edges(int(rng.integers(1024, 300000)))
        assert np.array_equal(edges, ref.default_bin_edges(int(edges[-1]) - 1))
        grid = np.unique(rng.integers(1, 100, size=8))
        ea = host.make_estimator(edges, grid, ema_alpha=float(rng.uniform(0.01, 1.0)), default_budget=float(grid[0]))
        eb = host.make_estimator(edges, grid, ema_alpha=ea.ema_alpha, default_budget=float(grid[0]))
        n = int(rng.integers(0, 40))
        ks = rng.integers(1, 120, size=n)
        ls = rng.integers(1, 400000, size=n)
        host.calibrate(ea, ks, ls)
        ref.calibrate(eb, ks, ls)
        assert np.array_equal(ea.ema_budget, eb.ema_budget)
        for L in rng.integers(1, 400000, size=20):
            assert host.estimate_sparsity(ea, int(L)) == ref.estimate_sparsity(eb, int(L))


def test_bin_packing_parity(host, ref):
    rng = np.random.default_rng(7)
    for _ in range(500):
        n = int(rng.integers(1, 40))
        nb = int(rng.integers(1, n + 1))
        cap = int(rng.choice([0, -(-n // nb), -(-n // nb) + 1]))
        w = rng.choice([rng.uniform(0, 10, size=n), rng.integers(0, 5, size=n).astype(float)])
        assert host.bin_packing(w, nb, cap) == ref.bin_packing(w, nb, cap)


def test_plan_batching_parity(host, ref):
    rng = np.random.default_rng(8)
    table = host.synthesize_table(block_size=128)
    for _ in range(100):
        dp, mbs = int(rng.integers(1, 9)), int(rng.integers(1, 6))
        gbs = dp * mbs * int(rng.integers(1, 5))
        ids = rng.permutation(1000)[:gbs]
        lengths = rng.integers(64, 65536, size=gbs)
        est = host.make_estimator(host.default_bin_edges(65536))
        est.ema_budget[:] = rng.uniform(1, 64, size=len(est.ema_budget))
        for strat in ("sab", "lbb", "sequential"):
            a = host.plan_batching(strat, ids, lengths, gbs, mbs, dp, est, table)
            b = ref.plan_batching(strat, ids, lengths, gbs, mbs, dp, est, table)
            assert a[0] == b[0] and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("strategy", ["baseline", "dst", "sab", "lbb", "sab_dst", "lbb_dst"])
@pytest.mark.parametrize("scope,base_mode,anchor", [("global", "coverage", "mean"), ("rank", "fixed", "min"),
                                                   ("global", "fixed", "max"), ("rank", "coverage", "min")])
def test_plan_step_parity_over_iterations(host, ref, strategy, scope, base_mode, anchor):
    """The decision half of the reference step driver, iterated so estimator state evolves
    exactly like run_scenarios (sim.cpp:548-561)."""
    table = host.synthesize_table(block_size=128)
    gbs, mbs, dp, nl = 16, 2, 2, 6
    est_a = host.make_estimator(host.default_bin_edges(65536))
    est_b = host.make_estimator(host.default_bin_edges(65536))
    for it in range(4):
        lengths, profs = host.generate_samples(gbs, nl, 128, seed=1000 + it)
        ids = np.arange(gbs)
        kw = dict(gbs=gbs, mbs=mbs, dp=dp, num_layers=nl, table=table, iter_index=it, dst_scope=scope,
                  base_mode=base_mode, anchor=anchor, threshold_p=0.1)
        a = host.plan_step(strategy, ids, lengths, profs, est=est_a, **kw)
        b = ref.plan_step(strategy, ids, lengths, profs, est=est_b, **kw)
        assert a["micro_batch_bins"] == b["micro_batch_bins"]
        assert a["decisions"] == b["decisions"]
        assert np.array_equal(a["budgets"], b["budgets"])
        assert a["mean_cov_drop"] == b["mean_cov_drop"] and a["avg_budget"] == b["avg_budget"]
        assert np.array_equal(est_a.ema_budget, est_b.ema_budget)


def test_plan_step_config3_shape(host, ref):
    """dp=8, 40% 32K / 60% 2K, gbs=40, mbs=5, Mean p=0.1, global scope,
    coverage base mode, B=128 -- decisions identical to the reference, with a dense 1..256 grid too."""
    dist = dict(short_weight=0.6, short_log_mean=float(np.log(2048)), short_log_sigma=0.0,
                long_log_mean=float(np.log(32768)), long_log_sigma=0.0)
    lengths, profs = host.generate_samples(40, 36, 128, seed=42, dist=dist)
    assert set(lengths.tolist()) <= {2048, 32768}
    for grid in (DEFAULT_BUDGET_GRID, list(range(1, 257))):
        table = host.synthesize_table(budget_grid=grid, block_size=128)
        est_a = host.make_estimator(host.default_bin_edges(65536), budget_grid=grid)
        est_b = host.make_estimator(host.default_bin_edges(65536), budget_grid=grid)
        kw = dict(gbs=40, mbs=5, dp=8, num_layers=36, table=table, anchor="mean", threshold_p=0.1,
                  dst_scope="global", base_mode="coverage")
        a = host.plan_step("sab_dst", np.arange(40), lengths, profs, est=est_a, **kw)
        b = ref.plan_step("sab_dst", np.arange(40), lengths, profs, est=est_b, **kw)
        assert a["decisions"] == b["decisions"] and np.array_equal(a["budgets"], b["budgets"])


@pytest.mark.parametrize("strategy", ["baseline", "dst", "sab_dst", "lbb_dst"])
def test_plan_step_replay_files_byte_identical(host, ref, strategy, tmp_path):
    """The step's replay files -- decisions CSV (dst.cpp:171-185) and plan JSON
    (sab.cpp:312-336) -- written by this build and by the reference's own writers are
    byte-identical, over iterations (estimator state evolving)."""
    table = host.synthesize_table(block_size=128)
    gbs, mbs, dp, nl = 16, 2, 2, 4
    est_a = host.make_estimator(host.default_bin_edges(65536))
    est_b = host.make_estimator(host.default_bin_edges(65536))
    for it in range(3):
        lengths, profs = host.generate_samples(gbs, nl, 128, seed=2000 + it)
        kw = dict(gbs=gbs, mbs=mbs, dp=dp, num_layers=nl, table=table, iter_index=it, anchor="mean",
                  threshold_p=0.1)
        pa = {k: tmp_path / f"a_{it}.{k}" for k in ("csv", "json")}
        pb = {k: tmp_path / f"b_{it}.{k}" for k in ("csv", "json")}
        host.plan_step(strategy, np.arange(gbs), lengths, profs, est=est_a, decisions_csv=pa["csv"],
                       plan_json=pa["json"], **kw)
        ref.plan_step(strategy, np.arange(gbs), lengths, profs, est=est_b, decisions_csv=pb["csv"],
                      plan_json=pb["json"], **kw)
        assert pa["csv"].read_bytes() == pb["csv"].read_bytes(), (strategy, it)
        assert pa["csv"].read_text().startswith("iter,mb,layer,k_base,k_anchor,k_final,cov_drop,dir,")
        # Plan JSON: identical documents. Byte layout: this build writes upstream nlohmann 3.11.3's
        # dump(2) (every array expanded); the oracle build's header is cudnn-frontend's copy, whose
        # "Custom from FE" patch (json.hpp:20610) prints integer arrays on one line -- so compare
        # bytes after collapsing integer arrays.
        ta, tb = pa["json"].read_text(), pb["json"].read_text()
        assert json.loads(ta) == json.loads(tb)
        collapse = re.compile(r"\[\s*(-?\d+(?:,\s*-?\d+)*)\s*\]")
        assert collapse.sub(lambda m: "[" + ",".join(x.strip() for x in m.group(1).split(",")) + "]", ta) == tb
