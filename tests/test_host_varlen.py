"""Opt-in varlen-aware DST cost (not in the reference).

predict_members = sum over members of predict(L_s, min(k, ceil(L_s / B))) in member order;
plan_step with varlen_block_size > 0 prices micro-batches with it (anchor alignment included)
and otherwise makes the reference's decisions (dst.cpp:107-143), restated here in Python over
the same host primitives. Off (0) stays bit-identical to the reference (test_host_parity.py)."""
import math

import numpy as np
import pytest

from paper_2604_13847_b200.host import api


@pytest.fixture(scope="module")
def host():
    return api()


def _members_cost(h, table, lengths, k, B):
    total, ex = 0.0, False
    for L in lengths:
        ms, e = h.predict(table, int(L), int(min(k, max(1, math.ceil(L / B)))))
        total += ms
        ex = ex or e
    return total, ex


def test_predict_members_is_member_sum(host):
    table = host.synthesize_table(block_size=128)
    rng = np.random.default_rng(3)
    for _ in range(50):
        lengths = rng.choice([300, 2048, 5000, 32768, 70000], size=rng.integers(1, 7))
        k = int(rng.choice(table.budget_grid))
        got = host.predict_members(table, lengths, k, 128)
        assert got == _members_cost(host, table, lengths, k, 128)
    # one member == predict at the clamped budget
    assert host.predict_members(table, [2048], 64, 128)[0] == host.predict(table, 2048, 16)[0]


def _align_members(h, table, lengths, target, B):
    g = list(table.budget_grid)
    fit = [k for k in g if _members_cost(h, table, lengths, k, B)[0] <= target]
    return (max(fit), False) if fit else (g[0], True)


def test_plan_step_varlen_decisions(host):
    """Global-scope SAB+DST on the C3 mix with the varlen cost: every decision equals the
    reference rule evaluated with predict_members / its alignment."""
    B, L, gbs, mbs, dp = 128, 4, 20, 5, 4
    dist = dict(short_weight=0.6, short_log_mean=float(np.log(2048)), short_log_sigma=0.0,
                long_log_mean=float(np.log(32768)), long_log_sigma=0.0)
    lengths, profs = host.generate_samples(gbs, L, B, seed=11, dist=dist)
    table = host.synthesize_table(block_size=B)
    grid = list(table.budget_grid)
    est = host.make_estimator(host.default_bin_edges(65536))
    sp = host.plan_step("sab_dst", np.arange(gbs), lengths, profs, gbs=gbs, mbs=mbs, dp=dp, num_layers=L,
                        table=table, est=est, anchor="mean", threshold_p=0.1, dst_scope="global",
                        base_mode="coverage", varlen_block_size=B)
    pooled = [ids for r in sp["micro_batch_bins"] for ids in r]  # rank-major (sim.cpp:357-369)
    mbl = [[int(lengths[i]) for i in ids] for ids in pooled]
    merged = [host.make_micro_batch(m, [profs[i] for i in ids])[1] for m, ids in zip(mbl, pooled)]
    k_base = [host.intrinsic_budget(mg, np.asarray(grid, np.int32), 0.9) for mg in merged]
    for l in range(L):
        base_ms = [_members_cost(host, table, m, kb, B)[0] for m, kb in zip(mbl, k_base)]
        anchor = sum(base_ms) / len(base_ms)
        for i, d in enumerate([d for d in sp["decisions"] if d.layer_id == l]):
            assert d.micro_batch_id == i and d.k_base == k_base[i]
            prof = merged[i][l]
            k_anchor = _align_members(host, table, mbl[i], anchor, B)[0]
            assert d.k_anchor == k_anchor
            cov = lambda k: host.coverage(prof, k)  # noqa: E731
            if base_ms[i] <= anchor or cov(k_base[i]) - cov(k_anchor) <= 0.1:
                k_final = k_anchor
            else:
                safe = [k for k in grid if cov(k_base[i]) - cov(k) <= 0.1]
                k_final = min(safe) if safe else grid[-1]
            assert d.k_final == k_final, (l, i)
            assert d.predicted_ms_final == _members_cost(host, table, mbl[i], k_final, B)[0]


def test_varlen_off_matches_reference(host, ref):
    table = host.synthesize_table(block_size=128)
    lengths, profs = host.generate_samples(8, 3, 128, seed=5)
    kw = dict(gbs=8, mbs=2, dp=2, num_layers=3, table=table, anchor="mean", threshold_p=0.1)
    a = host.plan_step("sab_dst", np.arange(8), lengths, profs, est=host.make_estimator(host.default_bin_edges(65536)),
                       varlen_block_size=0, **kw)
    b = ref.plan_step("sab_dst", np.arange(8), lengths, profs, est=ref.make_estimator(ref.default_bin_edges(65536)),
                      **kw)
    assert a["decisions"] == b["decisions"]
    with pytest.raises(Exception):
        ref.plan_step("sab_dst", np.arange(8), lengths, profs, est=ref.make_estimator(ref.default_bin_edges(65536)),
                      varlen_block_size=128, **kw)
