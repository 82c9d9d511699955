"""Multi-rank host logic of the DP step driver on CPU (gloo, world_size 2): the per-rank
workload-estimate all-gather and the pooled host DST give bit-identical budgets on every rank,
equal to the single-process pooled computation and to the compiled reference's
tune_global_batch on the same pooled micro-batches (sim.cpp:357-369 pooling order)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_13847_b200 import dp
from paper_2604_13847_b200.host import api

L, B, MAXM = 3, 128, 4


def rank_workload(rank):
    h = api()
    dist_spec = dict(short_weight=0.6, short_log_mean=float(np.log(2048)), short_log_sigma=0.0,
                     long_log_mean=float(np.log(32768)), long_log_sigma=0.0)
    lengths, profs = h.generate_samples(3, L, B, seed=100 + rank, dist=dist_spec)
    layer_profiles = [[profs[s][l] for s in range(len(lengths))] for l in range(L)]
    return lengths, layer_profiles


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lengths, layer_profiles = rank_workload(rank)
    cfg = dp.DstSettings()
    est = dp.rank_estimate(lengths, layer_profiles, cfg)
    pooled = dp.exchange_estimates(est, L, len(cfg.budget_grid), world=world, max_members=MAXM)
    assert [int(x) for x in pooled[rank].members] == [int(x) for x in lengths]
    table = api().synthesize_table(block_size=B)
    k_final, decisions, k_base, xs = dp.decide_budgets_cov(pooled, table, cfg, L)
    out[rank] = (k_final.tolist(), [(d.micro_batch_id, d.layer_id, d.k_final, d.coverage_drop) for d in decisions],
                 k_base.tolist())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_exchange_and_dst_identical():
    world = 2
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.start_processes(_worker, args=(world, port, out), nprocs=world, start_method="spawn", join=True)
    assert out[0] == out[1]
    # Single-process pooled computation (rank-major) gives the same decisions.
    pooled = []
    for r in range(world):
        lengths, layer_profiles = rank_workload(r)
        prof = [[layer_profiles[l][s] for l in range(L)] for s in range(len(lengths))]
        pooled.append((np.asarray(lengths), prof))
    table = api().synthesize_table(block_size=B)
    k_final, decisions, k_base, _ = dp.decide_budgets(pooled, table, dp.DstSettings(), L)
    assert out[0][0] == k_final.tolist()
    assert out[0][1] == [(d.micro_batch_id, d.layer_id, d.k_final, d.coverage_drop) for d in decisions]


def test_pooled_dst_matches_reference(ref):
    """The pooled decisions equal the compiled reference's make_micro_batch + intrinsic_budget +
    tune_global_batch on the same micro-batches."""
    h = api()
    pooled = []
    for r in range(3):
        lengths, layer_profiles = rank_workload(r)
        prof = [[layer_profiles[l][s] for l in range(L)] for s in range(len(lengths))]
        pooled.append((np.asarray(lengths), prof))
    table = h.synthesize_table(block_size=B)
    cfg = dp.DstSettings()
    k_final, decisions, k_base, xs = dp.decide_budgets(pooled, table, cfg, L)
    grid = np.asarray(cfg.budget_grid, np.int32)
    rx, rm, rk = [], [], []
    for lengths, prof in pooled:
        ld, mp_ = ref.make_micro_batch(lengths, prof)
        rx.append(ld)
        rm.append(mp_)
        rk.append(ref.intrinsic_budget(mp_, grid, cfg.coverage_target))
    assert rk == k_base.tolist() and rx == xs.tolist()
    for l in range(L):
        rd = ref.tune_global_batch(table, rx, rk, [m[l] for m in rm], layer=l, threshold_p=cfg.threshold_p,
                                   anchor=cfg.anchor, budget_grid=grid)
        assert rd == [d for d in decisions if d.layer_id == l]


def test_pack_unpack_roundtrip():
    """The exchanged estimate round-trips exactly, its size depends only on (L, |K|, max_members),
    and an over-long member list is rejected instead of spilling into the next field."""
    lengths, layer_profiles = rank_workload(0)
    cfg = dp.DstSettings()
    est = dp.rank_estimate(lengths, layer_profiles, cfg)
    G = len(cfg.budget_grid)
    vec = dp.pack_estimate(est, L, G, MAXM).numpy()
    assert vec.size == 3 + MAXM + L * (G + 1)
    got = dp.unpack_estimate(vec, L, G, MAXM)
    assert got.x == est.x and got.k_base == est.k_base
    assert np.array_equal(got.members, lengths) and np.array_equal(got.cov, est.cov)
    with pytest.raises(ValueError):
        dp.pack_estimate(est, L, G, 1)
    with pytest.raises(ValueError):
        dp.pack_estimate(est, L + 1, G, MAXM)


@pytest.mark.parametrize("anchor", ["min", "mean", "max"])
@pytest.mark.parametrize("base_mode", ["coverage", "fixed"])
def test_cov_exchange_decisions_equal_profile_decisions(anchor, base_mode):
    """Deciding from the exchanged {x, k_base, C(K)} tables gives exactly the decisions of the
    pooled PROFILES (decide_budgets -> tune_global_batch), fixed base off the grid included, on
    the default and the dense 1..256 grids."""
    table = api().synthesize_table(block_size=B)
    for grid in (None, list(range(1, 257))):
        cfg = dp.DstSettings(anchor=anchor, base_mode=base_mode, base_budget=37)
        if grid is not None:
            cfg.budget_grid = grid
        ests, pooled = [], []
        for r in range(4):
            lengths, layer_profiles = rank_workload(r)
            ests.append(dp.rank_estimate(lengths, layer_profiles, cfg))
            pooled.append((np.asarray(lengths), [[layer_profiles[l][s] for l in range(L)] for s in range(len(lengths))]))
        a = dp.decide_budgets(pooled, table, cfg, L)
        b = dp.decide_budgets_cov(ests, table, cfg, L)
        assert a[0].tolist() == b[0].tolist() and a[1] == b[1]
        assert a[2].tolist() == b[2].tolist() and a[3].tolist() == b[3].tolist()
