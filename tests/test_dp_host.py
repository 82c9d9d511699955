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

L, B = 3, 128


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
    pooled = dp.exchange_estimates(lengths, layer_profiles, width=256, block=B, world=world)
    table = api().synthesize_table(block_size=B)
    k_final, decisions, k_base, xs = dp.decide_budgets(pooled, table, dp.DstSettings(), L)
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
    lengths, layer_profiles = rank_workload(0)
    vec = dp.pack_estimate(np.asarray(lengths), layer_profiles, 256).numpy()
    got_len, got_prof = dp.unpack_estimate(vec, L, 256, B)
    assert np.array_equal(got_len, lengths)
    for s in range(len(lengths)):
        for l in range(L):
            assert np.array_equal(got_prof[s][l], layer_profiles[l][s])
