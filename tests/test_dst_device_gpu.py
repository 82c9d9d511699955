"""K8 on-device DST (fixed-base mode) against the host tuner: for random per-sequence K4-style
profiles grouped into micro-batches, the device decision (member merge + coverage test +
smallest safe budget) equals the host's make_micro_batch + tune_global_batch bit for bit
(k_final and coverage_drop), for every anchor and several thresholds."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _profiles(nb, nb_max, rng):
    P = np.zeros((len(nb), nb_max), np.float64)
    for s, n in enumerate(nb):
        v = np.sort(rng.gamma(rng.uniform(0.05, 2.0), size=n))[::-1]
        P[s, :n] = v / v.sum()
    return P


@pytest.mark.parametrize("anchor", ["min", "mean", "max"])
@pytest.mark.parametrize("p", [0.02, 0.1, 0.3])
def test_dst_decide_matches_host(anchor, p):
    from paper_2604_13847_b200 import dp, ops
    from paper_2604_13847_b200.host import DEFAULT_BUDGET_GRID, api

    h = api()
    B = 128
    rng = np.random.default_rng(hash((anchor, p)) % 2**32)
    table = h.synthesize_table(block_size=B)
    grid = np.asarray(DEFAULT_BUDGET_GRID, np.int32)
    cfg = dp.DstSettings(threshold_p=p, anchor=anchor, base_mode="fixed")
    for trial in range(6):
        n_mb = int(rng.integers(1, 6))
        members = [int(rng.integers(1, 5)) for _ in range(n_mb)]
        lengths = [int(rng.choice([700, 2048, 4096, 12288, 32768])) for _ in range(sum(members))]
        cu = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
        lay = ops.VarlenLayout.build(cu, B)
        nb = lay.nb_per_seq
        P = _profiles(nb, lay.nb_max, rng)
        mb_off = np.concatenate([[0], np.cumsum(members)]).astype(np.int32)
        xs = [int(sum(lengths[mb_off[i]:mb_off[i + 1]])) for i in range(n_mb)]
        k_base = [int(rng.choice(grid)) for _ in range(n_mb)]
        k_anchor, bottleneck, _ = dp.fixed_base_plan(table, xs, k_base, cfg)
        dev = lambda a, t: torch.as_tensor(np.asarray(a), dtype=t).cuda()  # noqa: E731
        kf, drop, kseq = ops.dst_decide(dev(P, torch.float64), lay, dev(mb_off, torch.int32), dev(k_base, torch.int32),
                                        dev(k_anchor, torch.int32), dev(bottleneck, torch.int32),
                                        dev(grid, torch.int32), p)
        merged = []
        for i in range(n_mb):
            sl = range(mb_off[i], mb_off[i + 1])
            _, mp = h.make_micro_batch([lengths[s] for s in sl], [[P[s, :nb[s]]] for s in sl])
            merged.append(mp[0])
        ref = h.tune_global_batch(table, xs, k_base, merged, layer=0, threshold_p=p, anchor=anchor, budget_grid=grid)
        assert [d.k_anchor for d in ref] == k_anchor.tolist()
        assert kf.cpu().tolist() == [d.k_final for d in ref], (trial, anchor, p)
        assert drop.cpu().tolist() == [d.coverage_drop for d in ref], (trial, anchor, p)
        ks = kseq.cpu().numpy()
        for i in range(n_mb):
            for s in range(mb_off[i], mb_off[i + 1]):
                assert ks[s] == min(ref[i].k_final, nb[s])


def test_dpstep_on_device_matches_host_path():
    """DPStep in fixed-base mode with this rank as the bottleneck of a 3-rank pool: the on-device
    DST path (no profile download, no exchange) picks the same per-layer keep counts as the host
    DST (decide_budgets) over the same GPU profiles."""
    from paper_2604_13847_b200 import dp, ops
    from paper_2604_13847_b200.host import api

    lens = [12288, 4096, 2048, 2048]
    X = int(sum(lens))
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    B, H, D, L = 128, 4, 128, 8
    lay = ops.VarlenLayout.build(cu, B)
    g = torch.Generator(device="cuda").manual_seed(3)
    q, k, v, do = (torch.randn((X, H, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
    scales = np.exp(np.random.default_rng(1).uniform(-0.5, 2.5, size=L))
    table = api().synthesize_table(block_size=B)
    others = [X // 3, X // 4]
    changed = False
    for p in (0.02, 0.1, 0.3):
        cfg = dp.DstSettings(base_mode="fixed", base_budget=32, anchor="mean", threshold_p=p)
        batch = dp.RankBatch(np.asarray(lens), list(range(len(lens))), lay)
        dev_step = dp.DPStep(batch, q, k, v, do, scales, table, cfg, pooled_xs=[X] + others)
        dev_step.run(backward=False)
        got = [int(t.item()) for t in dev_step.last["k_final_device"]]
        # host path over the same GPU profiles, the other ranks as single sequences
        host_step = dp.DPStep(batch, q, k, v, do, scales, table, cfg)
        _, profs = host_step.scorer_pass()
        own = [dp.profiles_to_host(profs[l], lay) for l in range(L)]
        pooled = [(np.asarray(lens), [[own[l][s] for l in range(L)] for s in range(len(lens))])]
        for x in others:
            nb = (x + B - 1) // B
            pooled.append((np.asarray([x]), [[np.full(nb, 1.0 / nb) for _ in range(L)]]))
        k_final, decisions, _, _ = dp.decide_budgets(pooled, table, cfg, L)
        assert got == k_final[0].tolist(), (p, got, k_final[0].tolist())
        changed = changed or any(d.micro_batch_id == 0 and d.k_final != d.k_base for d in decisions)
    assert changed  # the coverage test compressed this rank at least once: the comparison is not trivial


def test_dpstep_nvtx_ranges(monkeypatch):
    """SB_NVTX=1 (dp._NVTX): the host-DST step pushes / pops one NVTX range per layer phase and
    returns the same selections as without them."""
    from paper_2604_13847_b200 import dp, ops
    from paper_2604_13847_b200.host import api

    lens = [4096, 2048]
    X = int(sum(lens))
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    B, H, D, L = 128, 4, 128, 3
    lay = ops.VarlenLayout.build(cu, B)
    g = torch.Generator(device="cuda").manual_seed(5)
    q, k, v, do = (torch.randn((X, H, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
    scales = np.ones(L)
    batch = dp.RankBatch(np.asarray(lens), list(range(len(lens))), lay)
    step = dp.DPStep(batch, q, k, v, do, scales, api().synthesize_table(block_size=B), dp.DstSettings())
    plain = step.run(backward=True)
    pushes = []
    monkeypatch.setattr(dp, "_NVTX", True)
    monkeypatch.setattr(torch.cuda.nvtx, "range_push", lambda msg: pushes.append(msg))
    monkeypatch.setattr(torch.cuda.nvtx, "range_pop", lambda: None)
    traced = step.run(backward=True)
    torch.cuda.synchronize()
    assert len(pushes) == 2 * L and pushes[0].startswith("layer 0")
    for (i0, c0, *_), (i1, c1, *_) in zip(plain, traced):
        assert torch.equal(i0, i1) and torch.equal(c0, c1)
