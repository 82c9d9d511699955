"""PP projection: the 1F1B model fed with cost-table stage times
reproduces the reference's simulate_iteration timing bit for bit (iteration time, bubble,
critical-path bound, per-micro-batch max / mean, imbalance, average budget) for DP x PP
clusters, every strategy; plus hand-checkable schedules."""
import numpy as np
import pytest

from paper_2604_13847_b200 import pp_projection as ppj


def test_single_stage_is_serial():
    r = ppj.pipeline_1f1b([[1.0], [2.0]], [[3.0], [4.0]], 0.5)
    assert r["completion_ms"] == 10.0 and r["bubble_ms"] == 0.0


def test_two_stage_hand_schedule():
    # m = 2, pp = 2, unit forwards, backward 2, comm 0: stage 0 = F0 F1 B0 B1, stage 1 = F0 B0 F1 B1
    r = ppj.pipeline_1f1b([[1.0, 1.0], [1.0, 1.0]], [[2.0, 2.0], [2.0, 2.0]], 0.0)
    # stage1: F0 [1,2] B0 [2,4] F1 [4,5] B1 [5,7]; stage0: F0 [0,1] F1 [1,2] B0 [4,6] B1 [7,9]
    assert r["completion_ms"] == 9.0
    assert r["bubble_ms"] == 2 * 9.0 - 12.0
    assert ppj.critical_lower_bound([[1.0, 1.0], [1.0, 1.0]], [[2.0, 2.0], [2.0, 2.0]], 0.0) <= 9.0


@pytest.mark.parametrize("strategy", ["baseline", "dst", "sab", "sab_dst"])
@pytest.mark.parametrize("dp,pp,lps,gbs,mbs", [(2, 4, 2, 16, 2), (1, 2, 3, 8, 2), (2, 3, 2, 12, 1)])
def test_projection_matches_reference_simulate_iteration(host, ref, strategy, dp, pp, lps, gbs, mbs):
    table = host.synthesize_table(block_size=128)
    L = pp * lps
    cl = ppj.Cluster(pp=pp, layers_per_stage=lps, fwd_bwd_ratio=2.0, comm_ms=0.05, dp_sync_ms=5.0)
    lengths, profs = host.generate_samples(gbs, L, 128, seed=77 + gbs)
    kw = dict(gbs=gbs, mbs=mbs, dp=dp, table=table, iter_index=0, anchor="mean", threshold_p=0.1,
              base_mode="coverage")
    est_a = host.make_estimator(host.default_bin_edges(65536))
    est_b = ref.make_estimator(ref.default_bin_edges(65536))
    sp = host.plan_step(strategy, np.arange(gbs), lengths, profs, num_layers=L, est=est_a, **kw)
    want = ref.ref_simulate_iteration(strategy, np.arange(gbs), lengths, profs, pp=pp, layers_per_stage=lps,
                                      est=est_b, fwd_bwd_ratio=cl.fwd_bwd_ratio, comm_ms=cl.comm_ms,
                                      dp_sync_ms=cl.dp_sync_ms, **kw)
    rank_times, rank_budgets = [], []
    for r in range(dp):
        times, buds = [], []
        for i, ids in enumerate(sp["micro_batch_bins"][r]):
            x = int(sum(int(lengths[j]) for j in ids))
            b = [int(k) for k in sp["budgets"][r][i]]
            times.append(ppj.stage_times_from_table(host, table, x, b, cl))
            buds.append(b)
        rank_times.append(times)
        rank_budgets.append(buds)
    got = ppj.project_iteration(rank_times, rank_budgets, cl, L)
    for key in ("iter_ms", "bubble_ms", "critical_lb_ms", "max_mb_ms", "mean_mb_ms", "imbalance", "avg_budget"):
        assert got[key] == want[key], (key, got[key], want[key])
