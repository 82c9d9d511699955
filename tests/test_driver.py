"""Measured DP step driver (paper_2604_13847_b200/driver.py): the reference's seed stream and
iterations-CSV format on CPU; a short real run on the GPU."""
import numpy as np
import pytest

from paper_2604_13847_b200 import driver


def test_splitmix64_known_answer():
    # splitmix64 from state 0: first output 0xE220A8397B1DCDAF (the published reference vector).
    assert driver.splitmix64(0) == 0xE220A8397B1DCDAF
    assert driver.mix_seed(42, 0) == driver.splitmix64(driver.splitmix64(42) ^ 0)
    assert len({driver.mix_seed(42, t) for t in range(100)}) == 100


def test_iteration_row_format_and_summary():
    rec = driver.summarize([[10.0, 30.0], [20.0, 20.0]])
    assert rec["iter_ms"] == 40.0 and rec["max_mb_ms"] == 30.0 and rec["mean_mb_ms"] == 20.0
    assert rec["imbalance"] == 1.5 and rec["bubble_ms"] == 0.0
    rec.update(dst_overhead_ms=0.25, avg_budget=12.5, mean_cov_drop=0.0123456789)
    row = driver.iteration_row("sab_dst", 3, rec)
    assert row == "sab_dst,3,40.000000,1.500000,30.000000,20.000000,0.000000,0.250000,12.500000,0.012346\n"
    assert driver.ITER_HEADER.count(",") == row.count(",")


def test_cli_rejects_ungrouped_heads(monkeypatch):
    """--heads must be a multiple of --kv-heads (GQA groups); rejected before any CUDA call."""
    monkeypatch.setattr("sys.argv", ["driver", "--heads", "32", "--kv-heads", "5"])
    with pytest.raises(SystemExit) as e:
        driver.main()
    assert e.value.code == 2


@pytest.mark.gpu
def test_driver_short_run(tmp_path):
    import torch

    dist_spec = dict(short_weight=0.6, short_log_mean=float(np.log(512)), short_log_sigma=0.0,
                     long_log_mean=float(np.log(4096)), long_log_sigma=0.0, max_length=8192)
    drv = driver.Driver("sab_dst", gbs=4, mbs=1, layers=2, heads=4, kv_heads=2, head_dim=128, dist_spec=dist_spec,
                        project_pp=2, device=torch.device("cuda", 0))
    recs = drv.run(2, str(tmp_path))
    assert len(recs) == 2
    for r in recs:
        assert r["iter_ms"] > 0 and r["imbalance"] >= 1.0 and len(r["mb_ms"][0]) == 4
        assert r["pp"]["iter_ms"] > 0 and r["pp"]["bubble_ms"] >= 0  # 4 micro-batches through 2 projected stages
    lines = (tmp_path / "iterations.csv").read_text().splitlines()
    assert lines[0] + "\n" == driver.ITER_HEADER and len(lines) == 3
    assert (tmp_path / "decisions_1.csv").read_text().startswith("iter,mb,layer,")
    assert (tmp_path / "plan_0.json").exists()
    assert len((tmp_path / "iterations_pp2.csv").read_text().splitlines()) == 3
    # Closed loop: the decisions came from the GPU profiles; replaying them through the host
    # planner (fresh estimator = iteration 0's state) reproduces the decisions bit for bit.
    from paper_2604_13847_b200.host import api

    z = np.load(tmp_path / "gpu_profiles_0.npz")
    lengths = z["lengths"]
    profiles = [[z[f"p{i}_{l}"] for l in range(2)] for i in range(len(lengths))]
    h = api()
    est = h.make_estimator(h.default_bin_edges(8192), budget_grid=drv.grid)
    sp = h.plan_step("sab_dst", np.arange(4), lengths, profiles, gbs=4, mbs=1, dp=1, num_layers=2, table=drv.table,
                     est=est, iter_index=0, **drv.plan_kw)
    assert sp["decisions"] == recs[0]["decisions"]
    assert np.array_equal(sp["budgets"], recs[0]["budgets"])
