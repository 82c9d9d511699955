"""Host decision layer vs committed golden fixtures generated from the compiled reference
(oracle/gen_golden.py). Runs everywhere, including the GPU box where /root/reference and the
reference library are absent. Doubles are compared bit-exactly (stored as float.hex)."""
import numpy as np

from paper_2604_13847_b200.host import ProfileTable
from tests.golden_io import load_host_golden, load_routing_golden


def test_predict_align_golden(host):
    g = load_host_golden()
    t = g["table"]
    table = ProfileTable(t["length_bins"], t["budget_grid"], t["latency_ms"])
    for x, k, target, ms_hex, ex, b, inf in g["predict_align"]:
        ms, e = host.predict(table, x, k)
        assert ms == float.fromhex(ms_hex) and e == ex
        assert host.align(table, x, target) == (b, inf)


def test_plan_step_golden(host):
    g = load_host_golden()
    t = g["table"]
    table = ProfileTable(t["length_bins"], t["budget_grid"], t["latency_ms"])
    for run in g["plan_step"]:
        est = host.make_estimator(host.default_bin_edges(65536))
        for it, exp in enumerate(run["iterations"]):
            L, P = host.generate_samples(run["gbs"], run["num_layers"], 128, seed=exp["seed"], dist=run["dist"])
            res = host.plan_step(run["strategy"], np.arange(run["gbs"]), L, P, gbs=run["gbs"], mbs=run["mbs"],
                                 dp=run["dp"], num_layers=run["num_layers"], table=table, est=est, iter_index=it,
                                 anchor=run["anchor"], dst_scope=run["scope"], base_mode=run["base_mode"],
                                 threshold_p=0.1)
            assert res["budgets"].tolist() == exp["budgets"], run["name"]
            assert res["micro_batch_bins"] == exp["bins"]
            got = [[d.micro_batch_id, d.layer_id, d.k_base, d.k_anchor, d.k_final, d.direction, d.coverage_drop.hex(),
                    d.predicted_ms_base.hex(), d.predicted_ms_final.hex()] for d in res["decisions"]]
            assert got == exp["decisions"]
            assert [v.hex() for v in est.ema_budget] == exp["ema"]


def test_routing_golden_coverage(host):
    """Reference routing profiles (pre-sort + sorted) and reference coverage(): the sort of the
    pre-sort vector is the reference profile, and this repo's coverage() reproduces it."""
    for pre, srt, ks, cov in load_routing_golden():
        assert np.array_equal(np.sort(pre)[::-1], srt)
        for k, c in zip(ks, cov):
            assert host.coverage(srt, int(k)) == c
