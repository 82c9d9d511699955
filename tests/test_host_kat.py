"""Known-answer tests for the host decision layer, taken from the reference's own tests
(proj/tests/workload_test.cpp) and the SPEC's per-operation examples (SPEC.md:126-146,
206-240, 293-339, 402-404). CPU only."""
import numpy as np
import pytest

from paper_2604_13847_b200._native import ConfigError
from paper_2604_13847_b200.host import ProfileTable

PROF = [0.5, 0.3, 0.15, 0.05]


def spec_table():
    # x in {8192}, k in {16, 32}; padded to two rows (validate_table needs 2).
    return ProfileTable([8192, 16384], [16, 32], [[100.0, 140.0], [100.0, 140.0]])


def test_predict_kat(host):
    t = spec_table()
    assert host.predict(t, 8192, 16) == (100.0, False)
    assert host.predict(t, 8192, 24) == (120.0, False)
    ms, ex = host.predict(t, 32768, 16)
    assert ms == 100.0 and ex


def test_align_kat(host):
    t = spec_table()
    assert host.align(t, 8192, 130) == (16, False)
    assert host.align(t, 8192, 200) == (32, False)
    assert host.align(t, 8192, 50) == (16, True)


def test_coverage_kat(host):
    assert host.coverage(PROF, 2) == 0.5 + 0.3
    assert host.coverage(PROF, 0) == 0.0
    assert host.coverage(PROF, 4) == 1.0
    assert host.coverage(PROF, 10) == 1.0


def test_select_anchor_kat(host):
    assert host.select_anchor([2, 4, 6], "mean") == 4.0
    assert host.select_anchor([2, 4, 6], "min") == 2.0
    assert host.select_anchor([5], "max") == 5.0
    with pytest.raises(ConfigError):
        host.select_anchor([], "min")


def test_tune_budget_kat(host):
    # grid {1,2,3,4}, k_base 4, k_anchor 2; p=0.1 -> 3, p=0.2 -> 2.
    # Two micro-batches: the anchor one (x small) and the bottleneck (x large), min anchor.
    t = ProfileTable([1000, 2000], [1, 2, 3, 4], [[1, 2, 3, 4], [2, 4, 6, 8]])
    d = host.tune_global_batch(t, [2000, 1000], [4, 4], [np.array(PROF), np.array(PROF)], threshold_p=0.1,
                               anchor="min", budget_grid=[1, 2, 3, 4])
    assert d[0].k_anchor == 2 and d[0].k_final == 3 and d[0].direction == "compressed"
    assert abs(d[0].coverage_drop - 0.05) < 1e-12
    d = host.tune_global_batch(t, [2000, 1000], [4, 4], [np.array(PROF), np.array(PROF)], threshold_p=0.2,
                               anchor="min", budget_grid=[1, 2, 3, 4])
    assert d[0].k_final == 2


def test_bin_packing_kat(host):
    bins = host.bin_packing([8, 7, 6, 5, 4], 2)
    loads = sorted(sum([8, 7, 6, 5, 4][i] for i in b) for b in bins)
    assert loads == [15, 15]
    bins = host.bin_packing([10, 1, 9, 2], 2, 2)
    loads = sorted(sum([10, 1, 9, 2][i] for i in b) for b in bins)
    assert loads == [11, 11]
    with pytest.raises(ConfigError):
        host.bin_packing([1.0], 2)


def test_make_micro_batch_kat(host):
    # workload_test.cpp:277-295
    ld, merged = host.make_micro_batch([100, 300], [[np.array([0.6, 0.4])], [np.array([0.7, 0.2, 0.1])]])
    assert ld == 400
    np.testing.assert_allclose(merged[0], [0.675, 0.25, 0.075], atol=1e-12)


def test_coverage_budget_kat(host):
    # workload_test.cpp:391-397
    assert [host.coverage_budget(PROF, t) for t in (0.5, 0.8, 0.9, 0.96)] == [1, 2, 3, 4]


def test_intrinsic_budget_kat(host):
    # workload_test.cpp:399-411
    p = [np.array(PROF)]
    assert host.intrinsic_budget(p, [1, 2, 4, 8], 0.9) == 4
    assert host.intrinsic_budget(p, [1, 2, 4, 8], 0.5) == 1
    assert host.intrinsic_budget(p, [1, 2, 4, 8], 1.0) == 4
    assert host.intrinsic_budget(p, [1, 2], 0.99) == 2


def test_estimator_ema_kat(host):
    # 0.8*32 + 0.2*16 = 28.8; 0.8*28.8 + 0.2*24 = 27.84
    est = host.make_estimator([1024, 2048], ema_alpha=0.2, default_budget=32.0)
    host.calibrate(est, [16], [100])
    assert est.ema_budget[0] == 0.8 * 32 + 0.2 * 16
    host.calibrate(est, [24], [100])
    assert est.ema_budget[0] == 0.8 * (0.8 * 32 + 0.2 * 16) + 0.2 * 24
    assert host.estimate_sparsity(est, 100) == 24  # nearest grid to 27.84
    assert host.estimate_sparsity(est, 10 ** 9) == 32  # clamps to last bin


def test_generate_samples_invariants(host):
    # workload_test.cpp:38-55 and :110-126
    lengths, profs = host.generate_samples(8, 4, 256, seed=7)
    for s, L in enumerate(lengths):
        for p in profs[s]:
            assert len(p) == (L + 255) // 256
            assert abs(p.sum() - 1.0) < 1e-9
            assert np.all(np.diff(p) <= 0)
    l2, p2 = host.generate_samples(8, 4, 256, seed=7)
    assert np.array_equal(lengths, l2)
    assert all(np.array_equal(a, b) for x, y in zip(profs, p2) for a, b in zip(x, y))
    # Unsorted draws are the same multiset.
    l3, p3 = host.generate_samples(8, 4, 256, seed=7, sorted=False)
    assert np.array_equal(lengths, l3)
    for x, y in zip(profs, p3):
        for a, b in zip(x, y):
            assert np.array_equal(a, np.sort(b)[::-1])


def test_plan_divisibility_error(host):
    with pytest.raises(ConfigError):
        host.plan_batching("lbb", list(range(5)), [1, 2, 3, 4, 5], gbs=5, mbs=1, dp=2)


def test_table_roundtrip_and_isotonic_repair(host, tmp_path):
    t = host.synthesize_table(noise_sigma=0.3, seed=3)
    p = str(tmp_path / "t.csv")
    host.save_table(t, p)
    t2, repaired = host.load_table(p)
    assert np.all(np.diff(t2.latency_ms, axis=1) >= 0)
    raw = t.latency_ms
    expect = np.maximum.accumulate(raw, axis=1)
    np.testing.assert_array_equal(t2.latency_ms, expect)
    assert repaired == int(np.sum(expect != raw))
