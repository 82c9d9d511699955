"""GPU cost-table profiler: its CSVs round-trip through the reference
reader (proj/core/src/profile_table.cpp:168-182 writer, :190-263 loader) with the isotonic
repair in k, and on the GPU it measures fwd and bwd per cell (not bwd = 2 x fwd, sim.hpp:23)."""
import numpy as np
import pytest

from paper_2604_13847_b200 import profiler
from paper_2604_13847_b200.host import ProfileTable, api


def _fake(bins, grid, seed):
    rng = np.random.default_rng(seed)
    x = np.asarray(bins, float)[:, None]
    k = np.asarray(grid, float)[None, :]
    lat = 0.05 + 1e-6 * x + 3e-8 * x * np.minimum(k * 128, x)
    lat = lat * rng.uniform(0.9, 1.1, size=lat.shape)  # measurement noise: non-monotone in k
    return ProfileTable(np.asarray(bins), np.asarray(grid), lat)


def test_write_tables_roundtrip_and_isotonic_repair(tmp_path, ref):
    bins, grid = [256, 4096, 32768, 131072], [1, 2, 4, 8, 16, 32, 64]
    f, b = _fake(bins, grid, 1), _fake(bins, grid, 2)
    tot = ProfileTable(f.length_bins, f.budget_grid, f.latency_ms + b.latency_ms)
    prefix = str(tmp_path / "table")
    rep = profiler.write_tables(prefix, f, b, tot)
    h = api()
    for path, t in ((prefix + "_fwd.csv", f), (prefix + "_bwd.csv", b), (prefix + ".csv", tot)):
        loaded, repaired = h.load_table(path)
        assert repaired == rep[path]
        assert np.array_equal(loaded.length_bins, t.length_bins) and np.array_equal(loaded.budget_grid, t.budget_grid)
        # isotonic repair in k: non-decreasing rows; cells that were already monotone are unchanged
        assert (np.diff(loaded.latency_ms, axis=1) >= 0).all()
        # the compiled reference reads the same file into the same table, bit for bit
        rl, rr = ref.load_table(path)
        assert rr == repaired and np.array_equal(rl.latency_ms, loaded.latency_ms)
        # CSV bytes are the reference writer's (%.17g)
        ref.save_table(t, str(tmp_path / "ref.csv"))
        assert open(path, "rb").read() == open(tmp_path / "ref.csv", "rb").read()
    assert sum(rep.values()) > 0  # the noise made the repair do something


@pytest.mark.gpu
def test_profiler_measures_fwd_and_bwd(tmp_path):
    fwd, bwd, tot = profiler.profile_tables([2048, 65536], [1, 4, 16], heads=8, kv_heads=2, reps=2)
    assert (fwd.latency_ms > 0).all() and (bwd.latency_ms > 0).all()
    assert np.allclose(tot.latency_ms, fwd.latency_ms + bwd.latency_ms)
    # the larger cell costs more (x = 65536 at k = 16 vs x = 2048 at k = 1), in both passes; at
    # x = 8192 both forward cells were ~0.2 ms of fixed per-layer cost and compared by noise
    assert fwd.latency_ms[1, 2] > fwd.latency_ms[0, 0] and bwd.latency_ms[1, 2] > bwd.latency_ms[0, 0]
    rep = profiler.write_tables(str(tmp_path / "t"), fwd, bwd, tot)
    assert set(rep) == {str(tmp_path / "t_fwd.csv"), str(tmp_path / "t_bwd.csv"), str(tmp_path / "t.csv")}


def test_mix_lengths():
    """--mix cells: packed micro-batches of the 40 % 32K / 60 % 2K mix summing to x exactly."""
    for x in (256, 2048, 32768, 49152, 71680, 143360, 262144):
        m = profiler.mix_lengths(x)
        assert sum(m) == x and all(0 < v <= 32768 for v in m)
        if x >= 71680:
            full = [v for v in m if v in (32768, 2048)]
            frac = sum(v == 32768 for v in full) / len(full)
            assert 0.3 <= frac <= 0.5, (x, m)
    assert profiler.mix_lengths(71680) == [32768, 2048, 32768, 2048, 2048]
