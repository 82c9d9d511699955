"""Python mirror of the host decision layer: cost model, sparsity tuner, sparsity-aware batcher.

Names and argument meanings follow the reference C++ API (proj/core/include/sparsebalance/
profile_table.hpp, dst.hpp, sab.hpp, workload.hpp and the decision half of sim.hpp), so the
parity tests read like the reference's own tests. Every call goes to native C++ through the
flat C ABI declared in include/sb_host.h. ``HostAPI`` is parameterised by the symbol prefix so
the test-suite can bind the compiled reference (prefix ``sbref_``) with the very same
marshalling; the product instance is ``paper_2604_13847_b200.host.api`` (prefix ``sbh_``).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from . import _native

ANCHORS = {"min": 0, "mean": 1, "max": 2}
DIRECTIONS = ("compressed", "expanded", "unchanged")
STRATEGIES = {"baseline": 0, "dst": 1, "sab": 2, "lbb": 3, "sab_dst": 4, "lbb_dst": 5}

_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int)
_f64p = C.POINTER(C.c_double)


def _a(x, dtype):
    return np.ascontiguousarray(np.asarray(x, dtype=dtype))


def _p(arr):
    if arr is None:
        return None
    if arr.dtype == np.int64:
        return arr.ctypes.data_as(_i64p)
    if arr.dtype == np.int32:
        return arr.ctypes.data_as(_i32p)
    if arr.dtype == np.float64:
        return arr.ctypes.data_as(_f64p)
    raise TypeError(arr.dtype)


@dataclass
class ProfileTable:
    """(length-bin x budget) -> per-layer latency grid (reference profile_table.hpp:14-25)."""

    length_bins: np.ndarray
    budget_grid: np.ndarray
    latency_ms: np.ndarray  # [nx, nk]

    def __post_init__(self):
        self.length_bins = _a(self.length_bins, np.int64)
        self.budget_grid = _a(self.budget_grid, np.int32)
        self.latency_ms = _a(self.latency_ms, np.float64).reshape(len(self.length_bins), len(self.budget_grid))

    def args(self):
        return (_p(self.length_bins), len(self.length_bins), _p(self.budget_grid), len(self.budget_grid),
                _p(self.latency_ms))


@dataclass
class SparsityEstimator:
    """Per-length-bin EMA of DST budgets (reference sab.hpp:22-28)."""

    bin_edges: np.ndarray
    ema_budget: np.ndarray
    ema_alpha: float = 0.2
    budget_grid: np.ndarray = field(default_factory=lambda: np.array(DEFAULT_BUDGET_GRID, np.int32))

    def __post_init__(self):
        self.bin_edges = _a(self.bin_edges, np.int64)
        self.ema_budget = _a(self.ema_budget, np.float64).copy()
        self.budget_grid = _a(self.budget_grid, np.int32)


@dataclass
class Decision:
    micro_batch_id: int
    layer_id: int
    k_base: int
    k_anchor: int
    k_final: int
    direction: str
    coverage_drop: float
    predicted_ms_base: float
    predicted_ms_final: float


DEFAULT_LENGTH_BINS = [256, 512, 1024, 2048, 4096, 8192, 16384, 24576, 32768, 49152, 65536, 98304,
                       131072, 196608, 262144]
DEFAULT_BUDGET_GRID = [1, 2, 3, 4, 6, 8, 10, 12, 16, 20, 24, 32, 40, 48, 56, 64]


def _flatten(profiles: Sequence[np.ndarray]):
    off = np.zeros(len(profiles) + 1, np.int64)
    for i, p in enumerate(profiles):
        off[i + 1] = off[i] + len(p)
    flat = np.concatenate([_a(p, np.float64) for p in profiles]) if len(profiles) else np.zeros(0)
    return _a(flat if flat.size else np.zeros(1), np.float64), off


class HostAPI:
    """ctypes binding of the flat host ABI (include/sb_host.h) for one symbol prefix."""

    def __init__(self, cdll: C.CDLL, prefix: str = "sbh_"):
        self._lib = cdll
        self._pre = prefix
        self._err = self._fn("last_error")
        self._err.restype = C.c_char_p

    def _fn(self, name):
        return getattr(self._lib, self._pre + name)

    def _call(self, name, *args):
        f = self._fn(name)
        f.restype = C.c_int
        _native.check(f(*args), self._err)

    # ---- profile_table.hpp -------------------------------------------------------------
    def predict(self, table: ProfileTable, x: int, k: int):
        ms, ex = C.c_double(), C.c_int()
        self._call("predict", *table.args(), C.c_int64(x), C.c_int(k), C.byref(ms), C.byref(ex))
        return ms.value, bool(ex.value)

    def predict_members(self, table: ProfileTable, lengths, k: int, block_size: int):
        """Opt-in varlen-aware cost (not in the reference): sum over members of
        predict(L_s, min(k, ceil(L_s / block_size)))."""
        ms, ex = C.c_double(), C.c_int()
        la = _a(lengths, np.int64)
        self._call("predict_members", *table.args(), _p(la), len(la), int(k), int(block_size), C.byref(ms),
                   C.byref(ex))
        return ms.value, bool(ex.value)

    def align(self, table: ProfileTable, x: int, target_ms: float):
        b, inf = C.c_int(), C.c_int()
        self._call("align", *table.args(), C.c_int64(x), C.c_double(target_ms), C.byref(b), C.byref(inf))
        return b.value, bool(inf.value)

    def synthesize_table(self, length_bins=None, budget_grid=None, c_lin=2e-6, c_attn=6e-8, c_fixed=0.15,
                         noise_sigma=0.0, block_size=256, seed=42) -> ProfileTable:
        bins = _a(DEFAULT_LENGTH_BINS if length_bins is None else length_bins, np.int64)
        grid = _a(DEFAULT_BUDGET_GRID if budget_grid is None else budget_grid, np.int32)
        lat = np.zeros(len(bins) * len(grid), np.float64)
        self._call("synthesize_table", C.c_double(c_lin), C.c_double(c_attn), C.c_double(c_fixed),
                   C.c_double(noise_sigma), C.c_int(block_size), _p(bins), len(bins), _p(grid), len(grid),
                   C.c_uint64(seed), _p(lat))
        return ProfileTable(bins, grid, lat)

    def load_table(self, path: str):
        nx, nk, rep = C.c_int(), C.c_int(), C.c_int()
        self._call("load_table", path.encode(), C.byref(nx), C.byref(nk), None, None, None, C.byref(rep))
        bins = np.zeros(nx.value, np.int64)
        grid = np.zeros(nk.value, np.int32)
        lat = np.zeros(nx.value * nk.value, np.float64)
        self._call("load_table", path.encode(), C.byref(nx), C.byref(nk), _p(bins), _p(grid), _p(lat),
                   C.byref(rep))
        return ProfileTable(bins, grid, lat), rep.value

    def save_table(self, table: ProfileTable, path: str):
        self._call("save_table", path.encode(), *table.args())

    # ---- dst.hpp -----------------------------------------------------------------------
    def coverage(self, scores, k: int) -> float:
        s = _a(scores, np.float64)
        out = C.c_double()
        self._call("coverage", _p(s if s.size else np.zeros(1)), len(s), C.c_int(k), C.byref(out))
        return out.value

    def select_anchor(self, latencies, anchor: str) -> float:
        lat = _a(latencies, np.float64)
        out = C.c_double()
        self._call("select_anchor", _p(lat if lat.size else np.zeros(1)), len(lat), ANCHORS[anchor],
                   C.byref(out))
        return out.value

    def tune_global_batch(self, table: ProfileTable, x: Sequence[int], k_base: Sequence[int],
                          profiles: Sequence[np.ndarray], layer: int = 0, threshold_p: float = 0.1,
                          anchor: str = "min", budget_grid=None) -> List[Decision]:
        n = len(x)
        xs, kb = _a(x, np.int64), _a(k_base, np.int32)
        flat, off = _flatten(profiles)
        grid = _a(table.budget_grid if budget_grid is None else budget_grid, np.int32)
        oi = np.zeros(5 * n, np.int32)
        od = np.zeros(3 * n, np.float64)
        self._call("tune_global_batch", *table.args(), n, _p(xs), _p(kb), _p(flat), _p(off), layer,
                   C.c_double(threshold_p), ANCHORS[anchor], _p(grid), len(grid), _p(oi), _p(od))
        out = []
        for i in range(n):
            a, d = oi[5 * i:5 * i + 5], od[3 * i:3 * i + 3]
            out.append(Decision(int(a[0]), layer, int(a[1]), int(a[2]), int(a[3]), DIRECTIONS[a[4]],
                                float(d[0]), float(d[1]), float(d[2])))
        return out

    def coverage_table(self, scores, budget_grid, k_base: int) -> np.ndarray:
        """Extension (dst.hpp CoverageTable): [coverage(scores, g) for g in grid] + [coverage(scores, k_base)]."""
        s = _a(scores, np.float64)
        grid = _a(budget_grid, np.int32)
        out = np.zeros(len(grid) + 1, np.float64)
        self._call("coverage_table", _p(s if s.size else np.zeros(1)), len(s), _p(grid), len(grid), int(k_base),
                   _p(out))
        return out

    def tune_global_batch_cov(self, table: ProfileTable, x: Sequence[int], k_base: Sequence[int], cov,
                              layer: int = 0, threshold_p: float = 0.1, anchor: str = "min", budget_grid=None,
                              member_lengths: Sequence[Sequence[int]] | None = None,
                              varlen_block_size: int = 0) -> List[Decision]:
        """tune_global_batch over coverage tables cov[n_mb][len(grid) + 1] (coverage_table rows)
        instead of profiles; bit-identical decisions."""
        n = len(x)
        xs, kb = _a(x, np.int64), _a(k_base, np.int32)
        grid = _a(table.budget_grid if budget_grid is None else budget_grid, np.int32)
        cv = _a(np.asarray(cov, np.float64).reshape(n, len(grid) + 1), np.float64)
        ml = mo = None
        if member_lengths is not None:
            mo = _a(np.concatenate([[0], np.cumsum([len(m) for m in member_lengths])]), np.int64)
            flat = [int(v) for m in member_lengths for v in m]
            ml = _a(flat if flat else [0], np.int64)
        oi = np.zeros(5 * n, np.int32)
        od = np.zeros(3 * n, np.float64)
        self._call("tune_global_batch_cov", *table.args(), n, _p(xs), _p(kb), _p(cv), None if ml is None else _p(ml),
                   None if mo is None else _p(mo), int(varlen_block_size), layer, C.c_double(threshold_p),
                   ANCHORS[anchor], _p(grid), len(grid), _p(oi), _p(od))
        out = []
        for i in range(n):
            a, d = oi[5 * i:5 * i + 5], od[3 * i:3 * i + 3]
            out.append(Decision(int(a[0]), layer, int(a[1]), int(a[2]), int(a[3]), DIRECTIONS[a[4]],
                                float(d[0]), float(d[1]), float(d[2])))
        return out

    def rank_estimate(self, lengths, per_member_profiles, budget_grid, coverage_mode: bool = True,
                      base_budget: int = 32, coverage_target: float = 0.9):
        """Batched make_micro_batch + intrinsic_budget + per-layer coverage tables:
        per_member_profiles[s][l] -> (x, k_base, cov [L, len(grid) + 1])."""
        ns = len(lengths)
        nl = len(per_member_profiles[0]) if ns else 0
        flat, off = _flatten([p for m in per_member_profiles for p in m])
        grid = _a(budget_grid, np.int32)
        x, kb = C.c_int64(), C.c_int()
        cov = np.zeros((nl, len(grid) + 1), np.float64)
        self._call("rank_estimate", ns, _p(_a(lengths, np.int64)), nl, _p(flat), _p(off), _p(grid), len(grid),
                   1 if coverage_mode else 0, int(base_budget), C.c_double(coverage_target), C.byref(x), C.byref(kb),
                   _p(cov))
        return int(x.value), int(kb.value), cov

    def tune_layers_cov(self, table: ProfileTable, x, k_base, cov, budget_grid, threshold_p: float = 0.1,
                        anchor: str = "min", member_lengths=None, varlen_block_size: int = 0):
        """tune_global_batch_cov for every layer: cov [n_mb, L, len(grid) + 1] ->
        (k_final [n_mb, L], decisions in layer-major order)."""
        cov = _a(np.asarray(cov, np.float64), np.float64)
        n, nl = cov.shape[0], cov.shape[1]
        grid = _a(budget_grid, np.int32)
        ml = mo = None
        if member_lengths is not None:
            mo = _a(np.concatenate([[0], np.cumsum([len(m) for m in member_lengths])]), np.int64)
            flat = [int(v) for m in member_lengths for v in m]
            ml = _a(flat if flat else [0], np.int64)
        kf = np.zeros((n, nl), np.int32)
        oi = np.zeros(5 * n * nl, np.int32)
        od = np.zeros(3 * n * nl, np.float64)
        self._call("tune_layers_cov", *table.args(), n, _p(_a(x, np.int64)), _p(_a(k_base, np.int32)), _p(cov),
                   None if ml is None else _p(ml), None if mo is None else _p(mo), int(varlen_block_size), nl,
                   C.c_double(threshold_p), ANCHORS[anchor], _p(grid), len(grid), _p(kf), _p(oi), _p(od))
        out = []
        for l in range(nl):
            for i in range(n):
                o = l * n + i
                a, d = oi[5 * o:5 * o + 5], od[3 * o:3 * o + 3]
                out.append(Decision(int(a[0]), l, int(a[1]), int(a[2]), int(a[3]), DIRECTIONS[a[4]], float(d[0]),
                                    float(d[1]), float(d[2])))
        return kf, out

    # ---- workload.hpp ------------------------------------------------------------------
    def make_micro_batch(self, lengths: Sequence[int], profiles: Sequence[Sequence[np.ndarray]]):
        """profiles[s][l] -> (length_descriptor, merged[l])."""
        ns, nl = len(lengths), len(profiles[0]) if len(profiles) else 0
        flat, off = _flatten([p for s in profiles for p in s])
        cap = max(1, sum(max(len(profiles[s][l]) for s in range(ns)) for l in range(nl)))
        out = np.zeros(cap, np.float64)
        out_off = np.zeros(nl + 1, np.int64)
        ld = C.c_int64()
        self._call("make_micro_batch", ns, _p(_a(lengths, np.int64)), nl, _p(flat), _p(off), _p(out),
                   C.c_int64(cap), _p(out_off), C.byref(ld))
        return ld.value, [out[out_off[l]:out_off[l + 1]].copy() for l in range(nl)]

    def coverage_budget(self, scores, target: float) -> int:
        s = _a(scores, np.float64)
        out = C.c_int()
        self._call("coverage_budget", _p(s if s.size else np.zeros(1)), len(s), C.c_double(target), C.byref(out))
        return out.value

    def intrinsic_budget(self, merged_profiles: Sequence[np.ndarray], budget_grid, target: float) -> int:
        flat, off = _flatten(merged_profiles)
        g = _a(budget_grid, np.int32)
        out = C.c_int()
        self._call("intrinsic_budget", len(merged_profiles), _p(flat), _p(off), _p(g if g.size else np.zeros(1, np.int32)),
                   len(g), C.c_double(target), C.byref(out))
        return out.value

    def generate_samples(self, count: int, num_layers: int, block_size: int, seed: int, kind: str = "bimodal",
                         sorted: bool = True, dist: dict | None = None, conc: dict | None = None):
        """Reference generate_samples (workload.cpp:239-271) -> (lengths, profiles[s][l]).

        sorted=False returns the same draws before the per-profile descending sort."""
        d = dict(min_length=64, max_length=65536, fixed_length=8192, short_weight=0.55,
                 short_log_mean=7.3132203870903064, short_log_sigma=0.7, long_log_mean=10.308952660644293,
                 long_log_sigma=0.45, tail_exponent=1.1)
        d.update(dist or {})
        c = dict(alpha_log_mean=-1.0498221244986776, alpha_log_sigma=0.3, layer_log_sigma=0.35,
                 length_ref=12288.0, length_exponent=3.2)
        c.update(conc or {})
        dv = _a([d["min_length"], d["max_length"], d["fixed_length"], d["short_weight"], d["short_log_mean"],
                 d["short_log_sigma"], d["long_log_mean"], d["long_log_sigma"], d["tail_exponent"]], np.float64)
        cv = _a([c["alpha_log_mean"], c["alpha_log_sigma"], c["layer_log_sigma"], c["length_ref"],
                 c["length_exponent"]], np.float64)
        kinds = {"fixed": 0, "bimodal": 1, "long_tail": 2}
        lengths = np.zeros(count, np.int64)
        off = np.zeros(count * num_layers + 1, np.int64)
        args = (kinds[kind], _p(dv), _p(cv), C.c_int64(count), num_layers, block_size, C.c_uint64(seed),
                1 if sorted else 0, _p(lengths), _p(off))
        self._call("generate_samples", *args, None)
        flat = np.zeros(max(1, int(off[-1])), np.float64)
        self._call("generate_samples", *args, _p(flat))
        profiles = [[flat[off[s * num_layers + l]:off[s * num_layers + l + 1]].copy() for l in range(num_layers)]
                    for s in range(count)]
        return lengths, profiles

    # ---- sab.hpp -----------------------------------------------------------------------
    def default_bin_edges(self, max_length: int) -> np.ndarray:
        out = np.zeros(64, np.int64)
        n = C.c_int()
        self._call("default_bin_edges", C.c_int64(max_length), _p(out), 64, C.byref(n))
        return out[:n.value].copy()

    def make_estimator(self, bin_edges, budget_grid=None, ema_alpha=0.2, default_budget=32.0):
        grid = _a(DEFAULT_BUDGET_GRID if budget_grid is None else budget_grid, np.int32)
        edges = _a(bin_edges, np.int64)
        return SparsityEstimator(edges, np.full(len(edges), float(default_budget)), ema_alpha, grid)

    def estimate_sparsity(self, est: SparsityEstimator, length: int) -> int:
        out = C.c_int()
        self._call("estimate_sparsity", _p(est.bin_edges), len(est.bin_edges), _p(est.ema_budget),
                   _p(est.budget_grid), len(est.budget_grid), C.c_int64(length), C.byref(out))
        return out.value

    def calibrate(self, est: SparsityEstimator, k_final: Sequence[int], lengths: Sequence[int]) -> None:
        k = _a(k_final, np.int32)
        ln = _a(lengths, np.int64)
        self._call("calibrate", _p(est.bin_edges), len(est.bin_edges), _p(est.ema_budget), C.c_double(est.ema_alpha),
                   _p(est.budget_grid), len(est.budget_grid), len(k), _p(k if k.size else np.zeros(1, np.int32)),
                   _p(ln if ln.size else np.zeros(1, np.int64)))

    def bin_packing(self, weights, num_bins: int, max_items_per_bin: int = 0) -> List[List[int]]:
        w = _a(weights, np.float64)
        items = np.zeros(max(1, len(w)), np.int32)
        boff = np.zeros(max(1, num_bins) + 1, np.int32)
        self._call("bin_packing", _p(w if w.size else np.zeros(1)), len(w), num_bins, max_items_per_bin,
                   _p(items), _p(boff))
        return [items[boff[b]:boff[b + 1]].tolist() for b in range(num_bins)]

    def plan_batching(self, strategy: str, ids, lengths, gbs: int, mbs: int, dp: int,
                      est: SparsityEstimator | None = None, table: ProfileTable | None = None):
        """strategy in {sab, lbb, sequential} -> (micro_batch_bins[rank][mb] -> ids, weights)."""
        code = {"sab": 0, "lbb": 1, "sequential": 2}[strategy]
        ids_a, len_a = _a(ids, np.int64), _a(lengths, np.int64)
        if est is None:
            est = self.make_estimator(self.default_bin_edges(65536))
        if table is None:
            table = self.synthesize_table()
        n = len(ids_a)
        out_ids = np.zeros(max(1, n), np.int64)
        mpr = gbs // max(1, mbs * dp) if mbs * dp else 0
        out_off = np.zeros(max(1, dp * max(1, mpr)) + 1, np.int32)
        out_w = np.zeros(max(1, n), np.float64)
        self._call("plan_batching", code, n, _p(ids_a), _p(len_a), gbs, mbs, dp, _p(est.bin_edges),
                   len(est.bin_edges), _p(est.ema_budget), C.c_double(est.ema_alpha), _p(est.budget_grid),
                   len(est.budget_grid), *table.args(), _p(out_ids), _p(out_off), _p(out_w))
        bins = [[out_ids[out_off[r * mpr + m]:out_off[r * mpr + m + 1]].tolist() for m in range(mpr)]
                for r in range(dp)]
        return bins, out_w[:n].copy()

    # ---- step.hpp (decision half of the reference's simulate_iteration) -----------------
    def plan_step(self, strategy: str, ids, lengths, profiles, *, gbs: int, mbs: int, dp: int, num_layers: int,
                  table: ProfileTable, est: SparsityEstimator, iter_index: int = 0, base_budget: int = 32,
                  base_mode: str = "coverage", base_coverage_target: float = 0.9, dst_scope: str = "global",
                  threshold_p: float = 0.1, anchor: str = "min", dst_grid=None, calibrate_every: int = 1,
                  decisions_csv: str | None = None, plan_json: str | None = None, varlen_block_size: int = 0):
        n = len(ids)
        flat, off = _flatten([p for s in profiles for p in s])
        setup_i = _a([gbs, mbs, dp, num_layers, base_budget, 1 if base_mode == "coverage" else 0,
                      1 if dst_scope == "global" else 0, calibrate_every, varlen_block_size], np.int32)
        setup_d = _a([base_coverage_target, threshold_p], np.float64)
        grid = _a([] if dst_grid is None else dst_grid, np.int32)
        mpr = gbs // (mbs * dp)
        out_b = np.zeros(dp * mpr * num_layers, np.int32)
        out_ids = np.zeros(n, np.int64)
        out_off = np.zeros(dp * mpr + 1, np.int32)
        cap = dp * mpr * num_layers
        oi = np.zeros(6 * cap, np.int32)
        od = np.zeros(3 * cap, np.float64)
        nd = C.c_int()
        stats = np.zeros(2, np.float64)
        self._call("plan_step", STRATEGIES[strategy], n, _p(_a(ids, np.int64)), _p(_a(lengths, np.int64)), _p(flat),
                   _p(off), _p(setup_i), _p(setup_d), ANCHORS[anchor], _p(grid if grid.size else np.zeros(1, np.int32)),
                   len(grid), _p(est.bin_edges), len(est.bin_edges), _p(est.ema_budget), C.c_double(est.ema_alpha),
                   _p(est.budget_grid), len(est.budget_grid), *table.args(), iter_index, _p(out_b), _p(out_ids),
                   _p(out_off), _p(oi), _p(od), cap, C.byref(nd), _p(stats),
                   None if decisions_csv is None else str(decisions_csv).encode(),
                   None if plan_json is None else str(plan_json).encode())
        decisions = []
        for i in range(nd.value):
            a, d = oi[6 * i:6 * i + 6], od[3 * i:3 * i + 3]
            decisions.append(Decision(int(a[0]), int(a[1]), int(a[2]), int(a[3]), int(a[4]), DIRECTIONS[a[5]],
                                      float(d[0]), float(d[1]), float(d[2])))
        bins = [[out_ids[out_off[r * mpr + m]:out_off[r * mpr + m + 1]].tolist() for m in range(mpr)]
                for r in range(dp)]
        return dict(budgets=out_b.reshape(dp, mpr, num_layers), micro_batch_bins=bins, decisions=decisions,
                    mean_cov_drop=float(stats[0]), avg_budget=float(stats[1]))


    def ref_simulate_iteration(self, strategy: str, ids, lengths, profiles, *, gbs: int, mbs: int, dp: int, pp: int,
                               layers_per_stage: int, table: ProfileTable, est: SparsityEstimator, iter_index: int = 0,
                               fwd_bwd_ratio: float = 2.0, comm_ms: float = 0.05, dp_sync_ms: float = 5.0,
                               base_budget: int = 32, base_mode: str = "coverage", base_coverage_target: float = 0.9,
                               dst_scope: str = "global", threshold_p: float = 0.1, anchor: str = "min",
                               dst_grid=None, calibrate_every: int = 1) -> dict:
        """Test oracle only (the compiled reference, prefix sbref_): the reference step driver's
        ScheduleResult with a pipeline-parallel cluster (sim.cpp:277-489)."""
        n = len(ids)
        num_layers = pp * layers_per_stage
        flat, off = _flatten([p for s in profiles for p in s])
        setup_i = _a([gbs, mbs, dp, num_layers, base_budget, 1 if base_mode == "coverage" else 0,
                      1 if dst_scope == "global" else 0, calibrate_every, 0], np.int32)
        setup_d = _a([base_coverage_target, threshold_p], np.float64)
        grid = _a([] if dst_grid is None else dst_grid, np.int32)
        res = np.zeros(8, np.float64)
        self._call("ref_simulate_iteration", STRATEGIES[strategy], n, _p(_a(ids, np.int64)),
                   _p(_a(lengths, np.int64)), _p(flat), _p(off), _p(setup_i), _p(setup_d), ANCHORS[anchor],
                   _p(grid if grid.size else np.zeros(1, np.int32)), len(grid), _p(est.bin_edges), len(est.bin_edges),
                   _p(est.ema_budget), C.c_double(est.ema_alpha), _p(est.budget_grid), len(est.budget_grid),
                   *table.args(), iter_index, _p(_a([pp, layers_per_stage], np.int32)),
                   _p(_a([fwd_bwd_ratio, comm_ms, dp_sync_ms], np.float64)), _p(res))
        keys = ("iter_ms", "bubble_ms", "critical_lb_ms", "max_mb_ms", "mean_mb_ms", "imbalance", "avg_budget",
                "mean_cov_drop")
        return dict(zip(keys, res.tolist()))


_api = None


def api() -> HostAPI:
    """The product host layer (this repo's C++ re-implementation)."""
    global _api
    if _api is None:
        _api = HostAPI(_native.lib(), "sbh_")
    return _api
