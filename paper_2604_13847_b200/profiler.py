"""GPU cost-table profiler.

Replaces the reference's synthetic stand-in for hardware profiling (`synthesize_table`,
proj/core/src/profile_table.cpp:145-166) and its fixed backward ratio (`fwd_bwd_ratio` = 2.0,
sim.hpp:23, applied in micro_batch_time, sim.cpp:88-98) with measured latencies. For every
(length x, budget k) cell it runs one layer of the real hot path on x tokens -- one sequence, or
with --mix a packed micro-batch of the workload's length mix -- with keep count k (clamped per
member) and times, with CUDA events (median of `reps` windows),

  * fwd: block scorer (K1 + K2) + coverage profile (K4) + top-k selector (K3) + sparse attention
    forward (K5);
  * bwd: sparse attention backward (K6, recompute from the saved LSE);

and writes three CSVs in the reference schema `x,k,latency_ms` (profile_table.cpp:168-182):
`<out>_fwd.csv`, `<out>_bwd.csv` and `<out>.csv` = fwd + bwd per layer, the per-layer training
cost the tuner balances. load_table() applies the reference's isotonic repair in k to each
(profile_table.cpp:251-263). GQA tables (--kv-heads < --heads) use group-shared selection.

    python -m paper_2604_13847_b200.profiler --out profiles/b200_cost_table_h32_d128_b128
    python -m paper_2604_13847_b200.profiler --kv-heads 8 --out profiles/b200_cost_table_h32kv8_d128_b128
    python -m paper_2604_13847_b200.profiler --mix 40/60 --out profiles/b200_cost_table_mix4060_h32_d128_b128
    # dense budget grid + extra bins (the tables bench.py / the balance runs use): tools/gpu/tables_dense.sh
"""
from __future__ import annotations

import argparse
import math

import numpy as np
import torch

from . import ops
from .host import DEFAULT_BUDGET_GRID, DEFAULT_LENGTH_BINS, ProfileTable, api


def measure_cell(q, k, v, do, lay, kk: int, reps: int, scale: float, group: int):
    """(fwd ms, bwd ms) medians over `reps` timed windows; each window enqueues `n` layers back to
    back (as the step driver does) and divides, so host launch overhead only counts where it
    exceeds the GPU work. n shrinks for large cells so every cell costs ~ the same wall time."""
    k_seq = torch.from_numpy(np.minimum(kk, np.maximum(lay.nb_per_seq, 1)).astype(np.int32)).to(q.device)
    k_max = max(1, min(kk, lay.nb_max))
    state = {}

    def fwd():
        S = ops.block_scores(q, k, lay, scale)
        ops.coverage_profile(S, lay)  # the tuner's profile (K4) is part of every layer of the closed-loop step
        idx, cnt = ops.topk_select(S, lay, k_seq, k_max, group=group)
        o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt, scale)
        state.update(idx=idx, cnt=cnt, o=o, lse=lse)

    def bwd():
        ops.sparse_attn_bwd(q, k, v, state["o"], do, state["lse"], lay, state["idx"], state["cnt"], scale)

    fwd()
    bwd()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fwd()
    bwd()
    b.record()
    torch.cuda.synchronize()
    n = int(max(1, min(8, 20.0 / max(1e-3, a.elapsed_time(b)))))
    out = []
    for fn in (fwd, bwd):
        times = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(n):
                fn()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / n)
        out.append(float(np.median(times)))
    return out[0], out[1]


def mix_lengths(x: int, long_len: int = 32768, short_len: int = 2048, long_frac: float = 0.4):
    """A packed micro-batch of x tokens drawn from a long / short mix (the C3 / C4 workload: 40 %
    32K / 60 % 2K by count): members appended long or short to keep the running long fraction at
    long_frac, the last one truncated so the lengths sum to x exactly."""
    out, n_long = [], 0
    while sum(out) < x:
        take_long = n_long / (len(out) + 1) < long_frac
        n_long += take_long
        out.append(min(long_len if take_long else short_len, x - sum(out)))
    return out


def profile_tables(length_bins=None, budget_grid=None, heads=32, kv_heads=32, head_dim=128, block=128, reps=3,
                   seed=0, device="cuda", mix=None, passes=1):
    """-> (fwd, bwd, fwd + bwd) ProfileTables over the (length_bins x budget_grid) cells. With
    mix = (long_len, short_len, long_frac) every cell is a packed micro-batch of that mix
    (mix_lengths) with the cell's keep count clamped per member, as the kernels run it; the
    reference's predict(x = summed length, k) then prices packed micro-batches of that mix
    directly. Without it, a cell is one sequence of x tokens (the reference's model).

    passes > 1 sweeps the whole grid that many times and keeps each cell's median over the
    sweeps: a cell measured once varies by ~5 % between sweeps minutes apart (clock / power
    state under sw_power_cap), more than one budget step of the dense grid at large k."""
    length_bins = list(DEFAULT_LENGTH_BINS if length_bins is None else length_bins)
    budget_grid = list(DEFAULT_BUDGET_GRID if budget_grid is None else budget_grid)
    g = torch.Generator(device=device).manual_seed(seed)
    T = max(length_bins)
    q = torch.randn((T, heads, head_dim), generator=g, device=device).to(torch.bfloat16)
    k = torch.randn((T, kv_heads, head_dim), generator=g, device=device).to(torch.bfloat16)
    v = torch.randn((T, kv_heads, head_dim), generator=g, device=device).to(torch.bfloat16)
    do = torch.randn((T, heads, head_dim), generator=g, device=device).to(torch.bfloat16)
    scale = 1.0 / math.sqrt(head_dim)
    group = heads // kv_heads
    lf = np.zeros((passes, len(length_bins), len(budget_grid)))
    lb = np.zeros_like(lf)
    for p in range(passes):
        for xi, x in enumerate(length_bins):
            lens = mix_lengths(x, *mix) if mix else [x]
            lay = ops.VarlenLayout.build(np.concatenate([[0], np.cumsum(lens)]).astype(np.int32), block, device=device)
            for ki, kk in enumerate(budget_grid):
                lf[p, xi, ki], lb[p, xi, ki] = measure_cell(q[:x], k[:x], v[:x], do[:x], lay, kk, reps, scale, group)
    lf, lb = np.median(lf, axis=0), np.median(lb, axis=0)
    bins = np.asarray(length_bins, np.int64)
    grid = np.asarray(budget_grid, np.int32)
    return ProfileTable(bins, grid, lf), ProfileTable(bins, grid, lb), ProfileTable(bins, grid, lf + lb)


def write_tables(prefix: str, fwd: ProfileTable, bwd: ProfileTable, total: ProfileTable):
    """Save the three tables with the reference writer and load them back through load_table
    (isotonic repair in k); returns {path: repaired cell count}."""
    h = api()
    out = {}
    for path, t in ((prefix + "_fwd.csv", fwd), (prefix + "_bwd.csv", bwd), (prefix + ".csv", total)):
        h.save_table(t, path)
        out[path] = h.load_table(path)[1]
    return out


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--out", required=True, help="path prefix: writes <out>.csv, <out>_fwd.csv, <out>_bwd.csv")
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--kv-heads", type=int, default=32)
    ap.add_argument("--head-dim", type=int, default=128)
    ap.add_argument("--block", type=int, default=128)
    ap.add_argument("--max-x", type=int, default=262144)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--passes", type=int, default=1, help="sweeps of the whole grid; each cell keeps its median")
    ap.add_argument("--grid", default=None, help="comma-separated budget grid (default: the reference's 16 points)")
    ap.add_argument("--bins", default=None, help="comma-separated length bins (default: the reference's 15, <= --max-x)")
    ap.add_argument("--mix", default=None, help="'40/60': cells are packed micro-batches of the 40%% 32K / 60%% 2K "
                                                "mix (C3 / C4) instead of single sequences")
    args = ap.parse_args()
    if args.heads % args.kv_heads:
        ap.error("--heads must be a multiple of --kv-heads")
    prefix = args.out[:-4] if args.out.endswith(".csv") else args.out
    bins = [int(x) for x in args.bins.split(",")] if args.bins else [x for x in DEFAULT_LENGTH_BINS if x <= args.max_x]
    grid = [int(k) for k in args.grid.split(",")] if args.grid else None
    mix = (32768, 2048, 0.4) if args.mix == "40/60" else None
    fwd, bwd, tot = profile_tables(bins, grid, args.heads, args.kv_heads, args.head_dim, args.block, args.reps, mix=mix,
                                   passes=args.passes)
    rep = write_tables(prefix, fwd, bwd, tot)
    ratio = bwd.latency_ms / np.maximum(fwd.latency_ms, 1e-9)
    for p, r in rep.items():
        print(f"wrote {p}: {len(bins)} x {len(fwd.budget_grid)} cells, isotonic repair changed {r}")
    print(f"measured bwd/fwd ratio: min {ratio.min():.2f} median {np.median(ratio):.2f} max {ratio.max():.2f} "
          f"(reference stand-in: 2.0, sim.hpp:23)")


if __name__ == "__main__":
    main()
