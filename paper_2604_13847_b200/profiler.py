"""GPU cost-table profiler.

Replaces the reference's synthetic stand-in for hardware profiling (`synthesize_table`,
proj/core/src/profile_table.cpp:145-166) with measured latencies. For every (length x, budget k)
cell of the grid it runs the real per-layer forward hot path (block scorer + top-k selector +
sparse attention forward) on one packed sequence of x tokens with keep count k, times it with
CUDA events (median of `reps`) and writes the reference CSV schema `x,k,latency_ms`
(profile_table.cpp:168-182). load_table() then applies the same isotonic repair in k
(profile_table.cpp:251-263). The simulator's convention is kept: the table holds the forward
per-layer latency; backward = forward x fwd_bwd_ratio (sim.hpp:23).

    python -m paper_2604_13847_b200.profiler --out b200_cost_table.csv
"""
from __future__ import annotations

import argparse
import math

import numpy as np
import torch

from . import ops
from .host import DEFAULT_BUDGET_GRID, DEFAULT_LENGTH_BINS, ProfileTable, api


def measure_cell(q, k, v, lay, kk: int, reps: int, scale: float) -> float:
    """Median over `reps` timed windows of the per-layer forward hot path; each window enqueues 8
    layers back to back (as the step driver does) and divides, so the host's launch overhead
    only counts where it exceeds the GPU work."""
    k_seq = torch.full((lay.nseq,), kk, dtype=torch.int32, device=q.device)
    k_max = max(1, min(kk, lay.nb_max))

    def layer():
        S = ops.block_scores(q, k, lay, scale)
        idx, cnt = ops.topk_select(S, lay, k_seq, k_max)
        ops.sparse_attn_fwd(q, k, v, lay, idx, cnt, scale)

    layer()
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(8):
            layer()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 8)
    return float(np.median(times))


def profile_table(length_bins=None, budget_grid=None, heads=32, kv_heads=32, head_dim=128, block=128, reps=3,
                  seed=0, device="cuda") -> ProfileTable:
    length_bins = list(DEFAULT_LENGTH_BINS if length_bins is None else length_bins)
    budget_grid = list(DEFAULT_BUDGET_GRID if budget_grid is None else budget_grid)
    g = torch.Generator(device=device).manual_seed(seed)
    T = max(length_bins)
    q = torch.randn((T, heads, head_dim), generator=g, device=device).to(torch.bfloat16)
    k = torch.randn((T, kv_heads, head_dim), generator=g, device=device).to(torch.bfloat16)
    v = torch.randn((T, kv_heads, head_dim), generator=g, device=device).to(torch.bfloat16)
    scale = 1.0 / math.sqrt(head_dim)
    lat = np.zeros((len(length_bins), len(budget_grid)))
    for xi, x in enumerate(length_bins):
        lay = ops.VarlenLayout.build([0, x], block, device=device)
        qx, kx, vx = q[:x], k[:x], v[:x]
        for ki, kk in enumerate(budget_grid):
            lat[xi, ki] = measure_cell(qx, kx, vx, lay, kk, reps, scale)
    return ProfileTable(np.asarray(length_bins, np.int64), np.asarray(budget_grid, np.int32), lat)


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--out", required=True)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--kv-heads", type=int, default=32)
    ap.add_argument("--head-dim", type=int, default=128)
    ap.add_argument("--block", type=int, default=128)
    ap.add_argument("--max-x", type=int, default=262144)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    bins = [x for x in DEFAULT_LENGTH_BINS if x <= args.max_x]
    t = profile_table(bins, None, args.heads, args.kv_heads, args.head_dim, args.block, args.reps)
    h = api()
    h.save_table(t, args.out)
    loaded, repaired = h.load_table(args.out)
    print(f"wrote {args.out}: {len(bins)} x {len(t.budget_grid)} cells, isotonic repair changed {repaired}")


if __name__ == "__main__":
    main()
