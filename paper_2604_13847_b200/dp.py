"""Data-parallel SparseBalance step driver: one process per GPU, NCCL for the plumbing.

Re-hosts the reference step driver's decision path (proj/core/src/sim.cpp:277-432) on real
kernels. Per optimizer step:

  1. SAB plan (host, deterministic on every rank, no collective): the global batch's lengths ->
     rank -> micro-batch assignment (plan_batching / plan_lbb / plan_sequential, sab.cpp:224-310).
  2. Per rank, per layer: block scorer (K1+K2) + coverage profile (K4) on this rank's packed
     micro-batch -> one RoutingProfile per (sequence, layer), copied to the host.
  3. ONE all-gather of every rank's workload estimate: its micro-batch length descriptor and
     its per-layer member profiles (a few KB). Concatenating rank-major reproduces the
     reference's pooled order (sim.cpp:357-369).
  4. Every rank runs the identical host DST over the pooled micro-batches (make_micro_batch
     merge, coverage-mode intrinsic_budget, tune_global_batch per layer): bit-identical
     k_final on all ranks with no broadcast.
  5. Per layer: top-k selection with k_final clamped per sequence, sparse attention fwd + bwd.

There is no KV or sequence exchange between ranks (no CP / ring / Ulysses): the only
collectives are the step-3 all-gather and the caller's gradient all-reduce.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np
import torch

# SB_NVTX=1: an NVTX range per layer phase (select + fwd, bwd) for nsys / ncu --nvtx timelines.
_NVTX = os.environ.get("SB_NVTX", "0") == "1"

from . import ops
from .host import DEFAULT_BUDGET_GRID, ProfileTable, api


@dataclass
class DstSettings:
    threshold_p: float = 0.1
    anchor: str = "mean"           # paper default; the reference defaults to min
    base_mode: str = "coverage"    # or "fixed"
    base_budget: int = 32          # fixed mode
    coverage_target: float = 0.9
    budget_grid: Sequence[int] = field(default_factory=lambda: list(DEFAULT_BUDGET_GRID))


@dataclass
class RankBatch:
    """This rank's packed micro-batch (one micro-batch per rank per step)."""

    lengths: np.ndarray      # member sequence lengths
    sample_ids: List[int]
    layout: ops.VarlenLayout

    @property
    def length_descriptor(self) -> int:
        return int(self.lengths.sum())


def assign_rank_batches(global_lengths: Sequence[int], dp: int, mbs: int, strategy: str = "lbb", est=None,
                        table: ProfileTable | None = None):
    """SAB / LBB / sequential plan of the global batch (reference plan_batching / plan_lbb /
    plan_sequential, sab.cpp:224-310) -> per rank the list of micro-batches (sample ids)."""
    h = api()
    n = len(global_lengths)
    bins, _ = h.plan_batching(strategy, np.arange(n), np.asarray(global_lengths), n, mbs, dp, est, table)
    return bins


def profiles_to_host(prof: torch.Tensor, lay: ops.VarlenLayout) -> List[np.ndarray]:
    """[nseq, nb_max] fp64 device profiles -> per-sequence numpy vectors of nb_s entries."""
    p = prof.cpu().numpy()
    return [p[s, :nb].copy() for s, nb in enumerate(lay.nb_per_seq)]


@dataclass
class RankEstimate:
    """One micro-batch's workload estimate, everything the pooled DST reads:
    the length descriptor x, the base budget and, per layer, the merged profile's coverage at the
    budget grid plus at k_base (host CoverageTable). Member lengths ride along for the opt-in
    varlen cost model only."""

    x: int
    k_base: int
    cov: np.ndarray                 # [num_layers, len(grid) + 1] fp64
    members: np.ndarray | None = None


def rank_estimate(lengths, layer_profiles: List[List[np.ndarray]], cfg: DstSettings) -> RankEstimate:
    """Local half of the exchange: merge this rank's member profiles exactly as the reference's
    make_micro_batch (workload.cpp:64-99), take the coverage-mode base budget over all layers
    (intrinsic_budget, workload.cpp:389-411; sim.cpp:321-326) and tabulate C(k) per layer (one
    native call). layer_profiles[l][s] = member s's profile at layer l."""
    L = len(layer_profiles)
    per_member = [[layer_profiles[l][s] for l in range(L)] for s in range(len(lengths))]
    x, k_base, cov = api().rank_estimate(np.asarray(lengths, np.int64), per_member, cfg.budget_grid,
                                         cfg.base_mode == "coverage", cfg.base_budget, cfg.coverage_target)
    return RankEstimate(x, k_base, cov, np.asarray(lengths, np.int64))


def pack_estimate(est: RankEstimate, num_layers: int, n_grid: int, max_members: int = 0) -> torch.Tensor:
    """Fixed-size fp64 vector [x, k_base, n_members, members (padded to max_members), cov]. Every
    field is an integer < 2^53 or a double, so the round trip is exact. The size depends only on
    (num_layers, n_grid, max_members), which every rank knows: one all-gather, no size exchange."""
    if est.cov.shape != (num_layers, n_grid + 1):
        raise ValueError(f"coverage table shape {est.cov.shape} != {(num_layers, n_grid + 1)}")
    mem = est.members if (max_members and est.members is not None) else np.zeros(0, np.int64)
    if len(mem) > max_members:
        raise ValueError(f"{len(mem)} members exceed max_members={max_members}")
    out = np.zeros(3 + max_members + num_layers * (n_grid + 1), np.float64)
    out[0], out[1], out[2] = est.x, est.k_base, len(mem)
    out[3:3 + len(mem)] = mem
    out[3 + max_members:] = est.cov.reshape(-1)
    return torch.from_numpy(out)


def unpack_estimate(vec: np.ndarray, num_layers: int, n_grid: int, max_members: int = 0) -> RankEstimate:
    n = int(vec[2])
    members = vec[3:3 + n].astype(np.int64) if max_members else None
    cov = vec[3 + max_members:3 + max_members + num_layers * (n_grid + 1)].reshape(num_layers, n_grid + 1).copy()
    return RankEstimate(int(vec[0]), int(vec[1]), cov, members)


def exchange_estimates(est: RankEstimate, num_layers: int, n_grid: int, world: int, group=None, device="cpu",
                       max_members: int = 0) -> List[RankEstimate]:
    """All-gather every rank's estimate -> the pooled list, rank-major (the reference's pooled
    order, sim.cpp:357-369). 8 * (3 + max_members + L * (|K| + 1)) bytes per rank: 4.9 KB for 36
    layers on the default 16-point grid, 74 KB on the dense 1..256 grid. NCCL on GPU tensors,
    gloo on CPU."""
    mine = pack_estimate(est, num_layers, n_grid, max_members)
    if world == 1:
        return [unpack_estimate(mine.numpy(), num_layers, n_grid, max_members)]
    import torch.distributed as dist

    buf = mine.to(device)
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    flat = torch.stack(outs).cpu().numpy()  # one D2H for all ranks
    return [unpack_estimate(flat[r], num_layers, n_grid, max_members) for r in range(world)]


def decide_budgets_cov(pooled: List[RankEstimate], table: ProfileTable, cfg: DstSettings, num_layers: int,
                       varlen_block_size: int = 0):
    """Pooled host DST from the exchanged estimates (one native call for all layers): k_final
    [rank][layer] and the decisions, bit-identical to decide_budgets on the underlying profiles
    (tune_global_batch_cov)."""
    mem = [e.members for e in pooled] if varlen_block_size else None
    cov = np.stack([e.cov for e in pooled]) if pooled else np.zeros((0, num_layers, len(cfg.budget_grid) + 1))
    k_final, decisions = api().tune_layers_cov(table, [e.x for e in pooled], [e.k_base for e in pooled], cov,
                                               cfg.budget_grid, threshold_p=cfg.threshold_p, anchor=cfg.anchor,
                                               member_lengths=mem, varlen_block_size=varlen_block_size)
    return k_final, decisions, np.asarray([e.k_base for e in pooled]), np.asarray([e.x for e in pooled])


def decide_budgets(pooled, table: ProfileTable, cfg: DstSettings, num_layers: int):
    """Host DST over pooled micro-batch PROFILES (rank-major): the replay / parity form of
    decide_budgets_cov (same decisions). pooled = list over ranks of (lengths, per-member
    per-layer profiles)."""
    h = api()
    grid = np.asarray(cfg.budget_grid, np.int32)
    xs, merged, k_base = [], [], []
    for lengths, prof in pooled:
        ld, mp = h.make_micro_batch(lengths, prof)  # reference make_micro_batch merge (workload.cpp:64-99)
        xs.append(ld)
        merged.append(mp)
        if cfg.base_mode == "coverage":
            k_base.append(h.intrinsic_budget(mp, grid, cfg.coverage_target))
        else:
            k_base.append(cfg.base_budget)
    k_final = np.zeros((len(pooled), num_layers), np.int32)
    decisions = []
    for l in range(num_layers):
        ds = h.tune_global_batch(table, xs, k_base, [m[l] for m in merged], layer=l, threshold_p=cfg.threshold_p,
                                 anchor=cfg.anchor, budget_grid=grid)
        for d in ds:
            k_final[d.micro_batch_id, l] = d.k_final
        decisions.extend(ds)
    return k_final, decisions, np.asarray(k_base), np.asarray(xs)


def fixed_base_plan(table: ProfileTable, xs, k_base, cfg: DstSettings):
    """Host half of the on-device DST (fixed-base mode).

    Everything tune_budget needs except the profile follows from the pooled micro-batches'
    summed lengths and fixed base budgets (dst.cpp:107-169): T_base = predict(x, k_base), the
    anchor over all of them, k_anchor = align(x, anchor) and the bottleneck flag. Identical on
    every rank with no collective; the coverage test then runs on the device per layer
    (ops.dst_decide)."""
    h = api()
    base_ms = [h.predict(table, int(x), int(kb))[0] for x, kb in zip(xs, k_base)]
    anchor = h.select_anchor(base_ms, cfg.anchor)
    k_anchor = [h.align(table, int(x), anchor)[0] for x in xs]
    bottleneck = [1 if t > anchor else 0 for t in base_ms]
    return np.asarray(k_anchor, np.int32), np.asarray(bottleneck, np.int32), anchor


class DPStep:
    """One rank's hot-path step over its micro-batch for `num_layers` layers.

    Layers share the synthetic Q/K/V/dO tensors but each layer uses its own softmax
    temperature (scale_l / sqrt(d)), so per-layer routing profiles -- and the tuner's per-layer
    budgets -- differ as they do across real layers. The tuner is closed-loop: its profiles
    are this step's K4 coverage profiles of the GPU block scores (planted_qk() gives synthetic
    Q/K whose block scores carry the reference generator's routing structure)."""

    def __init__(self, batch: RankBatch, q, k, v, do, layer_scales, table: ProfileTable, cfg: DstSettings,
                 rank: int = 0, world: int = 1, group=None, pooled_xs=None, max_members: int = 0,
                 varlen_block_size: int = 0, fused_bwd: bool = False):
        self.batch, self.q, self.k, self.v, self.do = batch, q, k, v, do
        self.layer_scales = list(layer_scales)
        self.table, self.cfg = table, cfg
        self.rank, self.world, self.group = rank, world, group
        self.d = q.shape[2]
        self.sel_group = q.shape[1] // k.shape[1]  # GQA: group-shared selection
        self.block = batch.layout.block_size
        self.max_members = max(max_members, len(batch.lengths)) if varlen_block_size else 0
        self.varlen_block_size = varlen_block_size
        self.fused_bwd = fused_bwd  # backward: the opt-in fused single pass instead of the two-pass
        self.last = {}
        # On-device DST (fixed-base mode): with every rank's micro-batch
        # summed length known (the SAB plan is deterministic on every rank), the host half
        # (k_anchor, bottleneck) is computed here once and the per-layer coverage test runs on the
        # device: no profile download, no all-gather, no per-layer host round trip.
        self.on_device = pooled_xs is not None
        if self.on_device:
            if cfg.base_mode != "fixed":
                raise ValueError("on-device DST needs base_mode='fixed' (coverage mode needs the pooled profiles)")
            kb = [cfg.base_budget] * len(pooled_xs)
            ka, bn, _ = fixed_base_plan(table, pooled_xs, kb, cfg)
            dev = q.device
            self._dev_plan = dict(
                mb_off=torch.tensor([0, batch.layout.nseq], dtype=torch.int32, device=dev),
                k_base=torch.tensor([cfg.base_budget], dtype=torch.int32, device=dev),
                k_anchor=torch.tensor([int(ka[rank])], dtype=torch.int32, device=dev),
                bottleneck=torch.tensor([int(bn[rank])], dtype=torch.int32, device=dev),
                grid=torch.tensor(list(cfg.budget_grid), dtype=torch.int32, device=dev))

    def scorer_pass(self):
        """K1 + K2 + K4 for every layer (the scorer pre-pass coverage-mode budgets need) ->
        (block scores per layer, device profiles [L, nseq, nb_max] fp64)."""
        lay = self.batch.layout
        qbar, kbar = ops.block_pool(self.q, lay), ops.block_pool(self.k, lay)
        scores = []
        profs = torch.empty((len(self.layer_scales), lay.nseq, max(1, lay.nb_max)), dtype=torch.float64,
                            device=self.q.device)
        for l, s_l in enumerate(self.layer_scales):
            S = ops.block_scores(self.q, self.k, lay, s_l / math.sqrt(self.d), qbar=qbar, kbar=kbar)
            scores.append(S)
            profs[l] = ops.coverage_profile(S, lay)
        return scores, profs

    def local_estimate(self, profs: torch.Tensor) -> RankEstimate:
        """One D2H of all layers' profiles, then the local merge + coverage tables."""
        lay = self.batch.layout
        if getattr(self, "_prof_host", None) is None or self._prof_host.shape != profs.shape:
            self._prof_host = torch.empty(profs.shape, dtype=profs.dtype).pin_memory()
        self._prof_host.copy_(profs)  # synchronous D2H into persistent pinned memory
        host = self._prof_host.numpy()
        nb = lay.nb_per_seq
        layer_profiles = [[host[l, s, :nb[s]].copy() for s in range(lay.nseq)] for l in range(host.shape[0])]
        self.last_profiles = layer_profiles
        return rank_estimate(self.batch.lengths, layer_profiles, self.cfg)

    def run(self, backward: bool = True, mark=None, grad_buckets=None):
        """mark(tag) (optional) is called at phase boundaries: 'decided' after the scorer
        pre-pass + exchange + DST, then 'fwd' / 'bwd' after each layer's kernels.

        self.last['busy'] = (start, end) CUDA-event pairs bracketing this rank's own kernels
        (scorer pre-pass; layer loop), excluding the all-gather wait and the host DST: the
        per-rank busy time the imbalance metric uses (reference Eq. 9 over per-rank totals).

        grad_buckets (optional, one tensor per layer): the step-end gradient all-reduce of
        SURVEY.md section 8(e). The attention op has no parameters, so the caller passes a stand-in
        (e.g. the layer's output-projection gradient); each layer's bucket is all-reduced
        asynchronously on NCCL's stream as soon as that layer's backward is enqueued, DDP-style,
        overlapping the next layers' kernels, and the compute stream waits for all of them at
        the end."""
        lay = self.batch.layout
        if self.on_device:
            return self._run_on_device(backward, mark, grad_buckets)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        scores, profs = self.scorer_pass()
        ev[1].record()
        est = self.local_estimate(profs)
        L = len(self.layer_scales)
        pooled = exchange_estimates(est, L, len(self.cfg.budget_grid), self.world, self.group, self.q.device,
                                    self.max_members)
        k_final, decisions, k_base, xs = decide_budgets_cov(pooled, self.table, self.cfg, L, self.varlen_block_size)
        self.last = dict(k_final=k_final, decisions=decisions, k_base=k_base, xs=xs, estimate=est, pooled=pooled)
        if mark:
            mark("decided")
        nb = lay.nb_per_seq
        # All layers' per-sequence keep counts in one pinned, asynchronous H2D copy (a pageable
        # copy would block the host behind the GPU once per layer).
        k_all = np.minimum(k_final[self.rank][:, None], nb[None, :]).astype(np.int32)
        # persistent pinned staging (a fresh pin_memory() per step can cudaHostAlloc on the host path);
        # the previous step's copy out of it completed before this step's profile D2H returned
        if getattr(self, "_k_host", None) is None or self._k_host.shape != k_all.shape:
            self._k_host = torch.empty(k_all.shape, dtype=torch.int32).pin_memory()
        self._k_host.numpy()[...] = k_all
        k_dev = self._k_host.to(self.q.device, non_blocking=True)
        ev[2].record()
        outs, works = [], []
        for l, s_l in enumerate(self.layer_scales):
            k_max = int(max(1, k_all[l].max()))
            scale = s_l / math.sqrt(self.d)
            if _NVTX:
                torch.cuda.nvtx.range_push(f"layer {l} k<={k_max}: select + fwd")
            idx, cnt = ops.topk_select(scores[l], lay, k_dev[l], k_max, group=self.sel_group)
            o, lse = ops.sparse_attn_fwd(self.q, self.k, self.v, lay, idx, cnt, scale)
            if _NVTX:
                torch.cuda.nvtx.range_pop()
            if mark:
                mark("fwd")
            if _NVTX and backward:
                torch.cuda.nvtx.range_push(f"layer {l}: bwd")
            grads = (ops.sparse_attn_bwd(self.q, self.k, self.v, o, self.do, lse, lay, idx, cnt, scale,
                                         fused=self.fused_bwd) if backward else None)
            if _NVTX and backward:
                torch.cuda.nvtx.range_pop()
            if mark:
                mark("bwd")
            if grad_buckets is not None and self.world > 1:
                import torch.distributed as dist

                works.append(dist.all_reduce(grad_buckets[l], group=self.group, async_op=True))
            # Only the last layer's O / gradients stay referenced (a 36-layer step would otherwise
            # hold ~1.3 GB x 36 of activations); every layer keeps its selection.
            last = l == len(self.layer_scales) - 1
            outs.append((idx, cnt, o if last else None, grads if last else None))
        ev[3].record()
        self.last["busy"] = [(ev[0], ev[1]), (ev[2], ev[3])]
        for w_ in works:
            w_.wait()  # the compute stream waits for every bucket
        return outs

    def _run_on_device(self, backward, mark, grad_buckets):
        """The step with K8 deciding each layer's keep count on the device (fixed-base mode)."""
        lay = self.batch.layout
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        qbar, kbar = ops.block_pool(self.q, lay), ops.block_pool(self.k, lay)
        if mark:
            mark("decided")
        k_max = int(min(max(self.cfg.budget_grid), lay.nb_max))
        dp_ = self._dev_plan
        outs, works, k_finals = [], [], []
        for l, s_l in enumerate(self.layer_scales):
            scale = s_l / math.sqrt(self.d)
            S = ops.block_scores(self.q, self.k, lay, scale, qbar=qbar, kbar=kbar)
            prof = ops.coverage_profile(S, lay)
            k_final, _, k_seq = ops.dst_decide(prof, lay, dp_["mb_off"], dp_["k_base"], dp_["k_anchor"],
                                               dp_["bottleneck"], dp_["grid"], self.cfg.threshold_p)
            k_finals.append(k_final)
            idx, cnt = ops.topk_select(S, lay, k_seq, k_max, group=self.sel_group)
            o, lse = ops.sparse_attn_fwd(self.q, self.k, self.v, lay, idx, cnt, scale)
            if mark:
                mark("fwd")
            grads = (ops.sparse_attn_bwd(self.q, self.k, self.v, o, self.do, lse, lay, idx, cnt, scale,
                                         fused=self.fused_bwd) if backward else None)
            if mark:
                mark("bwd")
            if grad_buckets is not None and self.world > 1:
                import torch.distributed as dist

                works.append(dist.all_reduce(grad_buckets[l], group=self.group, async_op=True))
            # Only the last layer's O / gradients stay referenced (a 36-layer step would otherwise
            # hold ~1.3 GB x 36 of activations); every layer keeps its selection.
            last = l == len(self.layer_scales) - 1
            outs.append((idx, cnt, o if last else None, grads if last else None))
        ev[1].record()
        for w_ in works:
            w_.wait()
        self.last = dict(k_final_device=k_finals, busy=[(ev[0], ev[1])])
        return outs


