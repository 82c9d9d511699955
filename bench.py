#!/usr/bin/env python
"""Benchmark of the SparseBalance hot path on B200.

Headline workload at every N (BASELINE.json configs[2], "C3", one weak-scaling family from 1 to
8 GPUs): the reference workload generator's 40% 32K / 60% 2K global batch of gbs = 5 * N samples
(proj/core/src/workload.cpp:239-271, seed 42), planned by SAB into one packed micro-batch per
rank (sab.cpp:224-273), 36 layers, 32 heads MHA, d128, B128. Q/K carry planted block-routing
structure (synth.py: the generator's own pre-sort routing draws per member), so the GPU block
scores reproduce the generator's concentration. One step per rank =

    scorer pre-pass over all layers (K1 + K2 + K4 coverage profiles)
    -> one D2H of the profiles, local make_micro_batch merge + coverage tables
    -> one all-gather of {x, k_base, C(K) per layer} (N > 1)
    -> pooled host DST (Mean anchor, p = 0.1, global scope, coverage base) -> k_final per layer
    -> per layer: top-k selector (K3) + sparse attention fwd (K5) + bwd (K6)

value = useful TFLOP/s of the whole job = sum over ranks of useful selected-block FLOPs
(14 * d * sum e_ij per q head: 4 fwd + 10 bwd) / max-over-ranks step time. max_over_mean is
taken over per-rank BUSY time (CUDA events around each rank's own kernels, excluding the
all-gather wait and host DST), per step as the reference's Eq. 9 (sim.cpp:478-485).

At N = 1 the line also carries measured sub-records: C2 (configs[1], one 32K packed layer),
C5 (configs[4], one 128K sequence, GQA 32/8, keep 0.1) and C1 (configs[0], 4K, H8, d64, B64,
keep 0.25, forward latency beside the CPU oracle on the same input).
"""
from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "max-over-ranks sparse-attn step ms & useful TFLOPS at 1/2/4/8 B200 vs CPU ref"
CFG = dict(tokens=32768, heads=32, head_dim=128, block=128, keep_lo=0.05, keep_hi=0.5, seed=42)
C3_DIST = dict(short_weight=0.6, short_log_mean=float(np.log(2048)), short_log_sigma=0.0,
               long_log_mean=float(np.log(32768)), long_log_sigma=0.0)
FWD_TILE_M = {64: 128, 128: 128}  # query rows per forward UMMA tile at block size B (attn_fwd.cu)
# The C3 / C4 workload's own GPU-measured cost table: cells are packed micro-batches of the 40 %
# 32K / 60 % 2K mix (profiler.py --mix 40/60), fwd + bwd per layer, every budget 1..16 (align()
# returns table-grid budgets, so the grid step is DST's balance granularity; tables_dense.sh).
COST_TABLE = os.path.join(ROOT, "profiles", "b200_cost_table_mix4060dense_h32_d128_b128.csv")


def peaks():
    """MEASURED_PEAKS.json: (burst bf16 TF/s, sustained bf16 TF/s, sustained clock MHz, HBM GB/s, source).
    The roofline denominator is the BURST figure: the timed windows are ~0.1-1 s after idle, and
    the sustained figure was taken at a lower power-capped clock than these kernels run at."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return (float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", p["bf16_tflops"])),
                p.get("clocks_under_load", {}).get("sm_mhz_median"), float(p["hbm_gbs"]), "measured")
    except Exception:
        return 1590.0, 1400.0, 1300.0, 6650.0, "fallback (B200_PROFILING.md)"


def c2_workload(rank: int):
    """C2 micro-batch of 32768 tokens: the SURVEY.md section 8(d) example composition
    [12288, 8192, 4096, 2048 x 4] packed with cu_seqlens, and per-sequence keep ratios
    U[0.05, 0.5] seeded by rank."""
    lens = [12288, 8192, 4096, 2048, 2048, 2048, 2048]
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    rng = np.random.default_rng(CFG["seed"] + 7919 * rank)
    nb = (np.array(lens) + CFG["block"] - 1) // CFG["block"]
    keep = rng.uniform(CFG["keep_lo"], CFG["keep_hi"], size=len(lens))
    k_seq = np.maximum(1, np.ceil(keep * nb)).astype(np.int32)
    return cu, k_seq


workload = c2_workload  # tools/ import the old name


def pair_entries(cu, B, idx, cnt):
    """sum over selection rows of e_ij (unmasked score entries of pair (i, j)): r_i * c_j off the
    diagonal, r_i (r_i + 1) / 2 on it; and the executed-tile count."""
    cu = np.asarray(cu, np.int64)
    nb = (np.diff(cu) + B - 1) // B
    blk = np.concatenate([[0], np.cumsum(nb)])
    seq_of = np.repeat(np.arange(len(nb)), nb)
    local = np.arange(int(blk[-1])) - blk[seq_of]
    lens = np.diff(cu)[seq_of]
    rows = np.minimum(B, lens - local * B)
    k_max = idx.shape[2]
    valid = np.arange(k_max)[None, None, :] < cnt[:, :, None]
    sel = np.where(valid, idx, 0).astype(np.int64)
    kv_rows = rows[blk[seq_of][None, :, None] + sel]
    r = rows[None, :, None]
    diag = sel == local[None, :, None]
    e = np.where(valid, np.where(diag, r * (r + 1) // 2, r * kv_rows), 0).sum(dtype=np.int64)
    return float(e), float(valid.sum())


def useful_flops(cu, B, idx, cnt, d, hq=None):
    """(fwd, bwd) useful FLOPs: 4*d*sum(e_ij) and 10*d*sum(e_ij) over q heads. idx/cnt rows are
    per selection head; with group-shared selection (hsel < hq) each row serves hq / hsel heads."""
    e, _ = pair_entries(cu, B, idx, cnt)
    mult = (hq // idx.shape[0]) if hq else 1
    return 4.0 * d * e * mult, 10.0 * d * e * mult


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = f"/tmp/sb_clocks_{os.getpid()}.csv"

    def __enter__(self):
        if os.environ.get("SB_NO_CLOCK_SAMPLER"):  # debug: measure without nvidia-smi polling
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=open(self.path, "w"),
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        try:
            rows = [l.split(",") for l in open(self.path).read().strip().splitlines()]
        except Exception:
            return None
        sm, mx, reasons = [], 0, set()
        for r in rows:
            try:
                c, m = float(r[0]), float(r[1])
            except Exception:
                continue
            mx = max(mx, m)
            if len(r) > 7 and float(r[7]) > 0:
                sm.append(c)
            names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
            for n, val in zip(names, r[3:7]):
                if "Active" in val and "Not" not in val:
                    reasons.add(n)
        if not sm:
            sm = [float(r[0]) for r in rows if r and r[0].strip().replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(rows)}


C2_LABEL = ("C2: 32K-token packed varlen micro-batch ([12288, 8192, 4096, 2048x4], SURVEY 8d), 32 heads MHA, d128, "
            "B128, per-sequence keep U[0.05,0.5], scorer+profile+selector+fwd+bwd, one layer")


def c3_label(world: int, layers: int, table_src: str) -> str:
    return (f"C3: 40% 32K / 60% 2K global batch (reference generator, seed 42, gbs={5 * world}), SAB plan mbs=5 "
            f"(one packed micro-batch per rank), {layers} layers, planted block-routing Q/K (generator pre-sort "
            f"routing draws), closed-loop per-layer DST from the GPU coverage profiles (Mean anchor, p=0.1, global "
            f"scope, coverage base, {table_src}), 32 heads MHA, d128, B128, "
            "scorer+profile D2H+allgather+DST+selector+fwd+bwd")


def cost_table():
    from paper_2604_13847_b200.host import api

    if os.path.exists(COST_TABLE):
        return api().load_table(COST_TABLE)[0], "GPU-measured cost table " + os.path.relpath(COST_TABLE, ROOT)
    return api().synthesize_table(block_size=CFG["block"]), "synthetic cost table"


def host_cores() -> int:
    """Host threads this process may use (affinity / cgroup aware). torchrun sets
    OMP_NUM_THREADS=1 per rank; the CPU arm overrides that to use the whole host."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def c3_global_batch(world: int, seed: int, layers: int = 1, sorted_: bool = True):
    """C3: the reference workload generator's 40% 32K / 60% 2K bimodal mix, gbs = 5 * dp ->
    (lengths, per-sample per-layer routing profiles)."""
    from paper_2604_13847_b200.host import api

    lengths, profiles = api().generate_samples(5 * world, layers, CFG["block"], seed=seed, dist=C3_DIST,
                                               sorted=sorted_)
    return np.asarray(lengths), profiles


def c3_rank0_layer0(world, layers):
    """CPU-arm sample: rank 0's packed micro-batch of the C3 global batch (same SAB plan and cost
    table as the GPU arm) and a layer-0 keep count per sequence from the pooled host DST over the
    generator's routing profiles (the GPU arm's closed-loop counts come from its own scores)."""
    from paper_2604_13847_b200 import dp

    lengths_all, profiles_all = c3_global_batch(world, CFG["seed"], layers)
    table, _ = cost_table()
    bins = dp.assign_rank_batches(lengths_all, world, 5, "sab", table=table)
    pooled = []
    for r in range(world):
        ids = bins[r][0]
        pooled.append((np.asarray([int(lengths_all[i]) for i in ids]),
                       [[profiles_all[i][l] for l in range(layers)] for i in ids]))
    k_final, _, _, _ = dp.decide_budgets(pooled, table, dp.DstSettings(), layers)
    mine = [int(x) for x in pooled[0][0]]
    cu = np.concatenate([[0], np.cumsum(mine)]).astype(np.int32)
    nb = (np.diff(cu) + CFG["block"] - 1) // CFG["block"]
    return cu, np.minimum(int(k_final[0][0]), nb).astype(np.int32)


def _bf16_np(rng, shape):
    return (rng.standard_normal(shape).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)


def run_reference_arm(args, rank, world):
    """--impl reference: the reference has no CPU attention; the CPU arm is this repo's
    oracle port of the path (oracle/sb_oracle.c, fp64, all host threads) on a bounded sample of
    the same workload (q head 0 of rank 0's micro-batch: 1/32 of a layer), scaled per unit."""
    if rank != 0:
        return
    from oracle import device as orc

    c3 = args.workload == "c3"
    cu, k_seq = c3_rank0_layer0(world, args.layers) if c3 else c2_workload(0)
    T, D, B = int(cu[-1]), CFG["head_dim"], CFG["block"]
    rng = np.random.default_rng(1)
    q, k, v, do = (_bf16_np(rng, (T, 1, D)) for _ in range(4))
    threads = orc.set_threads(host_cores())
    scale = 1.0 / math.sqrt(D)
    times, flops = [], None
    budget_s, start, warm_done = args.ref_budget_s, time.perf_counter(), 0
    for it in range(args.warmup + args.steps):
        # Bounded run: the work per step is deterministic, so once one warm-up and one timed step
        # are in, further steps only tighten the mean; stop before the wall-clock budget is spent.
        spent = time.perf_counter() - start
        est = spent / it if it else 0.0
        if it < args.warmup:
            if warm_done and spent + 2 * est > budget_s:  # keep room for one timed step
                continue
        elif times and spent + est > budget_s:
            break
        t0 = time.perf_counter()
        qb, kb = orc.block_pool(q, cu, B), orc.block_pool(k, cu, B)
        S = orc.block_scores(qb, kb, cu, B, scale).astype(np.float32)
        orc.coverage_profile(S, cu, B)
        idx, cnt = orc.topk_select(S, cu, B, k_seq, int(k_seq.max()))
        o, lse = orc.sparse_attn_fwd(q, k, v, cu, B, idx, cnt, scale)
        orc.sparse_attn_bwd(q, k, v, o, do, lse, cu, B, idx, cnt, scale)
        dt = time.perf_counter() - t0
        if flops is None:
            f, b = useful_flops(cu, B, idx, cnt, D)
            flops = f + b
        if it >= args.warmup:
            times.append(dt)
        else:
            warm_done += 1
    ms = 1e3 * statistics.mean(times)
    value = flops / (ms * 1e-3) / 1e12
    sample = (f"q head 0 of 32, {'layer 0 (DST keep count)' if c3 else 'one layer'}, of rank 0's {T}-token "
              f"micro-batch ({len(cu) - 1} seqs): scorer, profile, selector, fwd, bwd")
    _, table_src = cost_table()
    label = c3_label(world, args.layers, table_src) if c3 else C2_LABEL
    line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": label, "sample": "CPU port: " + sample, "warmup_run": warm_done,
                       "steps_timed": len(times), "budget_s": budget_s},
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


class Marker:
    """Records CUDA events at tagged phase boundaries inside a step (on the launching stream)."""

    def __init__(self, torch, stream):
        self.torch, self.stream = torch, stream
        self.marks = []
        self.host = []

    def __call__(self, tag):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record(self.stream)
        self.marks.append((tag, e))
        self.host.append(time.perf_counter())

    def durations(self):
        """ms per tag: time from the previous mark to this one, summed per tag."""
        out = {}
        for (_, a), (tag, b) in zip(self.marks, self.marks[1:]):
            out[tag] = out.get(tag, 0.0) + a.elapsed_time(b)
        return out


def time_fn(torch, fn, steps, warmup=3):
    """Mean device ms of fn() over `steps` back-to-back calls after `warmup` (CUDA events)."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def sub_c2(torch, ops, dev, steps, burst):
    """C2 (configs[1]): one 32K packed layer, scorer -> profile -> selector -> fwd -> bwd."""
    H, D, B = CFG["heads"], CFG["head_dim"], CFG["block"]
    cu, k_seq = c2_workload(0)
    T = int(cu[-1])
    lay = ops.VarlenLayout.build(cu, B, device=dev)
    g = torch.Generator(device=dev).manual_seed(CFG["seed"])
    q, k, v, do = (torch.randn((T, H, D), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
    kseq_d = torch.from_numpy(k_seq).to(dev)
    k_max = int(k_seq.max())
    scale = 1.0 / math.sqrt(D)
    S = ops.block_scores(q, k, lay, scale)
    idx, cnt = ops.topk_select(S, lay, kseq_d, k_max)
    o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt, scale)
    f_fwd, f_bwd = useful_flops(cu, B, idx.cpu().numpy(), cnt.cpu().numpy(), D)

    def full():
        S_ = ops.block_scores(q, k, lay, scale)
        ops.coverage_profile(S_, lay)
        i_, c_ = ops.topk_select(S_, lay, kseq_d, k_max)
        o_, l_ = ops.sparse_attn_fwd(q, k, v, lay, i_, c_, scale)
        ops.sparse_attn_bwd(q, k, v, o_, do, l_, lay, i_, c_, scale)

    t_step = time_fn(torch, full, steps)
    t_fwd = time_fn(torch, lambda: ops.sparse_attn_fwd(q, k, v, lay, idx, cnt, scale), steps)
    t_bwd = time_fn(torch, lambda: ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt, scale), steps)
    return {"workload": C2_LABEL, "ms_per_step": t_step, "useful_tflop": (f_fwd + f_bwd) / 1e12,
            "tflops": (f_fwd + f_bwd) / (t_step * 1e-3) / 1e12,
            "fwd_ms": t_fwd, "fwd_tflops": f_fwd / (t_fwd * 1e-3) / 1e12,
            "fwd_frac_burst": f_fwd / (t_fwd * 1e-3) / 1e12 / burst,
            "bwd_ms": t_bwd, "bwd_tflops": f_bwd / (t_bwd * 1e-3) / 1e12,
            "bwd_frac_burst": f_bwd / (t_bwd * 1e-3) / 1e12 / burst}


def sub_c5(torch, ops, dev, steps, burst, keep=0.1):
    """C5 (configs[4]): one 131072-token sequence, GQA 32q / 8kv with group-shared selection,
    keep 0.1 (k = ceil(0.1 * 1024) = 103), fwd + bwd."""
    T, Hq, Hkv, D, B = 131072, 32, 8, 128, 128
    cu = np.array([0, T], np.int32)
    lay = ops.VarlenLayout.build(cu, B, device=dev)
    g = torch.Generator(device=dev).manual_seed(CFG["seed"] + 5)
    q = torch.randn((T, Hq, D), generator=g, device=dev).to(torch.bfloat16)
    k, v = (torch.randn((T, Hkv, D), generator=g, device=dev).to(torch.bfloat16) for _ in range(2))
    do = torch.randn((T, Hq, D), generator=g, device=dev).to(torch.bfloat16)
    nb = T // B
    kk = max(1, math.ceil(keep * nb))
    scale = 1.0 / math.sqrt(D)
    S = ops.block_scores(q, k, lay, scale)
    idx, cnt = ops.topk_select(S, lay, torch.tensor([kk], dtype=torch.int32, device=dev), kk, group=Hq // Hkv)
    o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt, scale)
    f_fwd, f_bwd = useful_flops(cu, B, idx.cpu().numpy(), cnt.cpu().numpy(), D, hq=Hq)
    t_fwd = time_fn(torch, lambda: ops.sparse_attn_fwd(q, k, v, lay, idx, cnt, scale), steps)
    t_bwd = time_fn(torch, lambda: ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt, scale), steps)
    del q, k, v, do, o, lse, S
    return {"workload": f"C5: one 131072-token sequence, GQA 32q/8kv (group-shared selection), d128, B128, keep "
                        f"{keep} (k={kk}), fwd + bwd", "useful_tflop": (f_fwd + f_bwd) / 1e12,
            "ms_per_step": t_fwd + t_bwd, "tflops": (f_fwd + f_bwd) / ((t_fwd + t_bwd) * 1e-3) / 1e12,
            "fwd_ms": t_fwd, "fwd_tflops": f_fwd / (t_fwd * 1e-3) / 1e12,
            "fwd_frac_burst": f_fwd / (t_fwd * 1e-3) / 1e12 / burst,
            "bwd_ms": t_bwd, "bwd_tflops": f_bwd / (t_bwd * 1e-3) / 1e12,
            "bwd_frac_burst": f_bwd / (t_bwd * 1e-3) / 1e12 / burst}


def sub_c1(torch, ops, dev, steps, with_cpu=True):
    """C1 (configs[0]): single 4096-token sequence, 8 heads MHA, d64, B64, keep 0.25 (k = 16):
    forward latency (the attention kernel alone and scorer + selector + fwd), beside the CPU
    oracle on the same bf16 input (all 8 heads, all host threads)."""
    T, H, D, B, kk = 4096, 8, 64, 64, 16
    cu = np.array([0, T], np.int32)
    lay = ops.VarlenLayout.build(cu, B, device=dev)
    rng = np.random.default_rng(CFG["seed"] + 1)
    qn, kn, vn = (_bf16_np(rng, (T, H, D)) for _ in range(3))
    to_t = lambda a: torch.from_numpy(a.view(np.int16)).to(dev).view(torch.bfloat16)  # noqa: E731
    q, k, v = to_t(qn), to_t(kn), to_t(vn)
    scale = 1.0 / math.sqrt(D)
    kseq = torch.tensor([kk], dtype=torch.int32, device=dev)
    S = ops.block_scores(q, k, lay, scale)
    idx, cnt = ops.topk_select(S, lay, kseq, kk)
    f_fwd, _ = useful_flops(cu, B, idx.cpu().numpy(), cnt.cpu().numpy(), D)
    e, tiles = pair_entries(cu, B, idx.cpu().numpy(), cnt.cpu().numpy())

    def full():
        S_ = ops.block_scores(q, k, lay, scale)
        i_, c_ = ops.topk_select(S_, lay, kseq, kk)
        ops.sparse_attn_fwd(q, k, v, lay, i_, c_, scale)

    t_fwd = time_fn(torch, lambda: ops.sparse_attn_fwd(q, k, v, lay, idx, cnt, scale), max(steps, 20))
    t_full = time_fn(torch, full, max(steps, 20))
    out = {"workload": "C1: one 4096-token sequence, 8 heads MHA, d64, B64, keep 0.25 (k=16), forward",
           "useful_gflop": f_fwd / 1e9, "fwd_attn_ms": t_fwd, "fwd_attn_tflops": f_fwd / (t_fwd * 1e-3) / 1e12,
           "scorer_selector_fwd_ms": t_full,
           # the forward kernel runs UMMA tiles of FWD_TILE_M query rows x B keys per pair
           "fwd_tile_m": FWD_TILE_M[B], "executed_over_useful": tiles * FWD_TILE_M[B] * B / e}
    if with_cpu:
        from oracle import device as orc

        threads = orc.set_threads(host_cores())
        cu_np = cu
        sel_i, sel_c = idx.cpu().numpy(), cnt.cpu().numpy()
        t0 = time.perf_counter()
        orc.sparse_attn_fwd(qn, kn, vn, cu_np, B, sel_i, sel_c, scale)
        dt = time.perf_counter() - t0
        out["cpu_oracle"] = {"fwd_attn_ms": dt * 1e3, "cores": threads, "kind": "port",
                             "sample": "the full C1 forward (all 8 heads), same bf16 input and selection"}
    return out


def main():
    if os.environ.get("SB_HANG_DUMP"):  # debug: dump every thread's Python stack, then exit
        import faulthandler

        faulthandler.dump_traceback_later(int(os.environ["SB_HANG_DUMP"]), exit=True)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=["c2", "c3"],
                    help="c3 (default, every N): 40/60 32K/2K global batch, SAB plan + closed-loop per-layer DST "
                         "across ranks; c2: the one-layer 32K packed micro-batch")
    ap.add_argument("--layers", type=int, default=36, help="c3: layers per step")
    ap.add_argument("--grid", default="dense", choices=["dense", "default"],
                    help="c3 DST budget grid: dense 1..256 (SURVEY 7.3(5), the 1.05x balance target) or the "
                         "reference's default 16 points")
    ap.add_argument("--bwd", default="two-pass", choices=["fused", "two-pass"],
                    help="backward: the bit-deterministic two-pass (default) or the opt-in fused single pass")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the N=1 C1 / C2 / C5 sub-records")
    ap.add_argument("--ref-budget-s", type=float, default=150.0,
                    help="--impl reference: wall-clock budget for the CPU arm (>= 1 warm-up + 1 timed step)")
    ap.add_argument("--profile-only", action="store_true", help="2 plain steps then exit (for ncu)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    # The host only enqueues kernels here: keep OpenMP worker threads from spinning on the cores
    # the launching thread needs (host stalls mid-enqueue idle the GPU inside the timed window).
    os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")

    import torch
    import torch.distributed as dist

    from paper_2604_13847_b200 import dp, ops, synth

    if os.environ.get("SB_OPS_TIMING"):  # debug: host time of every ops call, slow ones to stderr
        import functools

        def _timed(name, fn):
            @functools.wraps(fn)
            def w(*a, **kw):
                h0 = time.perf_counter()
                r = fn(*a, **kw)
                dt = (time.perf_counter() - h0) * 1e3
                if dt > 3.0:
                    shp = [tuple(x) if isinstance(x, (tuple, list)) else getattr(x, "shape", x) for x in a[:2]]
                    print(f"slow host call {name}: {dt:.1f} ms args {shp} {kw.get('dtype', '')}", file=sys.stderr)
                return r
            return w

        for _n in ("topk_select", "sparse_attn_fwd", "sparse_attn_bwd", "block_scores", "coverage_profile",
                   "block_pool", "_call"):
            setattr(ops, _n, _timed(_n, getattr(ops, _n)))
        torch.empty = _timed("torch.empty", torch.empty)
        torch.empty_like = _timed("torch.empty_like", torch.empty_like)

    torch.cuda.set_device(local_rank)
    torch.set_num_threads(1)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    H, D, B = CFG["heads"], CFG["head_dim"], CFG["block"]
    stream = torch.cuda.current_stream()
    burst, sustained, sustained_mhz, hbm_peak, peak_src = peaks()

    runner = None
    if args.workload == "c2":
        cu, k_seq = c2_workload(rank)
        config = {"workload": C2_LABEL, "seqs_rank0": int(len(cu) - 1)}
        T = int(cu[-1])
        lay = ops.VarlenLayout.build(cu, B, device=dev)
        g = torch.Generator(device=dev).manual_seed(CFG["seed"] + rank)
        q, k, v, do = (torch.randn((T, H, D), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
        scale = 1.0 / math.sqrt(D)
        kseq_d = torch.from_numpy(k_seq).to(dev)
        k_max = int(k_seq.max())
        grid = torch.tensor([1, 2, 3, 4, 6, 8, 10, 12, 16, 20, 24, 32, 40, 48, 56, 64], dtype=torch.int32, device=dev)

        def step(mark=None, bufs=None):
            q_, k_, v_, do_ = bufs if bufs is not None else (q, k, v, do)
            if mark:
                mark("start")
            S = ops.block_scores(q_, k_, lay, scale)
            prof = ops.coverage_profile(S, lay)
            ops.coverage_at_grid(prof, lay, grid)
            idx, cnt = ops.topk_select(S, lay, kseq_d, k_max)
            if mark:
                mark("decided")
            o, lse = ops.sparse_attn_fwd(q_, k_, v_, lay, idx, cnt, scale)
            if mark:
                mark("fwd")
            dq, dk, dv = ops.sparse_attn_bwd(q_, k_, v_, o, do_, lse, lay, idx, cnt, scale)
            if mark:
                mark("bwd")
            return [(idx, cnt, o, (dq, dk, dv))]

        busy_of = None
    else:
        lengths_all, routing_all = c3_global_batch(world, CFG["seed"], args.layers, sorted_=False)
        table, table_src = cost_table()
        bins = dp.assign_rank_batches(lengths_all, world, 5, "sab", table=table)
        ids = list(bins[rank][0])
        mine = [int(lengths_all[i]) for i in ids]
        cu = np.concatenate([[0], np.cumsum(mine)]).astype(np.int32)
        T = int(cu[-1])
        lay = ops.VarlenLayout.build(cu, B, device=dev)
        q, k, v, do = synth.planted_qkv(mine, [routing_all[i][0] for i in ids], H, H, D, B, seed=CFG["seed"] + rank,
                                        device=dev)
        layer_scales = synth.layer_scales(args.layers, CFG["seed"])
        dst_cfg = dp.DstSettings()
        if args.grid == "dense":
            dst_cfg.budget_grid = list(range(1, 257))
        runner = dp.DPStep(dp.RankBatch(np.asarray(mine), ids, lay), q, k, v, do, layer_scales, table, dst_cfg,
                           rank=rank, world=world, fused_bwd=args.bwd == "fused")
        config = {"workload": c3_label(world, args.layers, table_src), "dst_grid": args.grid, "bwd": args.bwd,
                  "tokens_per_rank": [int(sum(int(lengths_all[i]) for i in b[0])) for b in bins],
                  "members_rank0": [int(lengths_all[i]) for i in bins[0][0]]}

        def step(mark=None, bufs=None):
            if bufs is not None:
                runner.q, runner.k, runner.v, runner.do = bufs
            if mark:
                mark("start")
            return runner.run(backward=True, mark=mark)

        def busy_of():
            return sum(a.elapsed_time(b) for a, b in runner.last["busy"])

    outs = step()
    torch.cuda.synchronize()
    outs_k_final = np.array(runner.last["k_final"], copy=True) if runner is not None else None

    def step_flops(outs_):
        ff = fb = 0.0
        for idx, cnt, *_ in outs_:
            a, b_ = useful_flops(cu, B, idx.cpu().numpy(), cnt.cpu().numpy(), D, hq=H)
            ff, fb = ff + a, fb + b_
        return ff, fb

    if args.profile_only:
        step()
        torch.cuda.synchronize()
        print("profile-only: 2 steps done")
        return
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- device-timed region: inputs resident in HBM (Q/K/V/dO >= 256 MB each, larger than L2)
    markers = [Marker(torch, stream) for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ops.launch_count()
    step_outs, busy_pairs = [], []
    # Python's cyclic GC can pause the host for tens of ms while it enqueues a layer; the GPU
    # then drains its queue and idles inside the timed window (seen as erratic fwd phases).
    gc.collect()
    gc.disable()
    with ClockSampler(local_rank) as clk:
        time.sleep(0.3)  # let nvidia-smi start sampling
        t0.record(stream)
        for s_ in range(args.steps):
            # Retain nothing on the GPU across timed steps: growing the caching allocator here would
            # cudaMalloc mid-step (implicitly synchronising, the GPU then idles). Every step plans
            # the same inputs, so its selections equal the pre-timed step's; the keep counts are
            # kept (host ints) to check exactly that.
            step(markers[s_])
            if runner is not None:
                step_outs.append(np.array(runner.last["k_final"], copy=True))
            if runner is not None:
                busy_pairs.append(list(runner.last["busy"]))
        t1.record(stream)
        torch.cuda.synchronize()
        gc.enable()
        launches = ops.launch_count() - launches0
        # Keep the GPU under the same load (untimed) so the sampler sees >= ~1 s of it.
        t_load = time.perf_counter()
        while time.perf_counter() - t_load < 1.2:
            step()
            torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    # Useful work per timed step: the pre-timed step's selections (identical keep counts checked).
    f_fwd, f_bwd = step_flops(outs)
    if runner is not None:
        k0 = np.array(outs_k_final)
        if not all(np.array_equal(k0, kf) for kf in step_outs):
            raise RuntimeError("timed steps decided different keep counts than the step the FLOPs were counted on")
    f_step = f_fwd + f_bwd
    if busy_pairs:
        busy = [sum(a.elapsed_time(b) for a, b in bp) for bp in busy_pairs]
    else:
        busy = [m.marks[0][1].elapsed_time(m.marks[-1][1]) for m in markers]
    phase = {}
    for m in markers:
        for k_, v_ in m.durations().items():
            phase[k_] = phase.get(k_, 0.0) + v_ / args.steps
    sel_ms, fwd_ms, bwd_ms = phase.get("decided", 0.0), phase.get("fwd", 0.0), phase.get("bwd", 0.0)
    if os.environ.get("SB_PHASE_DUMP"):  # debug: every step's per-layer phase times
        free_b, total_b = torch.cuda.mem_get_info()
        print(f"memory: allocated {torch.cuda.memory_allocated() / 2**30:.1f} GiB reserved "
              f"{torch.cuda.memory_reserved() / 2**30:.1f} GiB free {free_b / 2**30:.1f} / {total_b / 2**30:.1f} GiB; "
              f"allocator stats: {dict((k, v) for k, v in torch.cuda.memory_stats().items() if 'num_alloc_retries' in k or 'num_device_alloc' in k or 'num_device_free' in k or 'num_sync_all_streams' in k)}",
              file=sys.stderr)
        for si, m in enumerate(markers):
            seg = [(tb, a.elapsed_time(b), 1e3 * (hb - ha))
                   for ((ta, a), ha), ((tb, b), hb) in zip(zip(m.marks, m.host), zip(m.marks[1:], m.host[1:]))]
            print(f"step {si}: " + " ".join(f"{t[0]}{d:.2f}/{hh:.2f}" for t, d, hh in seg), file=sys.stderr)
    if world > 1:
        dist.barrier()

    # ---- N > 1 (C3): the same step with the step-end gradient all-reduce of SURVEY 8(e), one
    # stand-in bucket per layer (the layer's output-projection gradient, H*D x H*D bf16),
    # all-reduced on NCCL's stream overlapping the following layers. Reported beside the main
    # number, which (like the metric's max/mean) is measured before this barrier.
    grad_ar = None
    if world > 1 and runner is not None:
        hidden = H * D
        buckets = [torch.zeros((hidden, hidden), dtype=torch.bfloat16, device=dev) for _ in range(args.layers)]
        runner.run(backward=True, grad_buckets=buckets)  # warm the NCCL path
        torch.cuda.synchronize()
        dist.barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ar_steps = max(1, min(args.steps, 3))
        a0.record(stream)
        for _ in range(ar_steps):
            runner.run(backward=True, grad_buckets=buckets)
        a1.record(stream)
        torch.cuda.synchronize()
        ar_ms = torch.tensor([a0.elapsed_time(a1) / ar_steps], dtype=torch.float64, device=dev)
        dist.all_reduce(ar_ms, op=dist.ReduceOp.MAX)
        grad_ar = {"stand_in": f"{args.layers} x [{hidden}, {hidden}] bf16 (output-projection gradient per layer)",
                   "bytes_per_step": int(args.layers * hidden * hidden * 2),
                   "ms_per_step_with_allreduce": float(ar_ms[0]),
                   "overlap": "per-layer async NCCL all_reduce issued after that layer's backward"}

    # ---- end-to-end region: every step copies its inputs in from pinned host memory and reads its
    # results (O, dQ, dK, dV of the last layer) back, through the same public calls. Double
    # buffered on separate copy streams: step i's H2D overlaps step i-1's kernels and step i-2's
    # D2H, as a training loop's data pipeline would.
    hin = [tuple(t.cpu().pin_memory() for t in (q, k, v, do)) for _ in range(2)]
    hout = [tuple(torch.empty(t.shape, dtype=torch.bfloat16).pin_memory() for t in (q, q, k, v)) for _ in range(2)]
    dbuf = [(q, k, v, do), tuple(torch.empty_like(t) for t in (q, k, v, do))]
    h2d, d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    e2e_steps = max(2, args.steps)  # the same K as the device-timed loop

    def pipelined(n):
        in_ready = [torch.cuda.Event() for _ in range(n)]
        done = [torch.cuda.Event() for _ in range(n)]
        h2d.wait_stream(stream)
        d2h.wait_stream(stream)
        keep = []
        pending = []  # (step done event, host buffer index, device outputs) not yet copied out

        def flush():
            # Step i-1's outputs leave once step i has made its host decision: enqueued earlier, the
            # 1.3 GB D2H held the copy engine ahead of step i's small profile D2H, and the host
            # decision -- hence every layer launch of step i -- waited ~20 ms behind it.
            while pending:
                ev, hb, outs = pending.pop(0)
                with torch.cuda.stream(d2h):
                    d2h.wait_event(ev)  # (in-order stream: the earlier copy into hout[hb] finished first)
                    for dst, src in zip(hout[hb], outs):
                        src.record_stream(d2h)
                        dst.copy_(src, non_blocking=True)

        for i in range(n):
            b = i % 2
            with torch.cuda.stream(h2d):
                if i >= 2:
                    h2d.wait_event(done[i - 2])  # device buffer b free again
                for dst, src in zip(dbuf[b], hin[b]):
                    dst.copy_(src, non_blocking=True)
                in_ready[i].record(h2d)
            stream.wait_event(in_ready[i])
            res = step(bufs=dbuf[b], mark=lambda tag: flush() if tag == "decided" else None)
            done[i].record(stream)
            _, _, o, (dq, dk, dv) = res[-1]
            pending.append((done[i], b, (o, dq, dk, dv)))
            keep = (keep + [res])[-2:]
        flush()
        stream.wait_stream(d2h)
        if runner is not None:
            runner.q, runner.k, runner.v, runner.do = q, k, v, do

    pipelined(e2e_steps)  # warm: the caching allocator sizes its pool for the in-flight steps
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    gc.collect()
    gc.disable()
    e0.record(stream)
    pipelined(e2e_steps)
    e1.record(stream)
    torch.cuda.synchronize()
    gc.enable()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    nbytes_in = sum(t.numel() * 2 for t in (q, k, v, do))
    nbytes_out = sum(t.numel() * 2 for t in (q, q, k, v))  # O, dQ, dK, dV

    # ---- max over ranks, whole-job aggregates; busy-time balance per step (Eq. 9)
    vals = torch.tensor([ms, e2e_ms, f_step] + busy, dtype=torch.float64, device=dev)
    if world > 1:
        per_rank = [torch.zeros_like(vals) for _ in range(world)]
        dist.all_gather(per_rank, vals)
        pr = torch.stack(per_rank).cpu().numpy()
    else:
        pr = vals.cpu().numpy()[None]
    ms_max, e2e_max, flops_all = float(pr[:, 0].max()), float(pr[:, 1].max()), float(pr[:, 2].sum())
    busy_mat = pr[:, 3:]  # [rank, step]
    step_ratio = busy_mat.max(axis=0) / busy_mat.mean(axis=0)
    busy_rank = busy_mat.mean(axis=1)

    if rank == 0:
        b_tflops = f_bwd / (bwd_ms * 1e-3) / 1e12 if bwd_ms else 0.0
        f_tflops = f_fwd / (fwd_ms * 1e-3) / 1e12 if fwd_ms else 0.0
        if bwd_ms >= fwd_ms:
            dom, dom_tf = "sb_sparse_attn_bwd (prep + transpose + dK/dV + dQ passes)", b_tflops
        else:
            dom, dom_tf = "sb_sparse_attn_fwd", f_tflops
        traffic, traffic_note = None, None
        prof_path = os.path.join(ROOT, "profiles", "dram_bytes_per_launch.json")
        if os.path.exists(prof_path):
            try:
                rec = json.load(open(prof_path)).get(args.workload, {})
                traffic, traffic_note = rec.get("dominant_traffic_bytes"), rec.get("note")
            except Exception:
                traffic = None
        clocks = clk.summary()
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(cu, np.maximum(1, (np.diff(cu) + B - 1) // B // 8))
        subs = None
        if world == 1 and not args.no_sub:
            subs = {"c2": sub_c2(torch, ops, dev, 5, burst), "c5_gqa_keep0.1": sub_c5(torch, ops, dev, 3, burst),
                    "c1": sub_c1(torch, ops, dev, 20, with_cpu=not args.no_cpu_baseline)}
        value = flops_all / (ms_max * 1e-3) / 1e12
        config.update({"tokens_rank0": T, "l2": "inputs 256 MB+ each > L2, no flush", "parallelism": f"dp{world}",
                       "layers": args.layers if runner is not None else 1})
        k_fin = runner.last.get("k_final") if runner is not None else None
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (planted block routing)" if runner else "synthetic",
            "config": config,
            "breakdown_ms_rank0": {"scorer_profile_exchange_dst": sel_ms, "selector_fwd": fwd_ms, "bwd": bwd_ms},
            "busy_ms_per_rank": [float(x) for x in busy_rank],
            "max_over_mean": float(busy_rank.max() / busy_rank.mean()),
            "max_over_mean_worst_step": float(step_ratio.max()),
            "balance_note": "per-rank busy time = CUDA events around the rank's own kernels (scorer pre-pass, "
                            "layer loop), excluding the all-gather wait and host DST",
            "per_rank_ms_wall": [float(x) for x in pr[:, 0]],
            "per_rank_useful_tflop": [float(x) / 1e12 for x in pr[:, 2]],
            "useful_tflop_per_step": flops_all / 1e12,
            "fwd_tflops_rank0": f_tflops, "bwd_tflops_rank0": b_tflops,
            "k_final_rank0": [int(x) for x in k_fin[0]] if k_fin is not None else None,
            "roofline": {"bound": "tensor", "kernel": dom, "achieved": dom_tf, "peak": burst, "unit": "TFLOP/s",
                         "frac": dom_tf / burst, "traffic": traffic, "traffic_note": traffic_note,
                         "peak_source": f"{peak_src} burst bf16 dense (MEASURED_PEAKS.json)",
                         "peak_sustained": sustained, "frac_sustained": dom_tf / sustained,
                         "sustained_measured_at_mhz": sustained_mhz,
                         "bench_sm_mhz": (clocks or {}).get("sm_mhz"),
                         "achieved_def": "useful selected-block FLOPs of the phase (10*d*sum e_ij bwd, 4*d*sum "
                                         "e_ij fwd, per q head) / its CUDA-event time on the launching stream"},
            "e2e": {"value": flops_all / (e2e_max * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": e2e_max,
                    "h2d_bytes_per_step": nbytes_in, "d2h_bytes_per_step": nbytes_out,
                    "steps": e2e_steps,
                    "note": "every step: pinned H2D of its Q,K,V,dO and D2H of its O,dQ,dK,dV (last layer), "
                            "double-buffered on two copy streams overlapping the neighbouring steps' kernels (a step's D2H is "
                            "enqueued once the next step has made its host decision); "
                            "the first step's H2D and the last step's D2H (pipeline fill / drain) are inside "
                            "the timed region"},
            "gpu_launches": int(launches),
            "grad_allreduce": grad_ar,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "sub": subs,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def cpu_baseline(cu, k_seq):
    """Oracle port (fp64 C, all host threads) on a bounded sample: q head 0 of 32, one layer fwd+bwd."""
    from oracle import device as orc

    T, D, B = int(cu[-1]), CFG["head_dim"], CFG["block"]
    rng = np.random.default_rng(1)
    q, k, v, do = (_bf16_np(rng, (T, 1, D)) for _ in range(4))
    threads = orc.set_threads(host_cores())
    _, tri = orc.layout(cu, B)
    S = rng.standard_normal((1, int(tri[-1]))).astype(np.float32)
    idx, cnt = orc.topk_select(S, cu, B, k_seq, int(k_seq.max()))
    scale = 1.0 / math.sqrt(D)
    t0 = time.perf_counter()
    o, lse = orc.sparse_attn_fwd(q, k, v, cu, B, idx, cnt, scale)
    orc.sparse_attn_bwd(q, k, v, o, do, lse, cu, B, idx, cnt, scale)
    dt = time.perf_counter() - t0
    f, b = useful_flops(cu, B, idx, cnt, D)
    return {"value": (f + b) / dt / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": "port",
            "sample": f"q head 0 of 32 of rank 0's micro-batch, one layer fwd+bwd at keep ~1/8, {dt:.1f} s",
            "seconds": dt}


if __name__ == "__main__":
    main()
