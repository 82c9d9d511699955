#!/usr/bin/env python
"""Benchmark of the SparseBalance hot path on B200.

Workload (BASELINE.json configs[1], "C2"): per rank one packed varlen micro-batch of 32768
tokens (cu_seqlens) drawn from the reference workload generator (40% 32K / 60% 2K bimodal,
proj/core/src/workload.cpp:239-271, seeded by rank), 32 heads, head_dim 128, block 128,
per-sequence keep ratios ~ U[0.05, 0.5]; synthetic bf16 Q/K/V/dO ~ N(0,1).

One step = the whole hot path over the micro-batch: block scorer (K1+K2), coverage profile +
coverage-at-grid (K4), top-k selector (K3), sparse attention forward (K5) and backward (K6),
and (N > 1) the per-rank workload-estimate allgather the tuner needs. Inputs (256 MB each) are
larger than the 126 MB L2, so no explicit flush between steps.

value = useful TFLOP/s of the whole job = sum over ranks of useful selected-block FLOPs
(14 * d * sum e_ij per q head: 4 fwd + 10 bwd) / max-over-ranks step time.
"""
from __future__ import annotations

import argparse
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


def peaks():
    """(bf16 TF/s, HBM GB/s, source). The roofline kernel runs inside a multi-millisecond step
    repeated back to back, so the SUSTAINED bf16 figure of MEASURED_PEAKS.json is the
    denominator (the burst figure applies to a kernel timed alone)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        if "bf16_tflops_sustained" in p:
            return float(p["bf16_tflops_sustained"]), float(p["hbm_gbs"]), "measured sustained"
        return float(p["bf16_tflops"]), float(p["hbm_gbs"]), "measured burst"
    except Exception:
        return 1590.0, 6650.0, "fallback"


def workload(rank: int):
    """C2 micro-batch of 32768 tokens: the SURVEY.md section 8(d) example composition
    [12288, 8192, 4096, 2048 x 4] packed with cu_seqlens, and per-sequence keep ratios
    U[0.05, 0.5] seeded by rank (so ranks carry different sparse work)."""
    lens = [12288, 8192, 4096, 2048, 2048, 2048, 2048]
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    rng = np.random.default_rng(CFG["seed"] + 7919 * rank)
    nb = (np.array(lens) + CFG["block"] - 1) // CFG["block"]
    keep = rng.uniform(CFG["keep_lo"], CFG["keep_hi"], size=len(lens))
    k_seq = np.maximum(1, np.ceil(keep * nb)).astype(np.int32)
    return cu, k_seq


def useful_flops(cu, B, idx, cnt, d):
    """(fwd, bwd) useful FLOPs: 4*d*sum(e_ij) and 10*d*sum(e_ij) over q heads, where e_ij is the
    number of unmasked score entries of pair (i, j): r_i * c_j off the diagonal and
    r_i (r_i + 1) / 2 on the causal diagonal."""
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
    return 4.0 * d * float(e), 10.0 * d * float(e)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = f"/tmp/sb_clocks_{os.getpid()}.csv"

    def __enter__(self):
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


C2_WORKLOAD = ("C2: 32K-token packed varlen micro-batch per rank ([12288, 8192, 4096, 2048x4], SURVEY 8d), "
               "32 heads MHA, d128, B128, per-sequence keep U[0.05,0.5], scorer+profile+selector+fwd+bwd")


def c3_workload(world: int, layers: int, table_src: str) -> str:
    """The C3 workload label, shared by our arm and the CPU reference arm."""
    return (f"C3: 40% 32K / 60% 2K global batch (reference generator, seed 42, gbs={5 * world}), "
            f"SAB plan mbs=5 (one packed micro-batch per rank), {layers} layers, per-layer DST "
            f"(Mean anchor, p=0.1, global scope, coverage base, {table_src}) on the generator's "
            "routing profiles (all-gathered), GPU block scores for selection, 32 heads MHA, d128, B128, "
            "scorer+allgather+DST+selector+fwd+bwd")


def cost_table_source() -> str:
    tpath = os.path.join(ROOT, "profiles", "b200_cost_table_h32_d128_b128.csv")
    return "GPU-measured cost table" if os.path.exists(tpath) else "synthetic cost table"


def host_cores() -> int:
    """Host threads this process may use (affinity / cgroup aware). torchrun sets
    OMP_NUM_THREADS=1 per rank; the CPU arm overrides that to use the whole host."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def c3_rank0_layer0(world, layers):
    """Rank 0's packed micro-batch of the C3 global batch (SAB plan on the same cost table as the
    GPU arm) and its layer-0 DST keep count per sequence (the pooled host DST, bit-identical to
    what every GPU rank decides)."""
    from paper_2604_13847_b200 import dp
    from paper_2604_13847_b200.host import api

    lengths_all, profiles_all = c3_global_batch(world, CFG["seed"], layers)
    tpath = os.path.join(ROOT, "profiles", "b200_cost_table_h32_d128_b128.csv")
    table = api().load_table(tpath)[0] if os.path.exists(tpath) else api().synthesize_table(block_size=CFG["block"])
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


def run_reference_arm(args, rank, world):
    """--impl reference: the reference has no CPU attention; the CPU arm is this repo's
    oracle port of the path (oracle/sb_oracle.c, fp64, all host threads) on a bounded sample of
    the same workload (q head 0 of rank 0's micro-batch: 1/32 of a step), scaled per unit."""
    if rank != 0:
        return
    from oracle import device as orc

    c3 = world > 1 or args.workload == "c3"
    if c3:
        cu, k_seq = c3_rank0_layer0(world, args.layers)
    else:
        cu, k_seq = workload(0)
    T, D, B = int(cu[-1]), CFG["head_dim"], CFG["block"]
    rng = np.random.default_rng(1)

    def bf(shape):
        return (rng.standard_normal(shape).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)

    q, k, v, do = bf((T, 1, D)), bf((T, 1, D)), bf((T, 1, D)), bf((T, 1, D))
    threads = orc.set_threads(host_cores())
    blk, tri = orc.layout(cu, B)
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
    workload_txt = c3_workload(world, args.layers, cost_table_source()) if c3 else C2_WORKLOAD
    line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": workload_txt, "sample": "CPU port: " + sample, "warmup_run": warm_done,
                       "steps_timed": len(times), "budget_s": budget_s},
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


class Marker:
    """Records CUDA events at tagged phase boundaries inside a step (on the launching stream)."""

    def __init__(self, torch, stream):
        self.torch, self.stream = torch, stream
        self.marks = []

    def __call__(self, tag):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record(self.stream)
        self.marks.append((tag, e))

    def durations(self):
        """ms per tag: time from the previous mark to this one, summed per tag."""
        out = {}
        for (_, a), (tag, b) in zip(self.marks, self.marks[1:]):
            out[tag] = out.get(tag, 0.0) + a.elapsed_time(b)
        return out


def c3_global_batch(world: int, seed: int, layers: int = 1):
    """C3: the reference workload generator's 40% 32K / 60% 2K bimodal mix
    (distribution={bimodal, short_weight 0.6, ln 2048 / ln 32768, sigma 0}, default
    concentration), gbs = 5 * dp -> (lengths, per-sample per-layer routing profiles)."""
    from paper_2604_13847_b200.host import api

    dist_spec = dict(short_weight=0.6, short_log_mean=float(np.log(2048)), short_log_sigma=0.0,
                     long_log_mean=float(np.log(32768)), long_log_sigma=0.0)
    lengths, profiles = api().generate_samples(5 * world, layers, CFG["block"], seed=seed, dist=dist_spec)
    return np.asarray(lengths), profiles


def main():
    if os.environ.get("SB_HANG_DUMP"):  # debug: dump every thread's Python stack, then exit
        import faulthandler

        faulthandler.dump_traceback_later(int(os.environ["SB_HANG_DUMP"]), exit=True)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=["c2", "c3"],
                    help="c2 (default at 1 GPU): 32K packed, per-sequence keeps; c3 (default at >1 GPU): 40/60 "
                         "32K/2K global batch, SAB plan + per-layer DST across ranks")
    ap.add_argument("--layers", type=int, default=36, help="c3: layers per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget-s", type=float, default=150.0,
                    help="--impl reference: wall-clock budget for the CPU arm (>= 1 warm-up + 1 timed step)")
    ap.add_argument("--profile-only", action="store_true", help="2 plain steps then exit (for ncu)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    workload_kind = args.workload or ("c2" if world == 1 else "c3")
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_2604_13847_b200 import dp, ops
    from paper_2604_13847_b200.host import api

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    H, D, B = CFG["heads"], CFG["head_dim"], CFG["block"]
    stream = torch.cuda.current_stream()

    if workload_kind == "c2":
        cu, k_seq = workload(rank)
        config = {"workload": C2_WORKLOAD, "seqs_rank0": int(len(cu) - 1)}
    else:
        lengths_all, profiles_all = c3_global_batch(world, CFG["seed"], args.layers)
        # GPU-measured cost table (profiler.py, committed under profiles/) when present, as SURVEY
        # 8(f) item 1 intends; the reference's synthetic table otherwise.
        tpath = os.path.join(ROOT, "profiles", "b200_cost_table_h32_d128_b128.csv")
        table = api().load_table(tpath)[0] if os.path.exists(tpath) else api().synthesize_table(block_size=B)
        table_src = cost_table_source()
        bins = dp.assign_rank_batches(lengths_all, world, 5, "sab", table=table)
        mine = [int(lengths_all[i]) for i in bins[rank][0]]
        cu = np.concatenate([[0], np.cumsum(mine)]).astype(np.int32)
        k_seq = None
        config = {"workload": c3_workload(world, args.layers, table_src),
                  "tokens_per_rank": [int(x) for x in np.array([sum(int(lengths_all[i]) for i in b[0]) for b in bins])]}
    T = int(cu[-1])
    lay = ops.VarlenLayout.build(cu, B, device=dev)
    g = torch.Generator(device=dev).manual_seed(CFG["seed"] + rank)
    q, k, v, do = (torch.randn((T, H, D), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
    scale = 1.0 / math.sqrt(D)

    if workload_kind == "c2":
        kseq_d = torch.from_numpy(k_seq).to(dev)
        k_max = int(k_seq.max())
        grid = torch.tensor([1, 2, 3, 4, 6, 8, 10, 12, 16, 20, 24, 32, 40, 48, 56, 64], dtype=torch.int32,
                            device=dev)

        def step(mark=None, bufs=None):
            q_, k_, v_, do_ = bufs if bufs is not None else (q, k, v, do)
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
    else:
        rng = np.random.default_rng(CFG["seed"])
        layer_scales = np.exp(rng.uniform(-0.5, 1.0, size=args.layers))  # per-layer softmax temperature
        routing = [[profiles_all[i][l] for i in bins[rank][0]] for l in range(args.layers)]
        runner = dp.DPStep(dp.RankBatch(np.diff(cu), list(bins[rank][0]), lay), q, k, v, do, layer_scales, table,
                           dp.DstSettings(), rank=rank, world=world, width=int(np.ceil(32768 / B)),
                           routing_profiles=routing)

        def step(mark=None, bufs=None):
            if bufs is not None:
                runner.q, runner.k, runner.v, runner.do = bufs
            return runner.run(backward=True, mark=mark)

    outs = step()
    torch.cuda.synchronize()
    f_fwd = f_bwd = 0.0
    for idx, cnt, *_ in outs:
        a, b_ = useful_flops(cu, B, idx.cpu().numpy(), cnt.cpu().numpy(), D)
        f_fwd, f_bwd = f_fwd + a, f_bwd + b_
    f_step = f_fwd + f_bwd
    if args.profile_only:
        step()
        torch.cuda.synchronize()
        print("profile-only: 2 steps done")
        return
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- device-timed region: inputs resident in HBM (each >= 256 MB, larger than L2)
    markers = [Marker(torch, stream) for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ops.launch_count()
    with ClockSampler(local_rank) as clk:
        time.sleep(0.3)  # let nvidia-smi start sampling
        t0.record(stream)
        for s_ in range(args.steps):
            markers[s_]("start")
            step(markers[s_])
        t1.record(stream)
        torch.cuda.synchronize()
        launches = ops.launch_count() - launches0
        # Keep the GPU under the same load (untimed) so the sampler sees >= ~1 s of it.
        t_load = time.perf_counter()
        while time.perf_counter() - t_load < 1.2:
            step()
            torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = t0.elapsed_time(t1) / args.steps

    # ---- N > 1 (C3): the same step with the step-end gradient all-reduce of SURVEY 8(e),
    # one stand-in bucket per layer (the layer's output-projection gradient, H*D x H*D bf16),
    # all-reduced on NCCL's stream overlapping the following layers. Reported beside the main
    # number, which (like the metric's max/mean) is measured before this barrier.
    grad_ar = None
    if world > 1 and workload_kind == "c3":
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
    phase = {}
    for m in markers:
        for k_, v_ in m.durations().items():
            phase[k_] = phase.get(k_, 0.0) + v_ / args.steps
    sel_ms, fwd_ms, bwd_ms = phase.get("decided", 0.0), phase.get("fwd", 0.0), phase.get("bwd", 0.0)

    # ---- end-to-end region: every step copies its inputs in from pinned host memory and reads its
    # results (O, dQ, dK, dV of the last layer) back, through the same public calls. Double
    # buffered on separate copy streams: step i's H2D overlaps step i-1's kernels and step i-2's
    # D2H, as a training loop's data pipeline would.
    hin = [tuple(t.cpu().pin_memory() for t in (q, k, v, do)) for _ in range(2)]
    hout = [tuple(torch.empty((T, H, D), dtype=torch.bfloat16).pin_memory() for _ in range(4)) for _ in range(2)]
    dbuf = [(q, k, v, do), tuple(torch.empty_like(t) for t in (q, k, v, do))]
    h2d, d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    e2e_steps = max(2, min(args.steps, 6))

    def pipelined(n):
        in_ready = [torch.cuda.Event() for _ in range(n)]
        done = [torch.cuda.Event() for _ in range(n)]
        h2d.wait_stream(stream)
        d2h.wait_stream(stream)
        keep = []
        for i in range(n):
            b = i % 2
            with torch.cuda.stream(h2d):
                if i >= 2:
                    h2d.wait_event(done[i - 2])  # device buffer b free again
                for dst, src in zip(dbuf[b], hin[b]):
                    dst.copy_(src, non_blocking=True)
                in_ready[i].record(h2d)
            stream.wait_event(in_ready[i])
            res = step(bufs=dbuf[b])
            done[i].record(stream)
            _, _, o, (dq, dk, dv) = res[-1]
            with torch.cuda.stream(d2h):
                d2h.wait_event(done[i])  # (in-order stream: step i-2's copy into hout[b] finished first)
                for dst, src in zip(hout[b], (o, dq, dk, dv)):
                    src.record_stream(d2h)
                    dst.copy_(src, non_blocking=True)
            keep = (keep + [res])[-2:]
        stream.wait_stream(d2h)

    pipelined(e2e_steps)  # warm: the caching allocator sizes its pool for the in-flight steps
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    pipelined(e2e_steps)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    nbytes = 4 * T * H * D * 2

    # ---- max over ranks, whole-job aggregates
    vals = torch.tensor([ms, e2e_ms, f_step], dtype=torch.float64, device=dev)
    if world > 1:
        mx = vals.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        tot = vals.clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        ms_max, e2e_max, flops_all = float(mx[0]), float(mx[1]), float(tot[2])
        per_rank = [torch.zeros(3, dtype=torch.float64, device=dev) for _ in range(world)]
        dist.all_gather(per_rank, vals)
        per_rank_ms = [float(x[0]) for x in per_rank]
        per_rank_tflop = [float(x[2]) / 1e12 for x in per_rank]
    else:
        ms_max, e2e_max, flops_all, per_rank_ms, per_rank_tflop = ms, e2e_ms, f_step, [ms], [f_step / 1e12]

    if rank == 0:
        bf16_peak, hbm_peak, peak_kind = peaks()
        if bwd_ms >= fwd_ms:
            dom, dom_ms, dom_flops = "sb_sparse_attn_bwd (dkv+dq passes)", bwd_ms, f_bwd
        else:
            dom, dom_ms, dom_flops = "sb_sparse_attn_fwd", fwd_ms, f_fwd
        achieved = dom_flops / (dom_ms * 1e-3) / 1e12
        traffic = None
        prof_path = os.path.join(ROOT, "profiles", "dram_bytes_per_launch.json")
        if os.path.exists(prof_path):
            try:
                traffic = json.load(open(prof_path)).get(workload_kind, {}).get("dominant_traffic_bytes")
            except Exception:
                traffic = None
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(cu, k_seq if k_seq is not None else np.maximum(1, (np.diff(cu) + B - 1) // B // 8))
        value = flops_all / (ms_max * 1e-3) / 1e12
        config.update({"tokens_per_rank" if workload_kind == "c2" else "tokens_rank0": T,
                       "l2": "inputs 256 MB+ each > L2, no flush", "parallelism": f"dp{world}"})
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic", "config": config,
            "breakdown_ms_rank0": {"scorer_profile_exchange_dst_selector": sel_ms, "fwd": fwd_ms, "bwd": bwd_ms},
            "per_rank_ms": per_rank_ms, "per_rank_useful_tflop": per_rank_tflop,
            "max_over_mean": ms_max / statistics.mean(per_rank_ms),
            "useful_tflop_per_step": flops_all / 1e12,
            "fwd_tflops_rank0": f_fwd / (fwd_ms * 1e-3) / 1e12 if fwd_ms else None,
            "bwd_tflops_rank0": f_bwd / (bwd_ms * 1e-3) / 1e12 if bwd_ms else None,
            "roofline": {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": bf16_peak,
                         "unit": "TFLOP/s", "frac": achieved / bf16_peak, "traffic": traffic,
                         "peak_source": f"{peak_kind} bf16 dense (MEASURED_PEAKS.json)"},
            "e2e": {"value": flops_all / (e2e_max * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": e2e_max,
                    "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                    "note": "every step: pinned H2D of its Q,K,V,dO and D2H of its O,dQ,dK,dV (last layer), "
                            "double-buffered on two copy streams overlapping the neighbouring steps' kernels"},
            "gpu_launches": int(launches),
            "grad_allreduce": grad_ar,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def cpu_baseline(cu, k_seq):
    """Oracle port (fp64 C, all host threads) on a bounded sample: q head 0 of 32, fwd+bwd."""
    from oracle import device as orc

    T, D, B = int(cu[-1]), CFG["head_dim"], CFG["block"]
    rng = np.random.default_rng(1)

    def bf(shape):
        return (rng.standard_normal(shape).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)

    q, k, v, do = bf((T, 1, D)), bf((T, 1, D)), bf((T, 1, D)), bf((T, 1, D))
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
            "sample": f"q head 0 of 32 (1/32 of the step's attention work), fwd+bwd, {dt:.1f} s",
            "seconds": dt}


if __name__ == "__main__":
    main()
