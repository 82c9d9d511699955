"""Measured data-parallel step driver.

The reference's scenario loop (run_scenarios, proj/core/src/sim.cpp:518-585) draws a global
batch per iteration, plans it (simulate_iteration's decision half, sim.cpp:277-432) and
*simulates* each rank's 1F1B pipeline from a cost table (simulate_pipeline / micro_batch_time,
sim.cpp:88-98, 180-275, 435-476). This driver keeps the first two steps bit-identical
(generate_samples with the reference's seed stream mix_seed(seed, iter), sim.cpp:555-558;
plan_step == simulate_iteration's decisions, checked in tests/test_host_parity.py) and replaces
the third with the real kernels: every rank runs its micro-batches' layers (block scorer ->
top-k selector with the DST keep count of that (micro-batch, layer), clamped per sequence ->
sparse attention fwd -> bwd) timed with CUDA events, and the per-(rank, micro-batch) times are
all-gathered.

The tuner is closed-loop: its routing profiles are not the generator's but the K4 coverage
profiles of the GPU block scores, measured by a scorer pre-pass over every layer on inputs that
carry the generator's routing draws (synth.py), exchanged with one all-reduce, and written per
iteration (gpu_profiles_<it>.npz) so the decisions can be replayed on the host and against the
compiled reference bit for bit (tests/test_driver.py).

It emits the reference's replay files per iteration, so a run can be replayed against the
oracle:
  * iterations CSV with the reference's header and %.6f fields (report.cpp:55-74):
    scenario,iter,iter_ms,imbalance,max_mb_ms,mean_mb_ms,bubble_ms,dst_overhead_ms,
    avg_budget,mean_cov_drop -- iter_ms = max over ranks of the rank's summed micro-batch
    time (pp = 1, so bubble_ms = 0 as in sim.cpp:272), imbalance = max / mean over all
    (rank, micro-batch) totals (sim.cpp:483-485), dst_overhead_ms = host planning wall time;
  * decisions CSV (dst.cpp:171-185) and plan JSON (sab.cpp:312-336) through plan_step.

    python -m torch.distributed.run --nproc-per-node 8 -m paper_2604_13847_b200.driver \\
        --strategy sab_dst --iters 4 --out runs/sab_dst
"""
from __future__ import annotations

import argparse
import copy
import json
import math
import os
import time

import numpy as np
import torch

from . import ops, synth
from . import pp_projection as ppj
from .host import DEFAULT_BUDGET_GRID, ProfileTable, api

MASK64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """rng.cpp:13-18."""
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def mix_seed(seed: int, a: int) -> int:
    """rng.cpp:23-25: the per-iteration seed of run_scenarios (sim.cpp:558)."""
    return splitmix64(splitmix64(seed & MASK64) ^ (a & MASK64))


ITER_HEADER = ("scenario,iter,iter_ms,imbalance,max_mb_ms,mean_mb_ms,bubble_ms,dst_overhead_ms,avg_budget,"
               "mean_cov_drop\n")


def iteration_row(scenario: str, it: int, rec: dict) -> str:
    """One iterations-CSV line exactly as report.cpp:60-70 formats it (fmt6 = %.6f)."""
    vals = [rec[k] for k in ("iter_ms", "imbalance", "max_mb_ms", "mean_mb_ms", "bubble_ms", "dst_overhead_ms",
                             "avg_budget", "mean_cov_drop")]
    return f"{scenario},{it}," + ",".join("%.6f" % float(v) for v in vals) + "\n"


def summarize(mb_ms: list[list[float]]) -> dict:
    """Per-(rank, micro-batch) measured totals -> the ScheduleResult fields (sim.cpp:448-485)."""
    flat = [t for r in mb_ms for t in r]
    mean_all = sum(flat) / len(flat) if flat else 0.0
    max_all = max(flat) if flat else 0.0
    return dict(iter_ms=max((sum(r) for r in mb_ms), default=0.0), max_mb_ms=max_all, mean_mb_ms=mean_all,
                imbalance=max_all / mean_all if mean_all > 0.0 else 1.0, bubble_ms=0.0)


class Driver:
    def __init__(self, strategy="sab_dst", gbs=16, mbs=2, layers=4, block=128, heads=32, kv_heads=32, head_dim=128,
                 seed=42, dist_spec=None, table: ProfileTable | None = None, anchor="mean", threshold_p=0.1,
                 dst_scope="global", base_mode="coverage", varlen_block_size=0, project_pp=0, rank=0, world=1,
                 group=None, device="cuda", dst_grid=None):
        self.h = api()
        self.strategy, self.gbs, self.mbs, self.layers, self.B = strategy, gbs, mbs, layers, block
        self.H, self.Hkv, self.D = heads, kv_heads, head_dim
        self.seed, self.dist_spec = seed, dist_spec
        self.rank, self.world, self.group, self.device = rank, world, group, device
        self.table = table if table is not None else self.h.synthesize_table(block_size=block)
        self.grid = list(self.table.budget_grid) if table is not None else list(DEFAULT_BUDGET_GRID)
        max_len = int((dist_spec or {}).get("max_length", 65536))
        self.est = self.h.make_estimator(self.h.default_bin_edges(max_len), budget_grid=self.grid)
        self.plan_kw = dict(anchor=anchor, threshold_p=threshold_p, dst_scope=dst_scope, base_mode=base_mode,
                            dst_grid=dst_grid,
                            varlen_block_size=varlen_block_size)
        self._buf_T = 0
        self._warm = False
        # PP projection: per-layer fwd / bwd kernel times feed a 1F1B model of
        # `project_pp` stages (pp_projection.py); 0 = off.
        self.project_pp = project_pp
        if project_pp and layers % project_pp:
            raise ValueError("layers must be a multiple of project_pp")
        # Per-layer softmax temperature, so layers differ as real layers do (fixed seed).
        self.layer_scales = np.exp(np.random.default_rng(seed).uniform(-0.5, 1.0, size=layers))

    def _inputs(self, ids, lengths, routing):
        """Planted-routing Q/K/V/dO of one micro-batch (synth.py): member s's keys carry the
        generator's pre-sort layer-0 routing draws, so the GPU block scores -- and the K4
        profiles the tuner reads -- carry the generator's concentration."""
        mem = [int(lengths[i]) for i in ids]
        seed = self.seed + 7919 * self.rank + int(ids[0])
        return synth.planted_qkv(mem, [routing[i][0] for i in ids], self.H, self.Hkv, self.D, self.B, seed,
                                 device=self.device)

    def _profile_pass(self, q, k, lay):
        """Scorer pre-pass (K1 + K2 + K4) over every layer -> host profiles [layer][member]."""
        qbar, kbar = ops.block_pool(q, lay), ops.block_pool(k, lay)
        profs = torch.empty((self.layers, lay.nseq, max(1, lay.nb_max)), dtype=torch.float64, device=self.device)
        for l in range(self.layers):
            scale = float(self.layer_scales[l]) / math.sqrt(self.D)
            profs[l] = ops.coverage_profile(ops.block_scores(q, k, lay, scale, qbar=qbar, kbar=kbar), lay)
        return profs

    def _run_micro_batch(self, inputs, lay, budgets: np.ndarray):
        q, k, v, do = inputs
        nb = lay.nb_per_seq
        k_all = torch.from_numpy(np.minimum(budgets[:, None], nb[None, :]).astype(np.int32)).to(self.device)
        # One untimed pass of every layer first: a new micro-batch shape, and every per-layer keep
        # count (the selection tensors are [Hsel, NB, k_max]), can grow the caching allocator; a
        # cudaMalloc inside the timed window stalls the host and idles the GPU (measured: +20-70 ms
        # on single micro-batches, i.e. false imbalance). A one-layer warm-up did not cover the
        # per-layer k_max shapes.
        self._layers(q, k, v, do, lay, nb, k_all, budgets, self.layers)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * self.layers + 1)]
        ev[0].record()
        self._layers(q, k, v, do, lay, nb, k_all, budgets, self.layers, ev)
        torch.cuda.synchronize()
        # per layer: fwd = scorer + selector + forward, bwd = backward (block pooling in layer 0's fwd)
        t = [ev[i].elapsed_time(ev[i + 1]) for i in range(2 * self.layers)]
        return ev[0].elapsed_time(ev[-1]), t[0::2], t[1::2]

    def _layers(self, q, k, v, do, lay, nb, k_all, budgets, n_layers, ev=None):
        qbar, kbar = ops.block_pool(q, lay), ops.block_pool(k, lay)
        for l in range(n_layers):
            scale = float(self.layer_scales[l]) / math.sqrt(self.D)
            S = ops.block_scores(q, k, lay, scale, qbar=qbar, kbar=kbar)
            k_max = int(max(1, min(int(budgets[l]), int(nb.max()))))
            idx, cnt = ops.topk_select(S, lay, k_all[l], k_max, group=self.H // self.Hkv)
            o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt, scale)
            if ev is not None:
                ev[2 * l + 1].record()
            ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt, scale)
            if ev is not None:
                ev[2 * l + 2].record()

    def _gpu_profiles(self, lengths, routing, bins):
        """Closed loop: this rank's micro-batches through the scorer pre-pass; every sample's
        per-layer GPU profile assembled on every rank with one all-reduce (each sample's slot is
        written by exactly one rank, the others add zeros: exact). -> (profiles[sample][layer],
        per-micro-batch pre-pass ms, cached (inputs, layout) per micro-batch)."""
        nb = (np.asarray(lengths, np.int64) + self.B - 1) // self.B
        off = np.concatenate([[0], np.cumsum(nb * self.layers)])
        flat = torch.zeros(int(off[-1]), dtype=torch.float64, device=self.device)
        pre_ms, cache = [], []
        for ids in bins[self.rank]:
            cu = np.concatenate([[0], np.cumsum([int(lengths[i]) for i in ids])]).astype(np.int64)
            lay = ops.VarlenLayout.build(cu, self.B, device=self.device)
            inputs = self._inputs(ids, lengths, routing)
            self._profile_pass(inputs[0], inputs[1], lay)  # untimed: allocator warm-up (see _run_micro_batch)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            profs = self._profile_pass(inputs[0], inputs[1], lay)
            e1.record()
            for s, i in enumerate(ids):
                flat[int(off[i]):int(off[i + 1])] = profs[:, s, :nb[i]].reshape(-1)
            cache.append((inputs, lay))
            pre_ms.append((e0, e1))
        if self.world > 1:
            import torch.distributed as dist

            dist.all_reduce(flat, group=self.group)
        host = flat.cpu().numpy()
        profiles = [[host[int(off[i]) + l * nb[i]:int(off[i]) + (l + 1) * nb[i]].copy() for l in range(self.layers)]
                    for i in range(len(lengths))]
        return profiles, [a.elapsed_time(b) for a, b in pre_ms], cache

    def iteration(self, it: int, decisions_csv=None, plan_json=None, profiles_npz=None) -> dict:
        lengths, routing = self.h.generate_samples(self.gbs, self.layers, self.B, seed=mix_seed(self.seed, it),
                                                   dist=self.dist_spec, sorted=False)
        ids = np.arange(self.gbs)
        kw = dict(gbs=self.gbs, mbs=self.mbs, dp=self.world, num_layers=self.layers, table=self.table, iter_index=it,
                  **self.plan_kw)
        # 1) the batch plan does not read profiles (SAB / LBB plan from lengths + the estimator,
        #    sequential from order): plan once on a scratch copy of the estimator to learn which
        #    samples this rank owns, 2) score them on the GPU, 3) plan the step for real on the
        #    GPU profiles (same plan, DST on measured routing; the estimator calibrates once).
        scratch = copy.deepcopy(self.est)
        gen_sorted = [[np.sort(p)[::-1] for p in r] for r in routing]
        bins = self.h.plan_step(self.strategy, ids, lengths, gen_sorted, est=scratch, **kw)["micro_batch_bins"]
        profiles, pre_ms, cache = self._gpu_profiles(lengths, routing, bins)
        t0 = time.perf_counter()
        sp = self.h.plan_step(self.strategy, ids, lengths, profiles, est=self.est, decisions_csv=decisions_csv,
                              plan_json=plan_json, **kw)
        host_ms = (time.perf_counter() - t0) * 1e3
        if sp["micro_batch_bins"] != bins:
            raise RuntimeError("batch plan changed between the pre-plan and the step plan")
        if profiles_npz is not None and self.rank == 0:
            np.savez_compressed(profiles_npz, lengths=np.asarray(lengths), layers=self.layers,
                                **{f"p{i}_{l}": profiles[i][l] for i in range(len(lengths)) for l in range(self.layers)})
        rows = []  # per micro-batch: [total, fwd_0..fwd_{L-1}, bwd_0..bwd_{L-1}]; total includes the pre-pass
        for m, (inputs, lay) in enumerate(cache):
            tot, tf, tb = self._run_micro_batch(inputs, lay, sp["budgets"][self.rank][m])
            rows.append([tot + pre_ms[m]] + tf + tb)
        del cache
        if self.world > 1:
            import torch.distributed as dist

            t = torch.tensor(rows, dtype=torch.float64, device=self.device)
            outs = [torch.zeros_like(t) for _ in range(self.world)]
            dist.all_gather(outs, t, group=self.group)
            all_rows = [o.cpu().tolist() for o in outs]
        else:
            all_rows = [rows]
        mb_ms = [[r[0] for r in rr] for rr in all_rows]
        if plan_json is not None and self.rank == 0:  # per-(rank, mb) measured detail beside the plan
            L = self.layers
            detail = [[dict(total_ms=r[0], fwd_ms=sum(r[1:1 + L]), bwd_ms=sum(r[1 + L:1 + 2 * L]),
                            budgets=[int(x) for x in sp["budgets"][ri][mi]])
                       for mi, r in enumerate(rr)] for ri, rr in enumerate(all_rows)]
            with open(plan_json[:-len(".json")] + "_measured.json", "w") as f:
                json.dump(dict(ranks=detail), f)
        rec = summarize(mb_ms)
        rec.update(dst_overhead_ms=host_ms, avg_budget=sp["avg_budget"], mean_cov_drop=sp["mean_cov_drop"],
                   mb_ms=mb_ms, budgets=sp["budgets"], decisions=sp["decisions"])
        if self.project_pp:
            L = self.layers
            cl = ppj.Cluster(pp=self.project_pp, layers_per_stage=L // self.project_pp, comm_ms=0.05, dp_sync_ms=0.0)
            times = [[ppj.stage_times_measured(r[1:1 + L], r[1 + L:1 + 2 * L], cl) for r in rr] for rr in all_rows]
            buds = [[[int(k) for k in sp["budgets"][r][i]] for i in range(len(all_rows[r]))] for r in range(self.world)]
            rec["pp"] = ppj.project_iteration(times, buds, cl, L)
            rec["pp"].update(dst_overhead_ms=host_ms, mean_cov_drop=sp["mean_cov_drop"])
        return rec

    def run(self, iters: int, out_dir: str | None = None):
        records = []
        if out_dir and self.rank == 0:
            os.makedirs(out_dir, exist_ok=True)
        for it in range(iters):
            files = {}
            if out_dir and self.rank == 0:
                files = dict(decisions_csv=os.path.join(out_dir, f"decisions_{it}.csv"),
                             plan_json=os.path.join(out_dir, f"plan_{it}.json"),
                             profiles_npz=os.path.join(out_dir, f"gpu_profiles_{it}.npz"))
            records.append(self.iteration(it, **files))
        if out_dir and self.rank == 0:
            with open(os.path.join(out_dir, "iterations.csv"), "w") as f:
                f.write(ITER_HEADER)
                for it, rec in enumerate(records):
                    f.write(iteration_row(self.strategy, it, rec))
            if self.project_pp:
                with open(os.path.join(out_dir, f"iterations_pp{self.project_pp}.csv"), "w") as f:
                    f.write(ITER_HEADER)
                    for it, rec in enumerate(records):
                        f.write(iteration_row(self.strategy, it, rec["pp"]))
        return records


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--strategy", default="sab_dst", choices=["baseline", "dst", "sab", "lbb", "sab_dst", "lbb_dst"])
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--gbs-per-rank", type=int, default=5)
    ap.add_argument("--mbs", type=int, default=5)
    ap.add_argument("--layers", type=int, default=36)
    ap.add_argument("--mix", default="40/60", help="'40/60' = the C3 40%% 32K / 60%% 2K bimodal mix; 'default' = "
                                                   "the reference generator's default distribution")
    ap.add_argument("--table", default=None, help="cost table CSV (x,k,latency_ms), e.g. from profiler.py")
    ap.add_argument("--varlen", action="store_true", help="opt-in varlen-aware DST cost (predict_members at B)")
    ap.add_argument("--dense-grid", action="store_true", help="DST budget grid 1..256 (SURVEY 7.3(5): the 1.05x "
                                                                   "balance target) instead of the table's 16 points")
    ap.add_argument("--project-pp", type=int, default=0, help="also project a PP-stage 1F1B pipeline from the "
                                                              "measured per-layer times (pp_projection.py)")
    ap.add_argument("--heads", type=int, default=32, help="query heads")
    ap.add_argument("--kv-heads", type=int, default=32, help="kv heads; < --heads = GQA with group-shared selection "
                                                             "(BASELINE C4: 32q / 8kv)")
    ap.add_argument("--anchor", default="mean", choices=["min", "mean", "max"],
                    help="DST anchor over the base-budget latencies (dst.cpp select_anchor)")
    ap.add_argument("--threshold-p", type=float, default=0.1, help="DST coverage-drop bound p")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    if args.heads % args.kv_heads:
        ap.error("--heads must be a multiple of --kv-heads")
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dist_spec = None
    if args.mix == "40/60":
        dist_spec = dict(short_weight=0.6, short_log_mean=float(np.log(2048)), short_log_sigma=0.0,
                         long_log_mean=float(np.log(32768)), long_log_sigma=0.0)
    table = api().load_table(args.table)[0] if args.table else None
    drv = Driver(args.strategy, gbs=args.gbs_per_rank * world, mbs=args.mbs, layers=args.layers, dist_spec=dist_spec,
                 table=table, varlen_block_size=128 if args.varlen else 0, project_pp=args.project_pp, rank=rank,
                 world=world, heads=args.heads, kv_heads=args.kv_heads,
                 dst_grid=list(range(1, 257)) if args.dense_grid else None, anchor=args.anchor,
                 threshold_p=args.threshold_p, device=torch.device("cuda", local))
    recs = drv.run(args.iters, args.out)
    if rank == 0:
        for it, r in enumerate(recs):
            print(iteration_row(args.strategy, it, r), end="")
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
