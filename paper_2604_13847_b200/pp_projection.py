"""Pipeline-parallel projection.

SparseBalance's claims include PP-mode imbalance. This repo is DP-only, so PP is
not built. Instead, per-(micro-batch, stage) times are fed into a non-interleaved 1F1B model.
The times are either measured on the kernels (driver.py per-layer CUDA events) or taken from a
cost table. The model restates the reference's pipeline semantics (sim.cpp:100-275 and
435-489):

  * each stage runs min(pp-1-stage, m) warm-up forwards, then alternates one forward / one
    backward, then the cool-down backwards;
  * an op waits for the previous op on its stage and for its upstream forward (or downstream
    backward) plus one point-to-point hop `comm_ms`;
  * a rank's completion is the max over stages;
  * iteration time is the max over ranks plus the DP sync;
  * bubble = pp * completion - sum of busy time.

With table-derived stage times it reproduces the reference's simulate_iteration timing bit for
bit (tests/test_pp_projection.py). Floating-point sums use the reference's operation order.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass
class Cluster:
    pp: int = 4
    layers_per_stage: int = 9
    fwd_bwd_ratio: float = 2.0
    comm_ms: float = 0.05
    dp_sync_ms: float = 5.0


def stage_op_order(m: int, pp: int, stage: int):
    """Non-interleaved 1F1B op sequence of one stage: [("F"|"B", micro-batch)]."""
    warm = min(pp - 1 - stage, m)
    ops = [("F", i) for i in range(warm)]
    for i in range(m - warm):
        ops.append(("F", warm + i))
        ops.append(("B", i))
    ops.extend(("B", i) for i in range(m - warm, m))
    return ops


def pipeline_1f1b(fwd, bwd, comm_ms: float):
    """fwd / bwd [m][pp] ms -> dict(completion_ms, stage_busy_ms, bubble_ms)."""
    m, pp = len(fwd), len(fwd[0])
    f_end = [[None] * pp for _ in range(m)]
    b_end = [[None] * pp for _ in range(m)]
    seq = [stage_op_order(m, pp, s) for s in range(pp)]
    pos = [0] * pp
    free = [0.0] * pp
    busy = [0.0] * pp
    left = 2 * m * pp
    while left:
        moved = False
        for s in range(pp):
            while pos[s] < len(seq[s]):
                kind, i = seq[s][pos[s]]
                if kind == "F":
                    if s == 0:
                        ready = 0.0
                    elif f_end[i][s - 1] is None:
                        break
                    else:
                        ready = f_end[i][s - 1] + comm_ms
                else:
                    if s < pp - 1:
                        if b_end[i][s + 1] is None:
                            break
                        ready = b_end[i][s + 1] + comm_ms
                    else:
                        if f_end[i][s] is None:
                            break
                        ready = f_end[i][s]
                start = max(free[s], ready)
                dur = fwd[i][s] if kind == "F" else bwd[i][s]
                end = start + dur
                (f_end if kind == "F" else b_end)[i][s] = end
                free[s] = end
                busy[s] += dur
                pos[s] += 1
                left -= 1
                moved = True
        if not moved:
            raise RuntimeError("1F1B schedule deadlock")
    completion = max(free)
    total = 0.0
    for b in busy:
        total += b
    return dict(completion_ms=completion, stage_busy_ms=busy, bubble_ms=pp * completion - total)


def critical_lower_bound(fwd, bwd, comm_ms: float) -> float:
    """Dependency-derived lower bound on the 1F1B completion (the reference's L0-L3 chains)."""
    m, pp = len(fwd), len(fwd[0])
    bound = 0.0
    for s in range(pp):  # a stage executes all its own work
        b = 0.0
        for i in range(m):
            b += fwd[i][s] + bwd[i][s]
        bound = max(bound, b)
    for s in range(pp):  # micro-batch 0 must reach stage s; micro-batch m-1 must come back
        head = tail = b = 0.0
        for q in range(s):
            head += fwd[0][q]
            tail += bwd[m - 1][q]
        for i in range(m):
            b += fwd[i][s] + bwd[i][s]
        bound = max(bound, head + b + tail + 2.0 * s * comm_ms)
    trip_comm = 2.0 * (pp - 1) * comm_ms
    for i in range(m):  # one micro-batch's round trip
        t = trip_comm
        for s in range(pp):
            t += fwd[i][s] + bwd[i][s]
        bound = max(bound, t)
    suffix = [0.0] * (m + 1)  # straggler chain through stage 0
    for i in range(m - 1, -1, -1):
        suffix[i] = suffix[i + 1] + bwd[i][0]
    prefix = 0.0
    for i in range(m):
        prefix += fwd[i][0]
        t = trip_comm
        for s in range(1, pp):
            t += fwd[i][s] + bwd[i][s]
        bound = max(bound, prefix + t + suffix[i])
    return bound


def stage_times_from_table(h, table, x: int, budgets, cl: Cluster):
    """Per-stage (fwd, bwd) of one micro-batch from the cost table: sum of predict(x, k_l) over
    the stage's layers; backward = forward * fwd_bwd_ratio (the reference's micro_batch_time)."""
    f, b = [], []
    for s in range(cl.pp):
        tot = 0.0
        for k in budgets[s * cl.layers_per_stage:(s + 1) * cl.layers_per_stage]:
            tot += h.predict(table, int(x), int(k))[0]
        f.append(tot)
        b.append(tot * cl.fwd_bwd_ratio)
    return f, b


def stage_times_measured(layer_fwd_ms, layer_bwd_ms, cl: Cluster):
    """Per-stage (fwd, bwd) of one micro-batch from measured per-layer kernel times."""
    f, b = [], []
    for s in range(cl.pp):
        sl = slice(s * cl.layers_per_stage, (s + 1) * cl.layers_per_stage)
        tf = tb = 0.0
        for v in layer_fwd_ms[sl]:
            tf += v
        for v in layer_bwd_ms[sl]:
            tb += v
        f.append(tf)
        b.append(tb)
    return f, b


def project_iteration(rank_stage_times, rank_budgets, cl: Cluster, num_layers: int):
    """rank_stage_times[r][i] = (fwd[pp], bwd[pp]) per micro-batch; rank_budgets[r][i][l] -> the
    ScheduleResult fields of the reference (sim.cpp:435-489): iter_ms, bubble_ms, critical_lb_ms,
    max_mb_ms, mean_mb_ms, imbalance, avg_budget."""
    max_completion = max_critical = 0.0
    bubble = total_all = max_all = budget_total = 0.0
    count = 0
    for r, mbs in enumerate(rank_stage_times):
        fwd = [f for f, _ in mbs]
        bwd = [b for _, b in mbs]
        res = pipeline_1f1b(fwd, bwd, cl.comm_ms)
        max_completion = max(max_completion, res["completion_ms"])
        max_critical = max(max_critical, critical_lower_bound(fwd, bwd, cl.comm_ms))
        bubble += res["bubble_ms"]
        for i in range(len(mbs)):
            tot = 0.0
            for s in range(cl.pp):
                tot += fwd[i][s] + bwd[i][s]
            total_all += tot
            max_all = max(max_all, tot)
            count += 1
        for mb_b in rank_budgets[r]:
            for k in mb_b:
                budget_total += float(k)
    mean_all = total_all / count
    return dict(iter_ms=max_completion + cl.dp_sync_ms, bubble_ms=bubble,
                critical_lb_ms=max_critical + cl.dp_sync_ms, max_mb_ms=max_all, mean_mb_ms=mean_all,
                imbalance=max_all / mean_all if mean_all > 0.0 else 1.0,
                avg_budget=budget_total / (count * num_layers))

