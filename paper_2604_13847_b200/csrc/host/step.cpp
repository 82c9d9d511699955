// Step planner: decision half of the reference step driver (proj/core/src/sim.cpp:277-432,
// :491-495). The simulated 1F1B pipeline (sim.cpp:435-476) is intentionally absent: on
// B200 each rank runs its micro-batches through the real kernels with the budgets here.
#include "sparsebalance/step.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <utility>

#include "sparsebalance/errors.hpp"

namespace sparsebalance {

const char* strategy_name(Strategy s) {
  switch (s) {
    case Strategy::kBaseline: return "baseline";
    case Strategy::kDst: return "dst";
    case Strategy::kSab: return "sab";
    case Strategy::kLbb: return "lbb";
    case Strategy::kSabDst: return "sab_dst";
    case Strategy::kLbbDst: return "lbb_dst";
  }
  return "?";
}

Strategy parse_strategy(const std::string& name) {
  for (Strategy s : {Strategy::kBaseline, Strategy::kDst, Strategy::kSab, Strategy::kLbb,
                     Strategy::kSabDst, Strategy::kLbbDst}) {
    if (name == strategy_name(s)) return s;
  }
  throw ConfigError("scenario.strategy: unknown strategy '" + name +
                    "' (expected baseline|dst|sab|lbb|sab_dst|lbb_dst)");
}

bool strategy_uses_dst(Strategy s) {
  return s == Strategy::kDst || s == Strategy::kSabDst || s == Strategy::kLbbDst;
}

bool strategy_plans_batches(Strategy s) {
  return s == Strategy::kSab || s == Strategy::kLbb || s == Strategy::kSabDst ||
         s == Strategy::kLbbDst;
}

const char* base_budget_mode_name(BaseBudgetMode m) {
  return m == BaseBudgetMode::kFixed ? "fixed" : "coverage";
}

BaseBudgetMode parse_base_budget_mode(const std::string& name) {
  if (name == "fixed") return BaseBudgetMode::kFixed;
  if (name == "coverage") return BaseBudgetMode::kCoverage;
  throw ConfigError("base_budget_mode: unknown mode '" + name + "' (expected fixed|coverage)");
}

const char* dst_scope_name(DstScope s) { return s == DstScope::kRank ? "rank" : "global"; }

DstScope parse_dst_scope(const std::string& name) {
  if (name == "rank") return DstScope::kRank;
  if (name == "global") return DstScope::kGlobal;
  throw ConfigError("dst_scope: unknown scope '" + name + "' (expected rank|global)");
}

namespace {

using Clock = std::chrono::steady_clock;

double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

// A tuning group: micro-batches that share one anchor, with their (rank, mb) origin.
struct TuneGroup {
  GlobalBatch batch;
  std::vector<std::pair<int, int>> origin;
};

}  // namespace

StepPlan plan_step(std::span<const Sample> samples, Strategy strategy, const StepSetup& setup,
                   const ProfileTable& table, SparsityEstimator& est, int iter_index) {
  validate_plan_shape(setup.shape);
  if (setup.num_layers < 1) throw ConfigError("step.num_layers: must be >= 1");
  if (samples.size() != static_cast<std::size_t>(setup.shape.gbs))
    throw ConfigError("plan_step: got " + std::to_string(samples.size()) +
                      " samples, expected gbs = " + std::to_string(setup.shape.gbs));
  const int dp = setup.shape.dp;
  const auto layers = static_cast<std::size_t>(setup.num_layers);
  StepPlan out;

  // (1) Batching plan.
  if (strategy_plans_batches(strategy)) {
    const auto t0 = Clock::now();
    out.plan = (strategy == Strategy::kSab || strategy == Strategy::kSabDst)
                   ? plan_batching(samples, setup.shape, est, table)
                   : plan_lbb(samples, setup.shape);
    out.sab_overhead_ms = ms_since(t0);
  } else {
    out.plan = plan_sequential(samples, setup.shape);
  }

  // (2) Assembly + base budgets (coverage mode: the method's own per-mb budget).
  const std::vector<int>& grid =
      setup.dst.budget_grid.empty() ? table.budget_grid : setup.dst.budget_grid;
  out.ranks.reserve(static_cast<std::size_t>(dp));
  for (int r = 0; r < dp; ++r) {
    GlobalBatch gb = assemble_global_batch(samples, out.plan, r, setup.base_budget);
    if (setup.base_mode == BaseBudgetMode::kCoverage) {
      for (std::size_t i = 0; i < gb.micro_batches.size(); ++i)
        gb.base_budgets[i] =
            intrinsic_budget(gb.micro_batches[i], grid, setup.base_coverage_target);
    }
    out.ranks.push_back(std::move(gb));
  }
  out.budgets.resize(static_cast<std::size_t>(dp));
  for (int r = 0; r < dp; ++r)
    for (int kb : out.ranks[static_cast<std::size_t>(r)].base_budgets)
      out.budgets[static_cast<std::size_t>(r)].emplace_back(layers, kb);

  // (3) Per-layer DST.
  std::vector<BudgetDecision> calib;
  std::vector<std::int64_t> calib_len;
  double drop_sum = 0.0;
  if (strategy_uses_dst(strategy)) {
    DstConfig cfg = setup.dst;
    if (cfg.budget_grid.empty()) cfg.budget_grid = table.budget_grid;
    validate_dst_config(cfg);

    std::vector<TuneGroup> groups;
    if (setup.dst_scope == DstScope::kGlobal) {
      // All ranks pooled rank-major: every rank levels toward one anchor (sim.cpp:357-369).
      TuneGroup g;
      for (int r = 0; r < dp; ++r) {
        const GlobalBatch& gb = out.ranks[static_cast<std::size_t>(r)];
        for (std::size_t i = 0; i < gb.micro_batches.size(); ++i) {
          g.batch.micro_batches.push_back(gb.micro_batches[i]);
          g.batch.base_budgets.push_back(gb.base_budgets[i]);
          g.origin.emplace_back(r, static_cast<int>(i));
        }
      }
      groups.push_back(std::move(g));
    } else {
      for (int r = 0; r < dp; ++r) {
        TuneGroup g;
        g.batch = out.ranks[static_cast<std::size_t>(r)];
        for (std::size_t i = 0; i < g.batch.micro_batches.size(); ++i)
          g.origin.emplace_back(r, static_cast<int>(i));
        groups.push_back(std::move(g));
      }
    }

    for (const TuneGroup& g : groups) {
      const std::size_t nmb = g.batch.micro_batches.size();
      // Per-member calibration share k_solo / k_base (sim.cpp:385-404).
      std::vector<std::vector<double>> share(nmb);
      for (std::size_t i = 0; i < nmb; ++i) {
        const MicroBatch& mb = g.batch.micro_batches[i];
        share[i].assign(mb.samples.size(), 1.0);
        if (setup.base_mode != BaseBudgetMode::kCoverage || mb.samples.size() <= 1) continue;
        for (std::size_t s = 0; s < mb.samples.size(); ++s) {
          const int k_solo = intrinsic_budget(make_micro_batch({mb.samples[s]}), grid,
                                              setup.base_coverage_target);
          share[i][s] = static_cast<double>(k_solo) / static_cast<double>(g.batch.base_budgets[i]);
        }
      }
      for (std::size_t layer = 0; layer < layers; ++layer) {
        TuneBatchResult tuned = tune_global_batch(g.batch, static_cast<int>(layer), cfg, table);
        out.dst_overhead_ms += tuned.overhead_ms;
        for (const BudgetDecision& d : tuned.decisions) {
          const auto mbi = static_cast<std::size_t>(d.micro_batch_id);
          const auto [rank, local] = g.origin[mbi];
          out.budgets[static_cast<std::size_t>(rank)][static_cast<std::size_t>(local)][layer] =
              d.k_final;
          drop_sum += d.coverage_drop;
          // Expansions track the batch-dependent anchor, not the sample's need: skip them.
          if (d.direction == TuneDirection::kExpanded) continue;
          const MicroBatch& mb = g.batch.micro_batches[mbi];
          for (std::size_t s = 0; s < mb.samples.size(); ++s) {
            BudgetDecision obs = d;
            obs.k_final = std::max(1, static_cast<int>(std::lround(d.k_final * share[mbi][s])));
            calib.push_back(obs);
            calib_len.push_back(mb.samples[s].length);
          }
        }
        out.decisions.insert(out.decisions.end(), tuned.decisions.begin(), tuned.decisions.end());
      }
    }
  }

  double ksum = 0.0;
  std::size_t cells = 0;
  for (const auto& rank : out.budgets)
    for (const auto& mb : rank) {
      for (int k : mb) ksum += static_cast<double>(k);
      cells += mb.size();
    }
  out.avg_budget = cells ? ksum / static_cast<double>(cells) : 0.0;
  out.mean_cov_drop =
      out.decisions.empty() ? 0.0 : drop_sum / static_cast<double>(out.decisions.size());

  // (5) Calibration.
  if (!calib.empty() && setup.calibrate_every > 0 && (iter_index + 1) % setup.calibrate_every == 0)
    calibrate(est, calib, calib_len);
  return out;
}

}  // namespace sparsebalance
