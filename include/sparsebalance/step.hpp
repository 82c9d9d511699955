// sparsebalance-b200 host layer: the per-step planner that drives the GPU hot path.
//
// Re-hosts the decision half of the reference step driver simulate_iteration
// (proj/core/src/sim.cpp:277-432 and :491-495): SAB / LBB / sequential planning,
// per-rank assembly, coverage-mode base budgets, per-layer DST with global or rank
// anchor scope and the estimator calibration shares. The reference's step 4 (the
// simulated 1F1B pipeline, sim.cpp:435-476) is replaced by real kernels: the planner's
// `budgets[rank][mb][layer]` is the keep count fed to sb_topk_select / sb_sparse_attn_*.
#pragma once

#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "sparsebalance/dst.hpp"
#include "sparsebalance/profile_table.hpp"
#include "sparsebalance/sab.hpp"
#include "sparsebalance/workload.hpp"

// Exported from libsparsebalance_b200.so (the library builds with -fvisibility=hidden): the
// C++ API is part of the drop-in boundary.
#pragma GCC visibility push(default)
namespace sparsebalance {

enum class Strategy { kBaseline, kDst, kSab, kLbb, kSabDst, kLbbDst };
enum class BaseBudgetMode { kFixed, kCoverage };
enum class DstScope { kRank, kGlobal };

const char* strategy_name(Strategy strategy);
Strategy parse_strategy(const std::string& name);
bool strategy_uses_dst(Strategy strategy);
bool strategy_plans_batches(Strategy strategy);
const char* base_budget_mode_name(BaseBudgetMode mode);
BaseBudgetMode parse_base_budget_mode(const std::string& name);
const char* dst_scope_name(DstScope scope);
DstScope parse_dst_scope(const std::string& name);

struct StepSetup {
  PlanShape shape;          // gbs / mbs / dp
  int num_layers = 36;
  int base_budget = 32;     // kFixed
  BaseBudgetMode base_mode = BaseBudgetMode::kCoverage;
  double base_coverage_target = 0.9;
  DstScope dst_scope = DstScope::kGlobal;
  DstConfig dst;            // empty grid -> table grid
  int calibrate_every = 1;
};

struct StepPlan {
  PackingPlan plan;
  std::vector<GlobalBatch> ranks;                         // per-rank assembled batch
  std::vector<std::vector<std::vector<int>>> budgets;     // [rank][mb][layer] keep count
  std::vector<BudgetDecision> decisions;                  // reference order (group, layer, mb)
  double sab_overhead_ms = 0.0;
  double dst_overhead_ms = 0.0;
  double mean_cov_drop = 0.0;
  double avg_budget = 0.0;
};

// One optimizer step's decisions. Mutates `est` exactly where the reference does
// (calibration after DST when (iter_index + 1) % calibrate_every == 0).
StepPlan plan_step(std::span<const Sample> samples, Strategy strategy, const StepSetup& setup,
                   const ProfileTable& table, SparsityEstimator& est, int iter_index);

}  // namespace sparsebalance
#pragma GCC visibility pop
