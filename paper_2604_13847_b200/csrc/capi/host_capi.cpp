// Flat C ABI over the host decision layer (declared in include/sb_host.h).
//
// Compiled twice from this one source:
//   * product:  -DSB_HOST_PREFIX=sbh_   against include/sparsebalance/*.hpp (this repo)
//   * oracle:   -DSB_HOST_PREFIX=sbref_ -DSB_REF against the reference headers/sources
//               (oracle/Makefile), so parity tests marshal both sides identically.
// Only plan_step differs: the reference exposes the step through simulate_iteration
// (sim.cpp:277), this repo through plan_step (step.hpp).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "sparsebalance/dst.hpp"
#include "sparsebalance/errors.hpp"
#include "sparsebalance/profile_table.hpp"
#include "sparsebalance/sab.hpp"
#include "sparsebalance/workload.hpp"
#ifdef SB_REF
#include "sparsebalance/sim.hpp"
#else
#include "sparsebalance/step.hpp"
#endif

#define SB_EXPORT __attribute__((visibility("default")))
#include "../../../include/sb_host.h"

namespace sb = sparsebalance;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const sb::ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  } catch (...) {
    g_err = "unknown exception";
    return 2;
  }
}

sb::ProfileTable make_table(const int64_t* bins, int nx, const int* grid, int nk,
                            const double* lat) {
  if (nx < 0 || nk < 0) throw sb::ConfigError("table: negative dimension");
  sb::ProfileTable t;
  t.length_bins.assign(bins, bins + nx);
  t.budget_grid.assign(grid, grid + nk);
  t.latency_ms.assign(lat, lat + static_cast<std::size_t>(nx) * static_cast<std::size_t>(nk));
  return t;
}

sb::RoutingProfile make_profile(const double* s, int64_t lo, int64_t hi) {
  sb::RoutingProfile p;
  p.scores.assign(s + lo, s + hi);
  return p;
}

std::vector<sb::Sample> make_samples(int n, const int64_t* ids, const int64_t* lengths, int nl,
                                     const double* profiles, const int64_t* off) {
  std::vector<sb::Sample> out(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    sb::Sample& s = out[static_cast<std::size_t>(i)];
    s.id = ids ? ids[i] : i;
    s.length = lengths[i];
    for (int l = 0; l < nl; ++l) {
      const std::size_t c = static_cast<std::size_t>(i) * static_cast<std::size_t>(nl) +
                            static_cast<std::size_t>(l);
      s.routing_profiles.push_back(make_profile(profiles, off[c], off[c + 1]));
    }
  }
  return out;
}

sb::SparsityEstimator make_est(const int64_t* edges, int ne, const double* ema, double alpha,
                               const int* grid, int ng) {
  sb::SparsityEstimator est = sb::make_estimator(std::vector<std::int64_t>(edges, edges + ne),
                                                 std::vector<int>(grid, grid + ng), alpha,
                                                 static_cast<double>(grid[0]));
  est.ema_budget.assign(ema, ema + ne);
  return est;
}

int direction_code(sb::TuneDirection d) {
  return d == sb::TuneDirection::kCompressed ? 0 : d == sb::TuneDirection::kExpanded ? 1 : 2;
}

sb::AnchorStrategy anchor_of(int a) {
  if (a == 0) return sb::AnchorStrategy::kMin;
  if (a == 1) return sb::AnchorStrategy::kMean;
  if (a == 2) return sb::AnchorStrategy::kMax;
  throw sb::ConfigError("anchor: expected 0 (min), 1 (mean) or 2 (max)");
}

void write_plan(const sb::PackingPlan& plan, int64_t* out_ids, int* out_mb_off,
                double* out_weights) {
  std::size_t pos = 0, mb = 0;
  out_mb_off[0] = 0;
  for (const auto& rank : plan.micro_batch_bins) {
    for (const auto& ids : rank) {
      for (std::int64_t id : ids) out_ids[pos++] = id;
      out_mb_off[++mb] = static_cast<int>(pos);
    }
  }
  if (out_weights)
    for (std::size_t i = 0; i < plan.weights.size(); ++i) out_weights[i] = plan.weights[i];
}

}  // namespace

extern "C" {

SB_EXPORT const char* SBH(last_error)(void) { return g_err.c_str(); }

SB_EXPORT int SBH(predict)(const int64_t* bins, int nx, const int* grid, int nk,
                           const double* lat, int64_t x, int k, double* out_ms,
                           int* out_extrapolated) {
  return guarded([&] {
    const auto est = sb::predict(make_table(bins, nx, grid, nk, lat), x, k);
    *out_ms = est.value_ms;
    if (out_extrapolated) *out_extrapolated = est.extrapolated ? 1 : 0;
  });
}

SB_EXPORT int SBH(align)(const int64_t* bins, int nx, const int* grid, int nk, const double* lat,
                         int64_t x, double target_ms, int* out_budget, int* out_infeasible) {
  return guarded([&] {
    const auto r = sb::align(make_table(bins, nx, grid, nk, lat), x, target_ms);
    *out_budget = r.budget;
    if (out_infeasible) *out_infeasible = r.infeasible ? 1 : 0;
  });
}

SB_EXPORT int SBH(synthesize_table)(double c_lin, double c_attn, double c_fixed,
                                    double noise_sigma, int block_size, const int64_t* bins,
                                    int nx, const int* grid, int nk, uint64_t seed,
                                    double* out_lat) {
  return guarded([&] {
    sb::CostModelSpec m;
    m.c_lin = c_lin;
    m.c_attn = c_attn;
    m.c_fixed = c_fixed;
    m.noise_sigma = noise_sigma;
    m.block_size = block_size;
    const auto t = sb::synthesize_table(m, std::vector<std::int64_t>(bins, bins + nx),
                                        std::vector<int>(grid, grid + nk), seed);
    std::memcpy(out_lat, t.latency_ms.data(), t.latency_ms.size() * sizeof(double));
  });
}

SB_EXPORT int SBH(load_table)(const char* path, int* nx, int* nk, int64_t* out_bins,
                              int* out_grid, double* out_lat, int* out_repaired_cells) {
  return guarded([&] {
    const auto r = sb::load_table(path);
    *nx = static_cast<int>(r.table.length_bins.size());
    *nk = static_cast<int>(r.table.budget_grid.size());
    if (out_repaired_cells) *out_repaired_cells = r.repaired_cells;
    if (out_bins) std::memcpy(out_bins, r.table.length_bins.data(), sizeof(int64_t) * *nx);
    if (out_grid) std::memcpy(out_grid, r.table.budget_grid.data(), sizeof(int) * *nk);
    if (out_lat) std::memcpy(out_lat, r.table.latency_ms.data(), sizeof(double) * *nx * *nk);
  });
}

SB_EXPORT int SBH(save_table)(const char* path, const int64_t* bins, int nx, const int* grid,
                              int nk, const double* lat) {
  return guarded([&] { sb::save_table(make_table(bins, nx, grid, nk, lat), path); });
}

SB_EXPORT int SBH(coverage)(const double* scores, int m, int k, double* out) {
  return guarded([&] { *out = sb::coverage(make_profile(scores, 0, m), k); });
}

SB_EXPORT int SBH(select_anchor)(const double* lat, int n, int anchor, double* out) {
  return guarded([&] {
    *out = sb::select_anchor(std::span<const double>(lat, static_cast<std::size_t>(n)),
                             anchor_of(anchor));
  });
}

SB_EXPORT int SBH(tune_global_batch)(const int64_t* bins, int nx, const int* grid, int nk,
                                     const double* lat, int n_mb, const int64_t* x,
                                     const int* k_base, const double* profiles,
                                     const int64_t* prof_off, int layer, double threshold_p,
                                     int anchor, const int* dst_grid, int n_dst_grid, int* out_i,
                                     double* out_d) {
  return guarded([&] {
    const auto table = make_table(bins, nx, grid, nk, lat);
    sb::GlobalBatch gb;
    for (int i = 0; i < n_mb; ++i) {
      sb::MicroBatch mb;
      mb.length_descriptor = x[i];
      // Only the tuned layer's profile matters; place it at index `layer`.
      mb.merged_profiles.resize(static_cast<std::size_t>(layer) + 1);
      mb.merged_profiles[static_cast<std::size_t>(layer)] =
          make_profile(profiles, prof_off[i], prof_off[i + 1]);
      gb.micro_batches.push_back(std::move(mb));
      gb.base_budgets.push_back(k_base[i]);
    }
    sb::DstConfig cfg;
    cfg.threshold_p = threshold_p;
    cfg.anchor = anchor_of(anchor);
    cfg.budget_grid.assign(dst_grid, dst_grid + n_dst_grid);
    sb::validate_dst_config(cfg);
    const auto res = sb::tune_global_batch(gb, layer, cfg, table);
    for (std::size_t i = 0; i < res.decisions.size(); ++i) {
      const auto& d = res.decisions[i];
      int* oi = out_i + 5 * i;
      oi[0] = d.micro_batch_id;
      oi[1] = d.k_base;
      oi[2] = d.k_anchor;
      oi[3] = d.k_final;
      oi[4] = direction_code(d.direction);
      double* od = out_d + 3 * i;
      od[0] = d.coverage_drop;
      od[1] = d.predicted_ms_base;
      od[2] = d.predicted_ms_final;
    }
  });
}

#ifndef SB_REF
// Extension (dst.hpp CoverageTable): the per-rank exchange payload and the tuner over it.
SB_EXPORT int SBH(coverage_table)(const double* scores, int m, const int* grid, int n_grid, int k_base,
                                  double* out) {
  return guarded([&] {
    if (n_grid < 1) throw sb::ConfigError("coverage_table: empty budget grid");
    const auto prof = make_profile(scores, 0, m);
    for (int g = 0; g < n_grid; ++g) out[g] = sb::coverage(prof, grid[g]);
    out[n_grid] = sb::coverage(prof, k_base);
  });
}

// One DP rank's whole workload estimate in one call: make_micro_batch over the members'
// per-layer profiles (member-major: profiles[s * nl + l] at off[...]), the base budget
// (coverage mode: intrinsic_budget, else `base_budget`) and per layer the coverage table
// out_cov[l][n_grid + 1] (grid points, then k_base).
SB_EXPORT int SBH(rank_estimate)(int ns, const int64_t* lengths, int nl, const double* profiles, const int64_t* off,
                                 const int* grid, int n_grid, int coverage_mode, int base_budget,
                                 double coverage_target, int64_t* out_x, int* out_k_base, double* out_cov) {
  return guarded([&] {
    const auto mb = sb::make_micro_batch(make_samples(ns, nullptr, lengths, nl, profiles, off));
    const std::span<const int> g(grid, static_cast<std::size_t>(n_grid));
    const int kb = coverage_mode ? sb::intrinsic_budget(mb, g, coverage_target) : base_budget;
    *out_x = mb.length_descriptor;
    *out_k_base = kb;
    for (int l = 0; l < nl; ++l) {
      const auto t = sb::coverage_table(mb.merged_profiles[static_cast<std::size_t>(l)], g, kb);
      double* row = out_cov + static_cast<std::size_t>(l) * static_cast<std::size_t>(n_grid + 1);
      for (int i = 0; i < n_grid; ++i) row[i] = t.values[static_cast<std::size_t>(i)];
      row[n_grid] = t.at(kb);
    }
  });
}

// tune_global_batch_cov for every layer at once: cov[n_mb][nl][n_dst_grid + 1];
// out_k_final[n_mb][nl]; out_i[nl][n_mb][5] / out_d[nl][n_mb][3] as tune_global_batch's.
SB_EXPORT int SBH(tune_layers_cov)(const int64_t* bins, int nx, const int* grid, int nk, const double* lat, int n_mb,
                                   const int64_t* x, const int* k_base, const double* cov, const int64_t* mem_len,
                                   const int64_t* mem_off, int varlen_block_size, int nl, double threshold_p,
                                   int anchor, const int* dst_grid, int n_dst_grid, int* out_k_final, int* out_i,
                                   double* out_d) {
  return guarded([&] {
    const auto table = make_table(bins, nx, grid, nk, lat);
    sb::DstConfig cfg;
    cfg.threshold_p = threshold_p;
    cfg.anchor = anchor_of(anchor);
    cfg.budget_grid.assign(dst_grid, dst_grid + n_dst_grid);
    cfg.varlen_block_size = varlen_block_size;
    sb::validate_dst_config(cfg);
    if (varlen_block_size > 0 && (mem_len == nullptr || mem_off == nullptr))
      throw sb::ConfigError("tune_layers_cov: varlen cost needs member lengths");
    sb::GlobalBatch gb;
    for (int i = 0; i < n_mb; ++i) {
      sb::MicroBatch mb;
      mb.length_descriptor = x[i];
      if (mem_len != nullptr && mem_off != nullptr)
        for (int64_t e = mem_off[i]; e < mem_off[i + 1]; ++e) {
          sb::Sample smp;
          smp.id = e;
          smp.length = mem_len[e];
          mb.samples.push_back(std::move(smp));
        }
      gb.micro_batches.push_back(std::move(mb));
      gb.base_budgets.push_back(k_base[i]);
    }
    const std::size_t G = static_cast<std::size_t>(n_dst_grid) + 1;
    std::vector<sb::CoverageTable> tabs(static_cast<std::size_t>(n_mb));
    for (int l = 0; l < nl; ++l) {
      for (int i = 0; i < n_mb; ++i) {
        const double* row = cov + (static_cast<std::size_t>(i) * static_cast<std::size_t>(nl) +
                                   static_cast<std::size_t>(l)) * G;
        auto& t = tabs[static_cast<std::size_t>(i)];
        t.budgets.assign(dst_grid, dst_grid + n_dst_grid);
        t.values.assign(row, row + n_dst_grid);
        t.budgets.push_back(k_base[i]);
        t.values.push_back(row[n_dst_grid]);
      }
      const auto res = sb::tune_global_batch_cov(gb, tabs, l, cfg, table);
      for (std::size_t i = 0; i < res.decisions.size(); ++i) {
        const auto& d = res.decisions[i];
        out_k_final[i * static_cast<std::size_t>(nl) + static_cast<std::size_t>(l)] = d.k_final;
        const std::size_t o = static_cast<std::size_t>(l) * static_cast<std::size_t>(n_mb) + i;
        int* oi = out_i + 5 * o;
        oi[0] = d.micro_batch_id;
        oi[1] = d.k_base;
        oi[2] = d.k_anchor;
        oi[3] = d.k_final;
        oi[4] = direction_code(d.direction);
        double* od = out_d + 3 * o;
        od[0] = d.coverage_drop;
        od[1] = d.predicted_ms_base;
        od[2] = d.predicted_ms_final;
      }
    }
  });
}

SB_EXPORT int SBH(tune_global_batch_cov)(const int64_t* bins, int nx, const int* grid, int nk, const double* lat,
                                         int n_mb, const int64_t* x, const int* k_base, const double* cov,
                                         const int64_t* mem_len, const int64_t* mem_off, int varlen_block_size,
                                         int layer, double threshold_p, int anchor, const int* dst_grid,
                                         int n_dst_grid, int* out_i, double* out_d) {
  return guarded([&] {
    const auto table = make_table(bins, nx, grid, nk, lat);
    sb::DstConfig cfg;
    cfg.threshold_p = threshold_p;
    cfg.anchor = anchor_of(anchor);
    cfg.budget_grid.assign(dst_grid, dst_grid + n_dst_grid);
    cfg.varlen_block_size = varlen_block_size;
    sb::validate_dst_config(cfg);
    if (varlen_block_size > 0 && (mem_len == nullptr || mem_off == nullptr))
      throw sb::ConfigError("tune_global_batch_cov: varlen cost needs member lengths");
    sb::GlobalBatch gb;
    std::vector<sb::CoverageTable> tabs;
    for (int i = 0; i < n_mb; ++i) {
      sb::MicroBatch mb;
      mb.length_descriptor = x[i];
      if (mem_len != nullptr && mem_off != nullptr)
        for (int64_t e = mem_off[i]; e < mem_off[i + 1]; ++e) {
          sb::Sample smp;
          smp.id = e;
          smp.length = mem_len[e];
          mb.samples.push_back(std::move(smp));
        }
      gb.micro_batches.push_back(std::move(mb));
      gb.base_budgets.push_back(k_base[i]);
      sb::CoverageTable t;
      const double* row = cov + static_cast<std::size_t>(i) * static_cast<std::size_t>(n_dst_grid + 1);
      t.budgets.assign(dst_grid, dst_grid + n_dst_grid);
      t.values.assign(row, row + n_dst_grid);
      t.budgets.push_back(k_base[i]);
      t.values.push_back(row[n_dst_grid]);
      tabs.push_back(std::move(t));
    }
    const auto res = sb::tune_global_batch_cov(gb, tabs, layer, cfg, table);
    for (std::size_t i = 0; i < res.decisions.size(); ++i) {
      const auto& d = res.decisions[i];
      int* oi = out_i + 5 * i;
      oi[0] = d.micro_batch_id;
      oi[1] = d.k_base;
      oi[2] = d.k_anchor;
      oi[3] = d.k_final;
      oi[4] = direction_code(d.direction);
      double* od = out_d + 3 * i;
      od[0] = d.coverage_drop;
      od[1] = d.predicted_ms_base;
      od[2] = d.predicted_ms_final;
    }
  });
}
#endif

SB_EXPORT int SBH(make_micro_batch)(int ns, const int64_t* lengths, int nl,
                                    const double* profiles, const int64_t* off, double* out,
                                    int64_t cap, int64_t* out_off,
                                    int64_t* out_length_descriptor) {
  return guarded([&] {
    const auto mb = sb::make_micro_batch(make_samples(ns, nullptr, lengths, nl, profiles, off));
    *out_length_descriptor = mb.length_descriptor;
    int64_t pos = 0;
    out_off[0] = 0;
    for (int l = 0; l < nl; ++l) {
      const auto& s = mb.merged_profiles[static_cast<std::size_t>(l)].scores;
      if (pos + static_cast<int64_t>(s.size()) > cap)
        throw sb::ConfigError("make_micro_batch: output capacity too small");
      std::memcpy(out + pos, s.data(), s.size() * sizeof(double));
      pos += static_cast<int64_t>(s.size());
      out_off[l + 1] = pos;
    }
  });
}

SB_EXPORT int SBH(coverage_budget)(const double* scores, int m, double target, int* out) {
  return guarded([&] { *out = sb::coverage_budget(make_profile(scores, 0, m), target); });
}

SB_EXPORT int SBH(intrinsic_budget)(int nl, const double* profiles, const int64_t* off,
                                    const int* grid, int ng, double target, int* out) {
  return guarded([&] {
    sb::MicroBatch mb;
    for (int l = 0; l < nl; ++l) mb.merged_profiles.push_back(make_profile(profiles, off[l], off[l + 1]));
    *out = sb::intrinsic_budget(mb, std::span<const int>(grid, static_cast<std::size_t>(ng)), target);
  });
}

#ifdef SB_REF
// The reference sorts profiles inside generation (workload.cpp:58). The pre-sort vectors
// are regenerated here with the reference's public Rng in generate_samples' call order
// (workload.cpp:239-271, draw_profile :42-57); the caller checks sort(pre) == sorted.
namespace {
std::vector<sb::Sample> ref_unsorted(const sb::LengthDistributionSpec& spec, int64_t count,
                                     const sb::ConcentrationSpec& c, int nl, int block,
                                     uint64_t seed) {
  sb::Rng rng(sb::mix_seed(seed));
  std::vector<sb::Sample> out;
  for (int64_t i = 0; i < count; ++i) {
    sb::Sample s;
    s.id = i;
    s.length = sb::sample_length(spec, rng);
    double a_seq = rng.lognormal(c.alpha_log_mean, c.alpha_log_sigma) *
                   std::pow(c.length_ref / static_cast<double>(s.length), c.length_exponent);
    for (int l = 0; l < nl; ++l) {
      double a = a_seq;
      if (c.layer_log_sigma > 0.0) a *= rng.lognormal(0.0, c.layer_log_sigma);
      a = std::clamp(a, 1e-4, 1e4);
      const auto m = static_cast<std::size_t>((s.length + block - 1) / block);
      sb::RoutingProfile p;
      p.scores.resize(m);
      double tot = 0.0;
      for (std::size_t j = 0; j < m; ++j) {
        double g = rng.gamma(a);
        p.scores[j] = g;
        tot += g;
      }
      if (tot <= 0.0) {
        std::fill(p.scores.begin(), p.scores.end(), 1.0 / static_cast<double>(m));
      } else {
        for (double& v : p.scores) v /= tot;
      }
      s.routing_profiles.push_back(std::move(p));
    }
    out.push_back(std::move(s));
  }
  return out;
}
}  // namespace
#endif

SB_EXPORT int SBH(generate_samples)(int kind, const double* dist, const double* conc,
                                    int64_t count, int num_layers, int block_size, uint64_t seed,
                                    int sorted, int64_t* out_lengths, int64_t* out_off,
                                    double* out_profiles) {
  return guarded([&] {
    sb::LengthDistributionSpec spec;
    if (kind == 0) spec.kind = sb::LengthDistributionSpec::Kind::kFixed;
    else if (kind == 1) spec.kind = sb::LengthDistributionSpec::Kind::kBimodal;
    else if (kind == 2) spec.kind = sb::LengthDistributionSpec::Kind::kLongTail;
    else throw sb::ConfigError("generate_samples: kind must be 0, 1 or 2");
    spec.min_length = static_cast<int64_t>(dist[0]);
    spec.max_length = static_cast<int64_t>(dist[1]);
    spec.fixed_length = static_cast<int64_t>(dist[2]);
    spec.short_weight = dist[3];
    spec.short_log_mean = dist[4];
    spec.short_log_sigma = dist[5];
    spec.long_log_mean = dist[6];
    spec.long_log_sigma = dist[7];
    spec.tail_exponent = dist[8];
    sb::ConcentrationSpec c;
    c.alpha_log_mean = conc[0];
    c.alpha_log_sigma = conc[1];
    c.layer_log_sigma = conc[2];
    c.length_ref = conc[3];
    c.length_exponent = conc[4];
    std::vector<sb::Sample> samples;
    if (sorted) {
      samples = sb::generate_samples(spec, count, c, num_layers, block_size, seed);
    } else {
#ifdef SB_REF
      sb::validate_distribution(spec);
      sb::validate_concentration(c);
      samples = ref_unsorted(spec, count, c, num_layers, block_size, seed);
#else
      samples = sb::generate_samples_unsorted(spec, count, c, num_layers, block_size, seed);
#endif
    }
    int64_t pos = 0;
    out_off[0] = 0;
    for (std::size_t i = 0; i < samples.size(); ++i) {
      out_lengths[i] = samples[i].length;
      for (int l = 0; l < num_layers; ++l) {
        const auto& s = samples[i].routing_profiles[static_cast<std::size_t>(l)].scores;
        if (out_profiles) std::memcpy(out_profiles + pos, s.data(), s.size() * sizeof(double));
        pos += static_cast<int64_t>(s.size());
        out_off[i * static_cast<std::size_t>(num_layers) + static_cast<std::size_t>(l) + 1] = pos;
      }
    }
  });
}

SB_EXPORT int SBH(default_bin_edges)(int64_t max_length, int64_t* out, int cap, int* out_n) {
  return guarded([&] {
    const auto e = sb::default_bin_edges(max_length);
    *out_n = static_cast<int>(e.size());
    if (static_cast<int>(e.size()) > cap) throw sb::ConfigError("default_bin_edges: capacity");
    std::memcpy(out, e.data(), e.size() * sizeof(int64_t));
  });
}

SB_EXPORT int SBH(estimate_sparsity)(const int64_t* edges, int ne, const double* ema,
                                     const int* grid, int ng, int64_t length, int* out) {
  return guarded([&] { *out = sb::estimate_sparsity(make_est(edges, ne, ema, 0.2, grid, ng), length); });
}

SB_EXPORT int SBH(calibrate)(const int64_t* edges, int ne, double* ema_inout, double alpha,
                             const int* grid, int ng, int n, const int* k_final,
                             const int64_t* lengths) {
  return guarded([&] {
    auto est = make_est(edges, ne, ema_inout, alpha, grid, ng);
    std::vector<sb::BudgetDecision> ds(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) ds[static_cast<std::size_t>(i)].k_final = k_final[i];
    sb::calibrate(est, ds, std::span<const std::int64_t>(lengths, static_cast<std::size_t>(n)));
    std::memcpy(ema_inout, est.ema_budget.data(), sizeof(double) * static_cast<std::size_t>(ne));
  });
}

SB_EXPORT int SBH(bin_packing)(const double* weights, int n, int num_bins, int max_items_per_bin,
                               int* out_items, int* out_bin_off) {
  return guarded([&] {
    const auto bins = sb::bin_packing(std::span<const double>(weights, static_cast<std::size_t>(n)),
                                      num_bins, max_items_per_bin);
    int pos = 0;
    out_bin_off[0] = 0;
    for (std::size_t b = 0; b < bins.size(); ++b) {
      for (int it : bins[b]) out_items[pos++] = it;
      out_bin_off[b + 1] = pos;
    }
  });
}

SB_EXPORT int SBH(plan_batching)(int strategy, int n, const int64_t* ids, const int64_t* lengths,
                                 int gbs, int mbs, int dp, const int64_t* edges, int ne,
                                 const double* ema, double alpha, const int* est_grid,
                                 int n_est_grid, const int64_t* bins, int nx, const int* grid,
                                 int nk, const double* lat, int64_t* out_ids, int* out_mb_off,
                                 double* out_weights) {
  return guarded([&] {
    std::vector<sb::Sample> batch(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) {
      batch[static_cast<std::size_t>(i)].id = ids[i];
      batch[static_cast<std::size_t>(i)].length = lengths[i];
    }
    sb::PlanShape shape{gbs, mbs, dp};
    sb::PackingPlan plan;
    if (strategy == 0) {
      plan = sb::plan_batching(batch, shape, make_est(edges, ne, ema, alpha, est_grid, n_est_grid),
                               make_table(bins, nx, grid, nk, lat));
    } else if (strategy == 1) {
      plan = sb::plan_lbb(batch, shape);
    } else if (strategy == 2) {
      plan = sb::plan_sequential(batch, shape);
    } else {
      throw sb::ConfigError("plan_batching: strategy must be 0 (sab), 1 (lbb) or 2 (sequential)");
    }
    write_plan(plan, out_ids, out_mb_off, out_weights);
  });
}

SB_EXPORT int SBH(predict_members)(const int64_t* bins, int nx, const int* grid, int nk, const double* lat,
                                   const int64_t* lengths, int n, int k, int block_size, double* out_ms,
                                   int* out_extrapolated) {
  return guarded([&] {
#ifdef SB_REF
    (void)bins, (void)nx, (void)grid, (void)nk, (void)lat, (void)lengths, (void)n, (void)k, (void)block_size;
    (void)out_ms, (void)out_extrapolated;
    throw sb::ConfigError("predict_members is not in the reference");
#else
    const auto table = make_table(bins, nx, grid, nk, lat);
    const auto e = sb::predict_members(table, std::span<const int64_t>(lengths, static_cast<std::size_t>(n)), k,
                                       block_size);
    *out_ms = e.value_ms;
    *out_extrapolated = e.extrapolated ? 1 : 0;
#endif
  });
}

#ifdef SB_REF
// Test oracle only (the reference build): the reference step driver with a pipeline-parallel
// cluster, so the PP projection (pp_projection.py) can be pinned against simulate_iteration's
// own 1F1B timing (sim.cpp:180-275, 435-489). pp_i = {pp, layers_per_stage};
// pp_d = {fwd_bwd_ratio, comm_ms, dp_sync_ms}; out_res = {iter_ms, bubble_ms, critical_lb_ms,
// max_mb_ms, mean_mb_ms, imbalance, avg_budget, mean_cov_drop}.
SB_EXPORT int SBH(ref_simulate_iteration)(int strategy, int n, const int64_t* ids, const int64_t* lengths,
                                          const double* profiles, const int64_t* off, const int* setup_i,
                                          const double* setup_d, int anchor, const int* dst_grid, int n_dst_grid,
                                          const int64_t* edges, int ne, double* ema_inout, double alpha,
                                          const int* est_grid, int n_est_grid, const int64_t* bins, int nx,
                                          const int* grid, int nk, const double* lat, int iter_index,
                                          const int* pp_i, const double* pp_d, double* out_res) {
  return guarded([&] {
    const int gbs = setup_i[0], mbs = setup_i[1], dp = setup_i[2];
    const int nl = pp_i[0] * pp_i[1];
    const auto samples = make_samples(n, ids, lengths, nl, profiles, off);
    const auto table = make_table(bins, nx, grid, nk, lat);
    auto est = make_est(edges, ne, ema_inout, alpha, est_grid, n_est_grid);
    sb::IterationSetup setup;
    setup.cluster.dp = dp;
    setup.cluster.pp = pp_i[0];
    setup.cluster.layers_per_stage = pp_i[1];
    setup.cluster.fwd_bwd_ratio = pp_d[0];
    setup.cluster.comm_ms = pp_d[1];
    setup.cluster.dp_sync_ms = pp_d[2];
    setup.shape = sb::PlanShape{gbs, mbs, dp};
    setup.base_budget = setup_i[4];
    setup.base_mode = setup_i[5] ? sb::BaseBudgetMode::kCoverage : sb::BaseBudgetMode::kFixed;
    setup.base_coverage_target = setup_d[0];
    setup.dst_scope = setup_i[6] ? sb::DstScope::kGlobal : sb::DstScope::kRank;
    setup.dst.threshold_p = setup_d[1];
    setup.dst.anchor = anchor_of(anchor);
    setup.dst.budget_grid.assign(dst_grid, dst_grid + n_dst_grid);
    setup.calibrate_every = setup_i[7];
    const auto r = sb::simulate_iteration(samples, static_cast<sb::Strategy>(strategy), setup, table, est, iter_index,
                                          nullptr, nullptr);
    const double v[8] = {r.iter_ms, r.bubble_ms, r.critical_lb_ms, r.max_mb_ms, r.mean_mb_ms, r.imbalance,
                         r.avg_budget, r.mean_cov_drop};
    std::memcpy(out_res, v, sizeof(v));
  });
}
#endif

SB_EXPORT int SBH(plan_step)(int strategy, int n, const int64_t* ids, const int64_t* lengths,
                             const double* profiles, const int64_t* off, const int* setup_i,
                             const double* setup_d, int anchor, const int* dst_grid,
                             int n_dst_grid, const int64_t* edges, int ne, double* ema_inout,
                             double alpha, const int* est_grid, int n_est_grid,
                             const int64_t* bins, int nx, const int* grid, int nk,
                             const double* lat, int iter_index, int* out_budgets,
                             int64_t* out_ids, int* out_mb_off, int* out_dec_i,
                             double* out_dec_d, int n_dec_cap, int* out_n_dec,
                             double* out_stats, const char* decisions_csv_path,
                             const char* plan_json_path) {
  return guarded([&] {
    const int gbs = setup_i[0], mbs = setup_i[1], dp = setup_i[2], nl = setup_i[3];
    const auto samples = make_samples(n, ids, lengths, nl, profiles, off);
    const auto table = make_table(bins, nx, grid, nk, lat);
    auto est = make_est(edges, ne, ema_inout, alpha, est_grid, n_est_grid);
    sb::DstConfig dcfg;
    dcfg.threshold_p = setup_d[1];
    dcfg.anchor = anchor_of(anchor);
    dcfg.budget_grid.assign(dst_grid, dst_grid + n_dst_grid);
#ifdef SB_REF
    if (setup_i[8] != 0) throw sb::ConfigError("plan_step: varlen cost is not in the reference");
#else
    dcfg.varlen_block_size = setup_i[8];
#endif
    if (strategy < 0 || strategy > 5) throw sb::ConfigError("plan_step: strategy out of range");
    const auto strat = static_cast<sb::Strategy>(strategy);
    const auto base_mode = setup_i[5] ? sb::BaseBudgetMode::kCoverage : sb::BaseBudgetMode::kFixed;
    const auto scope = setup_i[6] ? sb::DstScope::kGlobal : sb::DstScope::kRank;

    std::vector<sb::BudgetDecision> decisions;
    sb::PackingPlan plan;
    std::vector<std::vector<std::vector<int>>> budgets;
    double stats[2] = {0.0, 0.0};
#ifdef SB_REF
    sb::IterationSetup setup;
    setup.cluster.dp = dp;
    setup.cluster.pp = 1;
    setup.cluster.layers_per_stage = nl;
    setup.shape = sb::PlanShape{gbs, mbs, dp};
    setup.base_budget = setup_i[4];
    setup.base_mode = base_mode;
    setup.base_coverage_target = setup_d[0];
    setup.dst_scope = scope;
    setup.dst = dcfg;
    setup.calibrate_every = setup_i[7];
    const auto res = sb::simulate_iteration(samples, strat, setup, table, est, iter_index,
                                            &decisions, &plan);
    stats[0] = res.mean_cov_drop;
    stats[1] = res.avg_budget;
    // Rebuild the per-(rank, mb, layer) budgets the reference kept internally
    // (sim.cpp:312-343, then overwritten by decisions :406-413).
    const std::vector<int>& g = dcfg.budget_grid.empty() ? table.budget_grid : dcfg.budget_grid;
    std::vector<std::size_t> mb_count;
    for (int r = 0; r < dp; ++r) {
      auto gb = sb::assemble_global_batch(samples, plan, r, setup.base_budget);
      budgets.emplace_back();
      for (std::size_t i = 0; i < gb.micro_batches.size(); ++i) {
        int kb = gb.base_budgets[i];
        if (base_mode == sb::BaseBudgetMode::kCoverage)
          kb = sb::intrinsic_budget(gb.micro_batches[i], g, setup.base_coverage_target);
        budgets.back().emplace_back(static_cast<std::size_t>(nl), kb);
      }
      mb_count.push_back(gb.micro_batches.size());
    }
    std::size_t pos = 0;
    const int groups = scope == sb::DstScope::kGlobal ? 1 : dp;
    for (int gi = 0; gi < groups && !decisions.empty(); ++gi) {
      std::vector<std::pair<int, int>> origin;
      for (int r = 0; r < dp; ++r) {
        if (scope == sb::DstScope::kRank && r != gi) continue;
        for (std::size_t i = 0; i < mb_count[static_cast<std::size_t>(r)]; ++i)
          origin.emplace_back(r, static_cast<int>(i));
      }
      for (int l = 0; l < nl; ++l)
        for (std::size_t j = 0; j < origin.size(); ++j, ++pos) {
          const auto& d = decisions[pos];
          const auto [r, i] = origin[static_cast<std::size_t>(d.micro_batch_id)];
          budgets[static_cast<std::size_t>(r)][static_cast<std::size_t>(i)][static_cast<std::size_t>(l)] =
              d.k_final;
        }
    }
#else
    sb::StepSetup setup;
    setup.shape = sb::PlanShape{gbs, mbs, dp};
    setup.num_layers = nl;
    setup.base_budget = setup_i[4];
    setup.base_mode = base_mode;
    setup.base_coverage_target = setup_d[0];
    setup.dst_scope = scope;
    setup.dst = dcfg;
    setup.calibrate_every = setup_i[7];
    auto sp = sb::plan_step(samples, strat, setup, table, est, iter_index);
    decisions = std::move(sp.decisions);
    plan = std::move(sp.plan);
    budgets = std::move(sp.budgets);
    stats[0] = sp.mean_cov_drop;
    stats[1] = sp.avg_budget;
#endif
    // The step's replay files (decisions CSV dst.cpp:171-185, plan JSON sab.cpp:312-336),
    // written by this build's own write_decisions_csv / save_plan_json.
    if (decisions_csv_path != nullptr) sb::write_decisions_csv(decisions, iter_index, decisions_csv_path);
    if (plan_json_path != nullptr) sb::save_plan_json(plan, plan_json_path);
    if (static_cast<int>(decisions.size()) > n_dec_cap)
      throw sb::ConfigError("plan_step: decision capacity too small");
    *out_n_dec = static_cast<int>(decisions.size());
    for (std::size_t i = 0; i < decisions.size(); ++i) {
      const auto& d = decisions[i];
      int* oi = out_dec_i + 6 * i;
      oi[0] = d.micro_batch_id;
      oi[1] = d.layer_id;
      oi[2] = d.k_base;
      oi[3] = d.k_anchor;
      oi[4] = d.k_final;
      oi[5] = direction_code(d.direction);
      double* od = out_dec_d + 3 * i;
      od[0] = d.coverage_drop;
      od[1] = d.predicted_ms_base;
      od[2] = d.predicted_ms_final;
    }
    std::size_t bp = 0;
    for (const auto& r : budgets)
      for (const auto& m : r)
        for (int k : m) out_budgets[bp++] = k;
    write_plan(plan, out_ids, out_mb_off, nullptr);
    std::memcpy(ema_inout, est.ema_budget.data(), sizeof(double) * static_cast<std::size_t>(ne));
    out_stats[0] = stats[0];
    out_stats[1] = stats[1];
  });
}

}  // extern "C"
