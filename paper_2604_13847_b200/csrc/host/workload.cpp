// Workload hierarchy (semantics: reference proj/core/src/workload.cpp).
//
// Bit-exactness notes: merges and normalisations accumulate in the reference's order
// (member order, then block order; sums in index order) and the compile uses
// -ffp-contract=off, so merged profiles equal the reference's to the last bit.
#include "sparsebalance/workload.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <functional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <unordered_map>
#include <unordered_set>

#include "sparsebalance/errors.hpp"

namespace sparsebalance {

namespace {

constexpr int kTruncationAttempts = 256;  // workload.cpp:19

std::int64_t round_clamped(double v, std::int64_t lo, std::int64_t hi) {
  const auto r = static_cast<std::int64_t>(std::llround(v));
  return r < lo ? lo : (r > hi ? hi : r);
}

// Normalised gamma(alpha) scores in draw order (workload.cpp:42-57, before the sort).
std::vector<double> draw_scores(Rng& rng, std::int64_t length, int block_size, double alpha) {
  const auto m = static_cast<std::size_t>((length + block_size - 1) / block_size);
  std::vector<double> s(m);
  double sum = 0.0;
  for (std::size_t j = 0; j < m; ++j) {
    s[j] = rng.gamma(alpha);
    sum += s[j];
  }
  if (sum > 0.0) {
    for (double& v : s) v /= sum;
  } else {
    std::fill(s.begin(), s.end(), 1.0 / static_cast<double>(m));
  }
  return s;
}

std::vector<Sample> generate_impl(const LengthDistributionSpec& spec, std::int64_t count,
                                  const ConcentrationSpec& conc, int num_layers, int block_size,
                                  std::uint64_t seed, bool sorted) {
  if (count < 1) throw ConfigError("generate_samples: count must be >= 1");
  if (num_layers < 1) throw ConfigError("generate_samples: num_layers must be >= 1");
  if (block_size < 1) throw ConfigError("generate_samples: block_size must be >= 1");
  validate_distribution(spec);
  validate_concentration(conc);

  Rng rng(mix_seed(seed));
  std::vector<Sample> out;
  out.reserve(static_cast<std::size_t>(count));
  for (std::int64_t id = 0; id < count; ++id) {
    Sample s;
    s.id = id;
    s.length = sample_length(spec, rng);
    // Sequence-level concentration, then a per-layer lognormal perturbation
    // (workload.cpp:253-265).
    const double seq_alpha = rng.lognormal(conc.alpha_log_mean, conc.alpha_log_sigma) *
                             std::pow(conc.length_ref / static_cast<double>(s.length),
                                      conc.length_exponent);
    s.routing_profiles.resize(static_cast<std::size_t>(num_layers));
    for (int l = 0; l < num_layers; ++l) {
      double a = seq_alpha;
      if (conc.layer_log_sigma > 0.0) a *= rng.lognormal(0.0, conc.layer_log_sigma);
      a = std::clamp(a, 1e-4, 1e4);
      auto scores = draw_scores(rng, s.length, block_size, a);
      if (sorted) std::sort(scores.begin(), scores.end(), std::greater<double>());
      s.routing_profiles[static_cast<std::size_t>(l)].scores = std::move(scores);
    }
    out.push_back(std::move(s));
  }
  return out;
}

}  // namespace

MicroBatch make_micro_batch(std::vector<Sample> samples) {
  if (samples.empty()) throw ConfigError("micro-batch must contain at least one sample");
  MicroBatch mb;
  mb.samples = std::move(samples);
  for (const Sample& s : mb.samples) mb.length_descriptor += s.length;

  const std::size_t layers = mb.samples.front().routing_profiles.size();
  for (const Sample& s : mb.samples) {
    if (s.routing_profiles.size() != layers) {
      throw ConfigError("micro-batch members disagree on layer count");
    }
  }
  const double total_tokens = static_cast<double>(mb.length_descriptor);
  mb.merged_profiles.resize(layers);
  for (std::size_t l = 0; l < layers; ++l) {
    std::size_t width = 0;
    for (const Sample& s : mb.samples) width = std::max(width, s.routing_profiles[l].scores.size());
    std::vector<double> acc(width, 0.0);
    // Token-weighted sum, zero-padded to the widest member.
    for (const Sample& s : mb.samples) {
      const double w = static_cast<double>(s.length) / total_tokens;
      const std::vector<double>& src = s.routing_profiles[l].scores;
      for (std::size_t j = 0; j < src.size(); ++j) acc[j] += w * src[j];
    }
    double norm = 0.0;
    for (double v : acc) norm += v;
    if (norm > 0.0) {
      for (double& v : acc) v /= norm;
    }
    std::sort(acc.begin(), acc.end(), std::greater<double>());
    mb.merged_profiles[l].scores = std::move(acc);
  }
  return mb;
}

const char* distribution_kind_name(LengthDistributionSpec::Kind kind) {
  using K = LengthDistributionSpec::Kind;
  switch (kind) {
    case K::kFixed: return "fixed";
    case K::kBimodal: return "bimodal";
    case K::kLongTail: return "long_tail";
    case K::kHistogram: return "histogram";
  }
  return "?";
}

LengthDistributionSpec::Kind parse_distribution_kind(const std::string& name) {
  using K = LengthDistributionSpec::Kind;
  static const std::pair<const char*, K> table[] = {
      {"fixed", K::kFixed}, {"bimodal", K::kBimodal}, {"long_tail", K::kLongTail},
      {"histogram", K::kHistogram}};
  for (const auto& [n, k] : table) {
    if (name == n) return k;
  }
  throw ConfigError("distribution.kind: unknown kind '" + name +
                    "' (expected fixed|bimodal|long_tail|histogram)");
}

void validate_distribution(const LengthDistributionSpec& spec) {
  using K = LengthDistributionSpec::Kind;
  if (spec.min_length < 1) throw ConfigError("distribution.min_length: must be >= 1");
  if (spec.max_length < spec.min_length)
    throw ConfigError("distribution.max_length: must be >= min_length");
  if (spec.kind == K::kFixed) {
    if (spec.fixed_length < spec.min_length || spec.fixed_length > spec.max_length)
      throw ConfigError("distribution.fixed_length: outside [min_length, max_length]");
  } else if (spec.kind == K::kBimodal) {
    if (spec.short_weight < 0.0 || spec.short_weight > 1.0)
      throw ConfigError("distribution.short_weight: must be in [0,1]");
    if (spec.short_log_sigma < 0.0) throw ConfigError("distribution.short_log_sigma: must be >= 0");
    if (spec.long_log_sigma < 0.0) throw ConfigError("distribution.long_log_sigma: must be >= 0");
  } else if (spec.kind == K::kLongTail) {
    if (spec.tail_exponent <= 0.0) throw ConfigError("distribution.tail_exponent: must be > 0");
  } else {
    if (spec.bins.empty()) throw ConfigError("distribution.bins: histogram must be non-empty");
    double freq = 0.0;
    for (std::size_t i = 0; i < spec.bins.size(); ++i) {
      const HistogramBin& b = spec.bins[i];
      if (b.lo < 1 || b.hi <= b.lo)
        throw ConfigError("distribution.bins[" + std::to_string(i) + "]: requires 1 <= lo < hi");
      if (b.frequency < 0.0)
        throw ConfigError("distribution.bins[" + std::to_string(i) + "].frequency: must be >= 0");
      freq += b.frequency;
    }
    if (freq <= 0.0) throw ConfigError("distribution.bins: total frequency must be > 0");
  }
}

std::int64_t sample_length(const LengthDistributionSpec& spec, Rng& rng) {
  using K = LengthDistributionSpec::Kind;
  switch (spec.kind) {
    case K::kFixed:
      return spec.fixed_length;
    case K::kBimodal: {
      // Rejection into [min, max] with a bounded number of attempts (workload.cpp:26-36).
      auto draw = [&]() {
        const bool short_mode = rng.uniform01() < spec.short_weight;
        return short_mode ? rng.lognormal(spec.short_log_mean, spec.short_log_sigma)
                          : rng.lognormal(spec.long_log_mean, spec.long_log_sigma);
      };
      for (int attempt = 0; attempt < kTruncationAttempts; ++attempt) {
        const auto r = static_cast<std::int64_t>(std::llround(draw()));
        if (r >= spec.min_length && r <= spec.max_length) return r;
      }
      return round_clamped(draw(), spec.min_length, spec.max_length);
    }
    case K::kLongTail: {
      const double a = spec.tail_exponent;
      const double u = rng.uniform01();
      const double lo_p = std::pow(static_cast<double>(spec.min_length), -a);
      const double hi_p = std::pow(static_cast<double>(spec.max_length), -a);
      return round_clamped(std::pow(lo_p - u * (lo_p - hi_p), -1.0 / a), spec.min_length,
                           spec.max_length);
    }
    case K::kHistogram: {
      double total = 0.0;
      for (const HistogramBin& b : spec.bins) total += b.frequency;
      const double u = rng.uniform01() * total;
      std::size_t chosen = spec.bins.size() - 1;
      double run = 0.0;
      for (std::size_t i = 0; i < spec.bins.size(); ++i) {
        run += spec.bins[i].frequency;
        if (u < run) {
          chosen = i;
          break;
        }
      }
      return rng.uniform_int(spec.bins[chosen].lo, spec.bins[chosen].hi - 1);
    }
  }
  throw std::runtime_error("unreachable distribution kind");
}

void validate_concentration(const ConcentrationSpec& spec) {
  if (spec.alpha_log_sigma < 0.0) throw ConfigError("concentration.alpha_log_sigma: must be >= 0");
  if (spec.layer_log_sigma < 0.0) throw ConfigError("concentration.layer_log_sigma: must be >= 0");
  if (!(spec.length_ref > 0.0)) throw ConfigError("concentration.length_ref: must be > 0");
  if (spec.length_exponent < 0.0) throw ConfigError("concentration.length_exponent: must be >= 0");
  if (spec.drift_amplitude < 0.0) throw ConfigError("concentration.drift_amplitude: must be >= 0");
  if (spec.drift_period < 1) throw ConfigError("concentration.drift_period: must be >= 1");
}

ConcentrationSpec concentration_at(const ConcentrationSpec& spec, int iteration) {
  ConcentrationSpec now = spec;
  if (spec.drift_amplitude > 0.0) {
    const double phase = 6.283185307179586 * static_cast<double>(iteration) /
                         static_cast<double>(spec.drift_period);
    now.length_exponent =
        std::max(0.0, spec.length_exponent + spec.drift_amplitude * std::sin(phase));
  }
  return now;
}

std::vector<Sample> generate_samples(const LengthDistributionSpec& spec, std::int64_t count,
                                     const ConcentrationSpec& concentration, int num_layers,
                                     int block_size, std::uint64_t seed) {
  return generate_impl(spec, count, concentration, num_layers, block_size, seed, true);
}

std::vector<Sample> generate_samples_unsorted(const LengthDistributionSpec& spec,
                                              std::int64_t count,
                                              const ConcentrationSpec& concentration,
                                              int num_layers, int block_size,
                                              std::uint64_t seed) {
  return generate_impl(spec, count, concentration, num_layers, block_size, seed, false);
}

namespace {

std::string_view trim(std::string_view v) {
  const auto ws = [](char c) { return c == ' ' || c == '\t' || c == '\r'; };
  while (!v.empty() && ws(v.front())) v.remove_prefix(1);
  while (!v.empty() && ws(v.back())) v.remove_suffix(1);
  return v;
}

}  // namespace

LengthDistributionSpec load_histogram(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ConfigError("cannot open histogram file " + path);
  LengthDistributionSpec spec;
  spec.kind = LengthDistributionSpec::Kind::kHistogram;
  std::string raw;
  for (int line = 1; std::getline(in, raw); ++line) {
    const std::string_view v = trim(raw);
    if (v.empty() || v.front() == '#') continue;
    const auto where = [&] { return path + ":" + std::to_string(line) + ": "; };
    HistogramBin b;
    char sep1 = 0, sep2 = 0;
    std::istringstream fields{std::string(v)};
    const bool ok = static_cast<bool>(fields >> b.lo >> sep1 >> b.hi >> sep2 >> b.frequency) && sep1 == ',' &&
                    sep2 == ',' && (fields >> std::ws).eof();
    if (!ok) throw ConfigError(where() + "expected 'lo,hi,frequency', got '" + raw + "'");
    if (!(b.lo >= 1 && b.hi > b.lo)) throw ConfigError(where() + "bin bounds must satisfy 1 <= lo < hi");
    if (!(b.frequency >= 0.0)) throw ConfigError(where() + "bin frequency must be >= 0");
    spec.bins.push_back(b);
  }
  if (spec.bins.empty()) throw ConfigError("histogram file " + path + " has no bins");
  spec.min_length = spec.bins[0].lo;
  spec.max_length = spec.bins[0].hi - 1;
  for (const HistogramBin& b : spec.bins) {
    spec.min_length = std::min(spec.min_length, b.lo);
    spec.max_length = std::max(spec.max_length, b.hi - 1);
  }
  validate_distribution(spec);
  return spec;
}

void save_histogram(const std::vector<HistogramBin>& bins, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write histogram file " + path);
  out << "# lo_tokens,hi_tokens,frequency\n";
  for (const HistogramBin& b : bins) {
    char row[96];
    std::snprintf(row, sizeof(row), "%lld,%lld,%.6f\n", static_cast<long long>(b.lo), static_cast<long long>(b.hi),
                  b.frequency);
    out << row;
  }
  if (!out) throw std::runtime_error("write failed for histogram file " + path);
}

GlobalBatch assemble_global_batch(std::span<const Sample> samples, const PackingPlan& plan,
                                  int dp_rank, int base_budget) {
  if (dp_rank < 0 || static_cast<std::size_t>(dp_rank) >= plan.micro_batch_bins.size()) {
    throw ConfigError("assemble_global_batch: dp_rank " + std::to_string(dp_rank) +
                      " out of range for plan with " +
                      std::to_string(plan.micro_batch_bins.size()) + " ranks");
  }
  std::unordered_map<std::int64_t, std::size_t> index_of;
  index_of.reserve(samples.size());
  for (std::size_t i = 0; i < samples.size(); ++i) {
    if (!index_of.emplace(samples[i].id, i).second)
      throw ConfigError("assemble_global_batch: duplicate sample id " +
                        std::to_string(samples[i].id));
  }
  // Exact-cover check over all ranks (workload.cpp:286-320).
  std::unordered_set<std::int64_t> covered;
  covered.reserve(samples.size());
  for (const auto& rank : plan.micro_batch_bins) {
    for (const auto& mb : rank) {
      for (std::int64_t id : mb) {
        if (!index_of.count(id))
          throw ConfigError("assemble_global_batch: plan references unknown sample id " +
                            std::to_string(id));
        if (!covered.insert(id).second)
          throw ConfigError("assemble_global_batch: plan assigns sample id " +
                            std::to_string(id) + " more than once");
      }
    }
  }
  if (covered.size() != samples.size()) {
    for (const Sample& s : samples) {
      if (!covered.count(s.id))
        throw ConfigError("assemble_global_batch: plan omits sample id " + std::to_string(s.id));
    }
  }
  GlobalBatch gb;
  for (const auto& mb_ids : plan.micro_batch_bins[static_cast<std::size_t>(dp_rank)]) {
    std::vector<Sample> members;
    members.reserve(mb_ids.size());
    for (std::int64_t id : mb_ids) members.push_back(samples[index_of.at(id)]);
    gb.micro_batches.push_back(make_micro_batch(std::move(members)));
    gb.base_budgets.push_back(base_budget);
  }
  return gb;
}

int coverage_budget(const RoutingProfile& profile, double target) {
  double run = 0.0;
  const std::size_t m = profile.scores.size();
  for (std::size_t j = 0; j < m; ++j) {
    run += profile.scores[j];
    if (run >= target) return static_cast<int>(j) + 1;
  }
  return static_cast<int>(m);
}

int intrinsic_budget(const MicroBatch& mb, std::span<const int> budget_grid,
                     double coverage_target) {
  if (budget_grid.empty()) throw ConfigError("intrinsic_budget: empty budget grid");
  if (mb.merged_profiles.empty()) throw ConfigError("intrinsic_budget: micro-batch has no profiles");
  double mean_need = 0.0;
  for (const RoutingProfile& p : mb.merged_profiles)
    mean_need += static_cast<double>(coverage_budget(p, coverage_target));
  mean_need /= static_cast<double>(mb.merged_profiles.size());
  const int need = static_cast<int>(std::ceil(mean_need));
  // Snap up to the grid, cap at its maximum.
  for (int g : budget_grid) {
    if (g >= need) return g;
  }
  return budget_grid.back();
}

}  // namespace sparsebalance
