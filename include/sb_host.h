/* sparsebalance-b200: flat C ABI over the host decision layer (cost model, tuner, batcher).
 *
 * Every entry point mirrors one function of the reference's C++ API
 * (proj/core/include/sparsebalance/{profile_table,dst,sab,workload,sim}.hpp); the
 * C++ API itself is in include/sparsebalance/*.hpp with identical names and signatures.
 * This flat layer exists so that non-C++ callers (ctypes / cgo / JNI) can bind the host
 * half with plain pointers. Symbols are prefixed `sbh_`. The test oracle builds the same
 * shim source against the reference sources with prefix `sbref_` (oracle/Makefile), so
 * both sides are marshalled identically.
 *
 * Return codes (reference exit-code convention, commands.cpp:325-336):
 *   0 ok, 1 invalid argument (ConfigError), 2 runtime error. sbh_last_error() returns the
 *   message of the last failure on the calling thread.
 *
 * Tables are passed as (length_bins[nx], budget_grid[nk], latency_ms[nx*nk] row-major).
 * Profiles are concatenated vectors with int64 offsets (off[i]..off[i+1]).
 */
#ifndef SB_HOST_H_
#define SB_HOST_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#ifndef SB_HOST_PREFIX
#define SB_HOST_PREFIX sbh_
#endif
#define SB_HCAT2(a, b) a##b
#define SB_HCAT(a, b) SB_HCAT2(a, b)
#define SBH(name) SB_HCAT(SB_HOST_PREFIX, name)

const char* SBH(last_error)(void);

/* profile_table.hpp: predict / align / synthesize_table / load_table / save_table */
int SBH(predict)(const int64_t* bins, int nx, const int* grid, int nk, const double* lat,
                 int64_t x, int k, double* out_ms, int* out_extrapolated);
int SBH(align)(const int64_t* bins, int nx, const int* grid, int nk, const double* lat,
               int64_t x, double target_ms, int* out_budget, int* out_infeasible);
int SBH(synthesize_table)(double c_lin, double c_attn, double c_fixed, double noise_sigma,
                          int block_size, const int64_t* bins, int nx, const int* grid, int nk,
                          uint64_t seed, double* out_lat);
/* Two-phase: call with out arrays NULL to get *nx,*nk; then again with buffers. */
int SBH(load_table)(const char* path, int* nx, int* nk, int64_t* out_bins, int* out_grid,
                    double* out_lat, int* out_repaired_cells);
int SBH(save_table)(const char* path, const int64_t* bins, int nx, const int* grid, int nk,
                    const double* lat);

/* dst.hpp */
int SBH(coverage)(const double* scores, int m, int k, double* out);
int SBH(select_anchor)(const double* lat, int n, int anchor /*0 min,1 mean,2 max*/, double* out);
/* tune_global_batch for one layer of n_mb micro-batches whose layer profile is given.
 * out_i[n_mb][5] = {micro_batch_id, k_base, k_anchor, k_final, direction(0 comp,1 exp,2 unch)}
 * out_d[n_mb][3] = {coverage_drop, predicted_ms_base, predicted_ms_final} */
int SBH(tune_global_batch)(const int64_t* bins, int nx, const int* grid, int nk,
                           const double* lat, int n_mb, const int64_t* x, const int* k_base,
                           const double* profiles, const int64_t* prof_off, int layer,
                           double threshold_p, int anchor, const int* dst_grid, int n_dst_grid,
                           int* out_i, double* out_d);

/* workload.hpp */
/* Members' per-layer profiles: sample-major, off[(s*nl)+l]. Output merged profile per layer
 * into out (capacity cap doubles), out_off[nl+1]. */
int SBH(make_micro_batch)(int ns, const int64_t* lengths, int nl, const double* profiles,
                          const int64_t* off, double* out, int64_t cap, int64_t* out_off,
                          int64_t* out_length_descriptor);
#ifndef SB_REF
/* Extension, not in the reference (dst.hpp CoverageTable): the {x, k_base, C(K) per layer}
 * workload estimate DP ranks all-gather instead of their profiles.
 * coverage_table: out[g] = coverage(profile, grid[g]) for g < n_grid, out[n_grid] =
 * coverage(profile, k_base). tune_global_batch_cov: tune_global_batch for one layer with
 * cov[n_mb][n_dst_grid + 1] laid out as coverage_table writes it (k_base of micro-batch i
 * in k_base[i]); member lengths (mem_len, offsets mem_off[n_mb + 1]) are read only when
 * varlen_block_size > 0. Outputs as tune_global_batch. Decisions are bit-identical to
 * tune_global_batch on the profiles the tables were made from. */
int SBH(coverage_table)(const double* scores, int m, const int* grid, int n_grid, int k_base, double* out);
int SBH(tune_global_batch_cov)(const int64_t* bins, int nx, const int* grid, int nk, const double* lat,
                               int n_mb, const int64_t* x, const int* k_base, const double* cov,
                               const int64_t* mem_len, const int64_t* mem_off, int varlen_block_size, int layer,
                               double threshold_p, int anchor, const int* dst_grid, int n_dst_grid, int* out_i,
                               double* out_d);
/* The same two steps batched for a DP rank / step: rank_estimate = make_micro_batch +
 * (coverage-mode) intrinsic_budget + a coverage table per layer (profiles member-major,
 * profiles[s * nl + l]; out_cov[nl][n_grid + 1]); tune_layers_cov = tune_global_batch_cov
 * for layers 0..nl-1 (cov[n_mb][nl][n_dst_grid + 1] -> out_k_final[n_mb][nl], out_i[nl][n_mb][5],
 * out_d[nl][n_mb][3]). */
int SBH(rank_estimate)(int ns, const int64_t* lengths, int nl, const double* profiles, const int64_t* off,
                       const int* grid, int n_grid, int coverage_mode, int base_budget, double coverage_target,
                       int64_t* out_x, int* out_k_base, double* out_cov);
int SBH(tune_layers_cov)(const int64_t* bins, int nx, const int* grid, int nk, const double* lat, int n_mb,
                         const int64_t* x, const int* k_base, const double* cov, const int64_t* mem_len,
                         const int64_t* mem_off, int varlen_block_size, int nl, double threshold_p, int anchor,
                         const int* dst_grid, int n_dst_grid, int* out_k_final, int* out_i, double* out_d);
#endif
int SBH(coverage_budget)(const double* scores, int m, double target, int* out);
int SBH(intrinsic_budget)(int nl, const double* profiles, const int64_t* off, const int* grid,
                          int ng, double target, int* out);
/* kind: 0 fixed, 1 bimodal, 2 long_tail (histogram not exposed).
 * dist[9] = {min, max, fixed, short_w, short_mu, short_sigma, long_mu, long_sigma, tail_exp}
 * conc[5] = {alpha_mu, alpha_sigma, layer_sigma, length_ref, length_exp}
 * sorted=1: reference generate_samples; sorted=0: same stream, pre-sort (draw order).
 * Pass out_profiles NULL to obtain lengths + offsets only. */
int SBH(generate_samples)(int kind, const double* dist, const double* conc, int64_t count,
                          int num_layers, int block_size, uint64_t seed, int sorted,
                          int64_t* out_lengths, int64_t* out_off, double* out_profiles);

/* sab.hpp */
int SBH(default_bin_edges)(int64_t max_length, int64_t* out, int cap, int* out_n);
int SBH(estimate_sparsity)(const int64_t* edges, int ne, const double* ema, const int* grid,
                           int ng, int64_t length, int* out);
int SBH(calibrate)(const int64_t* edges, int ne, double* ema_inout, double alpha,
                   const int* grid, int ng, int n, const int* k_final, const int64_t* lengths);
/* out_items[n] lists item indices bin by bin (each bin ascending); out_bin_off[num_bins+1]. */
int SBH(bin_packing)(const double* weights, int n, int num_bins, int max_items_per_bin,
                     int* out_items, int* out_bin_off);
/* strategy: 0 sab (plan_batching), 1 lbb, 2 sequential.
 * out_ids[gbs] = sample ids rank-major then micro-batch-major; out_mb_off[dp*mpr+1];
 * out_weights[gbs] = plan weights in input order. */
int SBH(plan_batching)(int strategy, int n, const int64_t* ids, const int64_t* lengths,
                       int gbs, int mbs, int dp, const int64_t* edges, int ne, const double* ema,
                       double alpha, const int* est_grid, int n_est_grid, const int64_t* bins,
                       int nx, const int* grid, int nk, const double* lat, int64_t* out_ids,
                       int* out_mb_off, double* out_weights);

/* step.hpp: plan_step (reference: the decision half of simulate_iteration).
 * samples: n = gbs, ids, lengths, profiles sample-major with off[(s*nl)+l].
 * setup_i[9] = {gbs, mbs, dp, num_layers, base_budget, base_mode(0 fixed,1 coverage),
 *               dst_scope(0 rank,1 global), calibrate_every, varlen_block_size (0 = the
 *               reference's summed-length cost; > 0 = predict_members at that block size)}
 * setup_d[2] = {base_coverage_target, threshold_p}; anchor 0/1/2; dst grid (may be empty).
 * estimator: edges[ne], ema_inout[ne], alpha, est grid.
 * Outputs: out_budgets[dp * mpr * nl] ([rank][mb][layer]); out_ids / out_mb_off as in
 * plan_batching; decisions (cap n_dec_cap) out_dec_i[.][6] = {mb, layer, k_base, k_anchor,
 * k_final, direction}, out_dec_d[.][3]; *out_n_dec. out_stats[2] = {mean_cov_drop,
 * avg_budget}. decisions_csv_path / plan_json_path (nullable): the step's replay files in
 * the reference formats (write_decisions_csv dst.cpp:171-185 with iter = iter_index,
 * save_plan_json sab.cpp:312-336). */
/* Varlen-aware micro-batch cost (opt-in, not in the reference):
 * sum over members of predict(L_s, min(k, ceil(L_s / block_size))). */
int SBH(predict_members)(const int64_t* bins, int nx, const int* grid, int nk, const double* lat,
                         const int64_t* lengths, int n, int k, int block_size, double* out_ms,
                         int* out_extrapolated);

int SBH(plan_step)(int strategy, int n, const int64_t* ids, const int64_t* lengths,
                   const double* profiles, const int64_t* off, const int* setup_i,
                   const double* setup_d, int anchor, const int* dst_grid, int n_dst_grid,
                   const int64_t* edges, int ne, double* ema_inout, double alpha,
                   const int* est_grid, int n_est_grid, const int64_t* bins, int nx,
                   const int* grid, int nk, const double* lat, int iter_index, int* out_budgets,
                   int64_t* out_ids, int* out_mb_off, int* out_dec_i, double* out_dec_d,
                   int n_dec_cap, int* out_n_dec, double* out_stats,
                   const char* decisions_csv_path, const char* plan_json_path);

#ifdef __cplusplus
}
#endif

#endif /* SB_HOST_H_ */
