/* sparsebalance-b200: C ABI of the sm_100a hot-path kernels (block scorer, top-k selector,
 * coverage profile, varlen block-sparse attention forward / backward).
 *
 * The reference has no device implementation of this path (SPEC.md:8 puts "Eqs. 1-2
 * attention math executed on tensors" out of scope); each entry point below REPLACES a
 * reference stand-in, cited per function. Semantics follow Eq. 2 of the paper
 * with MoBA mean-of-key-block gating and the block
 * geometry m = ceil(L / B) of the reference (workload.cpp:43).
 *
 * Conventions
 *  - All pointers are caller-owned DEVICE memory unless named *_host. bf16 tensors are
 *    passed as uint16_t*. No allocation and no host synchronisation inside any call; every
 *    call is asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream).
 *  - A workspace belongs to one call at a time: the attention kernels keep their work order
 *    and a work-claiming cursor in it (reset inside the call), so calls that may overlap in
 *    time (different streams) need separate workspaces. Results do not depend on which CTA
 *    claims which work item: outputs are bit-identical run to run.
 *  - Packed varlen batch: cu_seqlens int32 [nseq+1] (cu[0] = 0, T = cu[nseq]).
 *    Block size B in {64, 128}; nb_s = ceil(L_s / B).
 *    blk_off int32 [nseq+1]: prefix sums of nb_s (NB = blk_off[nseq] blocks in total).
 *    tri_off int64 [nseq+1]: prefix sums of nb_s (nb_s + 1) / 2 (TRI = tri_off[nseq]).
 *    sb_block_layout_host() computes both from a host copy of cu_seqlens.
 *  - Tensors: Q [T][Hq][D], K,V [T][Hkv][D], O,dO,dQ [T][Hq][D], dK,dV [T][Hkv][D] (bf16,
 *    row stride = H*D elements), LSE fp32 [Hq][T] (natural log), D in {64, 128}.
 *  - Block scores S fp32 [Hs][TRI]: row (s, i) of head h starts at tri_off[s] + i(i+1)/2 and
 *    holds key blocks j = 0..i of the same sequence.
 *  - Selections idx int32 [Hsel][NB][k_max] (ascending block indices j, local to the sequence,
 *    padded with -1), cnt int32 [Hsel][NB]. Hsel = Hq (per-head selection) or Hkv
 *    (GQA group-shared selection); q head h uses selection row h / (Hq / Hsel).
 *  - Return codes (reference exit-code convention, commands.cpp:325-336): 0 ok,
 *    1 invalid argument, 2 CUDA / runtime error; sb_last_error() gives the message of the
 *    calling thread's last failure.
 */
#ifndef SB_KERNELS_H_
#define SB_KERNELS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* sb_last_error(void);

/* Host helper: blk_off / tri_off from host cu_seqlens. Returns NB in *nb_total, TRI in
 * *tri_total and max nb_s in *nb_max. */
int sb_block_layout_host(const int32_t* cu_seqlens_host, int nseq, int block_size,
                         int32_t* blk_off_host, int64_t* tri_off_host, int* nb_total,
                         int64_t* tri_total, int* nb_max);

/* K1: mean-pool every (block, head) of X [T][H][D] over its valid rows -> Xbar fp32
 * [NB][H][D]. Used for K (K-bar, MoBA gate keys) and Q (Q-bar).
 * Replaces: the routing-score synthesis of generate_samples / draw_profile
 * (reference workload.cpp:42-60, :239-271). */
int sb_block_pool(const uint16_t* x, const int32_t* cu_seqlens, const int32_t* blk_off, int nseq,
                  int nb_total, int heads, int head_dim, int block_size, float* xbar,
                  void* stream);

/* K2: S[h][row(s,i)][j] = scale * <Qbar[s,i,h], Kbar[s,j,h / (Hq/Hkv)]> for j <= i
 * (head_dim 64 or 128; fp32 fma over d in order).
 * Replaces: the RoutingProfile score vectors (reference workload.hpp:15-22). */
int sb_block_scores(const float* qbar, const float* kbar, const int32_t* blk_off,
                    const int64_t* tri_off, int nseq, int nb_max, int hq, int hkv, int head_dim,
                    float scale, float* scores, void* stream);

/* K3: per selection row (hs, s, i): keep k = max(1, min(k_seq[s], i + 1, k_max)) blocks (k_max is
 * the idx row stride; a larger k_seq is clamped, never written past the row). force_diag=1
 * (causal MoBA): block i always, then the top-(k-1) of j < i; force_diag=0: top-k of j <= i.
 * Order: score descending, ties to the lower j; NaN ranks as -inf and -0.0 as +0.0.
 * group = Hs / Hsel score heads are summed (in head order, fp32) per selection row.
 * Output indices ascending, padded with -1 up to k_max.
 * Replaces: "top-K blocks" = the sorted profile prefix consumed by coverage()
 * (reference workload.cpp:58, dst.cpp:53-61). */
int sb_topk_select(const float* scores, const int32_t* blk_off, const int64_t* tri_off, int nseq,
                   int nb_total, int nb_max, int hs, int group, const int32_t* k_seq, int k_max, int force_diag,
                   int32_t* idx, int32_t* cnt, void* stream);

/* K4a: routing profile per sequence as the DST consumes it: for every score row, softmax over
 * its i+1 entries, sorted descending; profile[s][r] = mean over (head, row) of the r-th
 * largest mass (rows shorter than r+1 contribute 0). Sum = 1, non-increasing, nb_s entries;
 * coverage(profile, k) is then the mean top-k mass. profile fp64 [nseq][nb_max] (zero
 * padded). workspace: sb_coverage_profile_workspace_size() bytes.
 * Replaces: RoutingProfile of a sequence-layer (reference workload.hpp:15-22) fed to
 * make_micro_batch / coverage / intrinsic_budget. */
size_t sb_coverage_profile_workspace_size(int64_t tri_total, int hs, int nseq, int nb_max);
int sb_coverage_profile(const float* scores, const int32_t* blk_off, const int64_t* tri_off,
                        int nseq, int nb_total, int64_t tri_total, int nb_max, int hs, void* workspace,
                        double* profile, void* stream);

/* K4b: C[s][g] = coverage(profile[s], grid[g]) exactly as reference dst.cpp:53-61
 * (sequential double sum; 0 for k <= 0; 1 for k >= nb_s). */
int sb_coverage_at_grid(const double* profile, const int32_t* blk_off, int nseq, int nb_max,
                        const int32_t* grid, int ngrid, double* coverage, void* stream);

/* K8: on-device DST decision, fixed-base mode. For micro-batch i =
 * sequences [mb_off[i], mb_off[i+1]): merges the members' K4 profiles (profile [nseq][nb_max],
 * one layer) exactly as make_micro_batch (workload.cpp:64-99) and applies tune_budget's rule
 * (dst.cpp:107-143) with the host-precomputed k_base[i], k_anchor[i] = align(x_i, anchor) and
 * bottleneck[i] = (predict(x_i, k_base_i) > anchor): k_final[i], coverage_drop[i] bit-exact
 * with the host, and k_seq[s] = min(k_final, nb_s) for the selector. Device pointers. */
int sb_dst_decide(const double* profile, const int32_t* blk_off, const int32_t* cu_seqlens, int nb_max,
                  const int32_t* mb_off, int n_mb, const int32_t* k_base, const int32_t* k_anchor,
                  const int32_t* bottleneck, const int32_t* grid, int ngrid, double threshold_p,
                  int32_t* k_final, double* coverage_drop, int32_t* k_seq, void* stream);

/* K5: O = softmax(scale * Q K[I]^T) V[I] over the selected blocks of each q block, causal
 * inside the diagonal block, keys beyond the sequence end masked. Saves LSE (natural log).
 * tcgen05/TMEM tensor-core kernel with TMA-loaded K/V blocks; persistent, longest-item-first
 * (workspace: sb_sparse_attn_fwd_workspace_size() bytes for the work order).
 * Replaces: predict()-based attention latency in micro_batch_time (reference sim.cpp:88-98). */
size_t sb_sparse_attn_fwd_workspace_size(int nb_total, int hq, int k_max);
/* Workspace for any block size, including 256 (the paper's MoBA B = 256): a
 * B = 256 selection runs on the B = 128 kernels through an exact re-expression over 128-row /
 * 128-key sub-tiles (expand256.cu), whose index lists live in this workspace. */
size_t sb_sparse_attn_fwd_workspace_size_ex(int nseq, int nb_total, int hq, int hsel, int k_max, int block_size);
int sb_sparse_attn_fwd(const uint16_t* q, const uint16_t* k, const uint16_t* v,
                       const int32_t* cu_seqlens, const int32_t* blk_off, int nseq, int total_tokens,
                       int nb_total, int hq, int hkv, int head_dim, int block_size,
                       const int32_t* idx, const int32_t* cnt, int hsel, int k_max, float scale,
                       uint16_t* o, float* lse, void* workspace, void* stream);

/* K5 with the bf16 rounding residual of O: o_res = bf16(O - bf16(O)) (NULL: not written). Fed to
 * sb_sparse_attn_bwd_ex, it makes D = rowsum(dO * O) accurate to ~2^-16 instead of bf16 (dS on
 * rows that attend few keys is a difference of nearly equal terms; see tests/tolerance.py). */
int sb_sparse_attn_fwd_ex(const uint16_t* q, const uint16_t* k, const uint16_t* v,
                          const int32_t* cu_seqlens, const int32_t* blk_off, int nseq, int total_tokens,
                          int nb_total, int hq, int hkv, int head_dim, int block_size,
                          const int32_t* idx, const int32_t* cnt, int hsel, int k_max, float scale,
                          uint16_t* o, uint16_t* o_res, float* lse, void* workspace, void* stream);

/* K6 (+K7): dQ, dK, dV from dO with P recomputed from the saved LSE; D = rowsum(dO * O).
 * K/V gradients accumulate over the q heads of each GQA group and over every q block that
 * selected the key block (deterministic: a kv-major pass over the transposed selection).
 * Replaces: fwd_bwd_ratio (reference sim.hpp:23, sim.cpp:97). */
size_t sb_sparse_attn_bwd_workspace_size(int total_tokens, int nb_total, int hq, int hkv,
                                         int head_dim, int hsel, int k_max);
size_t sb_sparse_attn_bwd_workspace_size_ex(int nseq, int total_tokens, int nb_total, int hq, int hkv,
                                            int head_dim, int hsel, int k_max, int block_size, int flags);
int sb_sparse_attn_bwd(const uint16_t* q, const uint16_t* k, const uint16_t* v,
                       const uint16_t* o, const uint16_t* d_o, const float* lse,
                       const int32_t* cu_seqlens, const int32_t* blk_off, int nseq,
                       int total_tokens, int nb_total, int hq, int hkv, int head_dim,
                       int block_size, const int32_t* idx, const int32_t* cnt, int hsel,
                       int k_max, float scale, uint16_t* dq, uint16_t* dk, uint16_t* dv,
                       void* workspace, void* stream);

/* K6 with flags. Default (flags = 0) and SB_BWD_DETERMINISTIC: the two-pass backward (dK/dV
 * pass over the transposed selection, then a dQ pass; 7 UMMAs per pair; bit-identical run to
 * run). SB_BWD_FUSED (d = B = 128 only; other shapes ignore it): the single pass with 5 UMMAs per
 * pair whose dQ partials are TMA-reduce-added in fp32 (reproducible to summation order). On B200
 * the fused pass is shared-memory-bandwidth bound (SS dQ operands + fp32 dQ staging: ~480 KB of
 * shared-memory traffic per pair vs ~420 KB for both two-pass kernels together, K6) and
 * measures slower, so it is opt-in. sb_sparse_attn_bwd == sb_sparse_attn_bwd_ex(..., flags = 0).
 * Same workspace size. */
#define SB_BWD_DETERMINISTIC 1
#define SB_BWD_FUSED 2
int sb_sparse_attn_bwd_ex(const uint16_t* q, const uint16_t* k, const uint16_t* v,
                          const uint16_t* o, const uint16_t* o_res /* may be NULL */,
                          const uint16_t* d_o, const float* lse,
                          const int32_t* cu_seqlens, const int32_t* blk_off, int nseq,
                          int total_tokens, int nb_total, int hq, int hkv, int head_dim,
                          int block_size, const int32_t* idx, const int32_t* cnt, int hsel,
                          int k_max, float scale, uint16_t* dq, uint16_t* dk, uint16_t* dv,
                          void* workspace, void* stream, int flags);

/* Diagnostics: number of hot-path kernel launches issued by this library since load. */
uint64_t sb_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* SB_KERNELS_H_ */
