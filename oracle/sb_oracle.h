/* CPU restatement (fp64 accumulation) of the device half of the hot path. TEST ORACLE and
 * CPU baseline only -- never linked into the product library.
 *
 * Parity status: the reference has NO implementation of the scorer, selector or attention
 * (SPEC.md:8), so these functions restate the paper's semantics -- Eq. 2,
 * MoBA mean-of-key-block gating, block geometry m = ceil(L/B)
 * (workload.cpp:43), dense when k >= m (dst.cpp:58-59), coverage as the sequential prefix sum
 * (dst.cpp:53-61) -- and are pinned by the reference only where it has data: the selector and
 * coverage against the reference's own routing-score vectors (tests/golden). Layouts match
 * include/sb_kernels.h, but every array here is HOST memory.
 */
#ifndef SB_ORACLE_H_
#define SB_ORACLE_H_
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int orc_set_threads(int n);

void orc_block_pool(const uint16_t* x, const int32_t* cu, const int32_t* blk_off, int nseq,
                    int heads, int d, int bsz, double* xbar);

void orc_block_scores(const double* qbar, const double* kbar, const int32_t* blk_off,
                      const int64_t* tri_off, int nseq, int hq, int hkv, int d, double scale,
                      double* scores);

void orc_topk_select(const float* scores, const int32_t* blk_off, const int64_t* tri_off,
                     int nseq, int hs, int group, const int32_t* k_seq, int k_max,
                     int force_diag, int32_t* idx, int32_t* cnt);

void orc_coverage_profile(const float* scores, const int32_t* blk_off, const int64_t* tri_off,
                          int nseq, int nb_max, int hs, double* profile);

void orc_coverage_at_grid(const double* profile, const int32_t* blk_off, int nseq, int nb_max,
                          const int32_t* grid, int ngrid, double* cov);

void orc_sparse_attn_fwd(const uint16_t* q, const uint16_t* k, const uint16_t* v,
                         const int32_t* cu, const int32_t* blk_off, int nseq, int total,
                         int hq, int hkv, int d, int bsz, const int32_t* idx, const int32_t* cnt,
                         int hsel, int k_max, double scale, double* o, double* lse);

void orc_sparse_attn_bwd(const uint16_t* q, const uint16_t* k, const uint16_t* v,
                         const double* o, const uint16_t* d_o, const double* lse,
                         const int32_t* cu, const int32_t* blk_off, int nseq, int total, int hq,
                         int hkv, int d, int bsz, const int32_t* idx, const int32_t* cnt,
                         int hsel, int k_max, double scale, double* dq, double* dk, double* dv);

#ifdef __cplusplus
}
#endif
#endif
