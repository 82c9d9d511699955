/* CPU restatement of the device half (see sb_oracle.h). TEST ORACLE / CPU BASELINE ONLY.
 * Straightforward loops, fp64 accumulation, OpenMP over independent (head, row) work. */
#include "sb_oracle.h"

#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>

int orc_set_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
}

static inline double bf(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return (double)f;
}

static inline int seq_len(const int32_t* cu, int s) { return cu[s + 1] - cu[s]; }

/* Mean of the valid rows of every (block, head). */
void orc_block_pool(const uint16_t* x, const int32_t* cu, const int32_t* blk_off, int nseq,
                    int heads, int d, int bsz, double* xbar) {
  for (int s = 0; s < nseq; ++s) {
    const int nb = blk_off[s + 1] - blk_off[s];
#pragma omp parallel for collapse(2) schedule(static)
    for (int i = 0; i < nb; ++i)
      for (int h = 0; h < heads; ++h) {
        const int t0 = cu[s] + i * bsz;
        int t1 = t0 + bsz;
        if (t1 > cu[s + 1]) t1 = cu[s + 1];
        double* out = xbar + ((size_t)(blk_off[s] + i) * heads + h) * d;
        for (int c = 0; c < d; ++c) out[c] = 0.0;
        for (int t = t0; t < t1; ++t)
          for (int c = 0; c < d; ++c) out[c] += bf(x[((size_t)t * heads + h) * d + c]);
        for (int c = 0; c < d; ++c) out[c] /= (double)(t1 - t0);
      }
  }
}

void orc_block_scores(const double* qbar, const double* kbar, const int32_t* blk_off,
                      const int64_t* tri_off, int nseq, int hq, int hkv, int d, double scale,
                      double* scores) {
  const int grp = hq / hkv;
  const int64_t tri = tri_off[nseq];
  for (int s = 0; s < nseq; ++s) {
    const int nb = blk_off[s + 1] - blk_off[s];
#pragma omp parallel for collapse(2) schedule(dynamic, 4)
    for (int h = 0; h < hq; ++h)
      for (int i = 0; i < nb; ++i) {
        const double* qb = qbar + ((size_t)(blk_off[s] + i) * hq + h) * d;
        double* row = scores + (size_t)h * tri + tri_off[s] + (int64_t)i * (i + 1) / 2;
        for (int j = 0; j <= i; ++j) {
          const double* kb = kbar + ((size_t)(blk_off[s] + j) * hkv + h / grp) * d;
          double acc = 0.0;
          for (int c = 0; c < d; ++c) acc += qb[c] * kb[c];
          row[j] = acc * scale;
        }
      }
  }
}

/* Canonical selection key: NaN -> -inf, -0.0 -> +0.0. */
static inline float canon(float x) {
  if (x != x) return -INFINITY;
  if (x == 0.0f) return 0.0f;
  return x;
}

typedef struct {
  float v;
  int j;
} cand_t;

static int cand_cmp(const void* a, const void* b) {
  const cand_t* x = (const cand_t*)a;
  const cand_t* y = (const cand_t*)b;
  if (x->v > y->v) return -1;
  if (x->v < y->v) return 1;
  return x->j < y->j ? -1 : (x->j > y->j);
}

static int int_cmp(const void* a, const void* b) {
  return *(const int*)a - *(const int*)b;
}

void orc_topk_select(const float* scores, const int32_t* blk_off, const int64_t* tri_off,
                     int nseq, int hs, int group, const int32_t* k_seq, int k_max,
                     int force_diag, int32_t* idx, int32_t* cnt) {
  const int hsel = hs / group;
  const int64_t tri = tri_off[nseq];
  const int nbt = blk_off[nseq];
  for (int s = 0; s < nseq; ++s) {
    const int nb = blk_off[s + 1] - blk_off[s];
#pragma omp parallel for collapse(2) schedule(dynamic, 8)
    for (int g = 0; g < hsel; ++g)
      for (int i = 0; i < nb; ++i) {
        const int n = i + 1;
        cand_t* c = (cand_t*)malloc(sizeof(cand_t) * (size_t)n);
        for (int j = 0; j < n; ++j) {
          float acc = 0.0f;
          for (int q = 0; q < group; ++q) {
            const float* row = scores + (size_t)(g * group + q) * tri + tri_off[s] + (int64_t)i * (i + 1) / 2;
            acc = (q == 0) ? row[j] : acc + row[j];
          }
          c[j].v = canon(acc);
          c[j].j = j;
        }
        int k = k_seq[s] < n ? k_seq[s] : n;
        if (k < 1) k = 1;
        int* sel = (int*)malloc(sizeof(int) * (size_t)k);
        int ns = 0;
        if (force_diag) {
          sel[ns++] = i;
          qsort(c, (size_t)(n - 1), sizeof(cand_t), cand_cmp); /* candidates j < i */
          for (int r = 0; r < k - 1; ++r) sel[ns++] = c[r].j;
        } else {
          qsort(c, (size_t)n, sizeof(cand_t), cand_cmp);
          for (int r = 0; r < k; ++r) sel[ns++] = c[r].j;
        }
        qsort(sel, (size_t)ns, sizeof(int), int_cmp);
        int32_t* out = idx + ((size_t)g * nbt + blk_off[s] + i) * k_max;
        for (int r = 0; r < k_max; ++r) out[r] = r < ns ? sel[r] : -1;
        cnt[(size_t)g * nbt + blk_off[s] + i] = ns;
        free(sel);
        free(c);
      }
  }
}

static int dbl_desc(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x < y) - (x > y);
}

void orc_coverage_profile(const float* scores, const int32_t* blk_off, const int64_t* tri_off,
                          int nseq, int nb_max, int hs, double* profile) {
  const int64_t tri = tri_off[nseq];
  for (int s = 0; s < nseq; ++s) {
    const int nb = blk_off[s + 1] - blk_off[s];
    double* acc = profile + (size_t)s * nb_max;
    for (int r = 0; r < nb_max; ++r) acc[r] = 0.0;
    double* sorted = (double*)malloc(sizeof(double) * (size_t)nb * (size_t)hs * (size_t)nb);
#pragma omp parallel for collapse(2) schedule(dynamic, 8)
    for (int h = 0; h < hs; ++h)
      for (int i = 0; i < nb; ++i) {
        const float* row = scores + (size_t)h * tri + tri_off[s] + (int64_t)i * (i + 1) / 2;
        double* m = sorted + ((size_t)h * nb + i) * nb;
        double mx = -INFINITY;
        for (int j = 0; j <= i; ++j) mx = row[j] > mx ? row[j] : mx;
        double z = 0.0;
        for (int j = 0; j <= i; ++j) z += exp((double)row[j] - mx);
        for (int j = 0; j <= i; ++j) m[j] = exp((double)row[j] - mx) / z;
        qsort(m, (size_t)(i + 1), sizeof(double), dbl_desc);
      }
    for (int h = 0; h < hs; ++h)
      for (int i = 0; i < nb; ++i)
        for (int r = 0; r <= i; ++r) acc[r] += sorted[((size_t)h * nb + i) * nb + r];
    for (int r = 0; r < nb; ++r) acc[r] /= (double)hs * (double)nb;
    free(sorted);
  }
}

void orc_coverage_at_grid(const double* profile, const int32_t* blk_off, int nseq, int nb_max,
                          const int32_t* grid, int ngrid, double* cov) {
  for (int s = 0; s < nseq; ++s) {
    const int nb = blk_off[s + 1] - blk_off[s];
    for (int g = 0; g < ngrid; ++g) {
      const int k = grid[g];
      double c = 0.0;
      if (k <= 0) {
        c = 0.0;
      } else if (k >= nb) {
        c = 1.0;
      } else {
        for (int r = 0; r < k; ++r) c += profile[(size_t)s * nb_max + r];
      }
      cov[(size_t)s * ngrid + g] = c;
    }
  }
}

/* Visit the keys of query row t (q block i of sequence s) under selection list sel[0..n). */
#define FOR_KEYS(...)                                                                   \
  for (int r_ = 0; r_ < n; ++r_) {                                                     \
    const int j_ = sel[r_];                                                            \
    const int u0_ = cu[s] + j_ * bsz;                                                  \
    int u1_ = u0_ + bsz;                                                               \
    if (u1_ > cu[s + 1]) u1_ = cu[s + 1];                                              \
    if (j_ == i && u1_ > t + 1) u1_ = t + 1;                                           \
    for (int u = u0_; u < u1_; ++u) { __VA_ARGS__ }                                       \
  }

void orc_sparse_attn_fwd(const uint16_t* q, const uint16_t* k, const uint16_t* v,
                         const int32_t* cu, const int32_t* blk_off, int nseq, int total,
                         int hq, int hkv, int d, int bsz, const int32_t* idx, const int32_t* cnt,
                         int hsel, int k_max, double scale, double* o, double* lse) {
  const int grp = hq / hkv;
  const int sgrp = hq / hsel;
  const int nbt = blk_off[nseq];
  for (int s = 0; s < nseq; ++s) {
#pragma omp parallel for collapse(2) schedule(dynamic, 16)
    for (int h = 0; h < hq; ++h)
      for (int t = cu[s]; t < cu[s + 1]; ++t) {
        const int i = (t - cu[s]) / bsz;
        const int gi = blk_off[s] + i;
        const int32_t* sel = idx + ((size_t)(h / sgrp) * nbt + gi) * k_max;
        const int n = cnt[(size_t)(h / sgrp) * nbt + gi];
        const int kh = h / grp;
        const uint16_t* qt = q + ((size_t)t * hq + h) * d;
        double mx = -INFINITY;
        FOR_KEYS({
          const uint16_t* ku = k + ((size_t)u * hkv + kh) * d;
          double a = 0.0;
          for (int c = 0; c < d; ++c) a += bf(qt[c]) * bf(ku[c]);
          a *= scale;
          if (a > mx) mx = a;
        })
        double z = 0.0;
        double* ot = o + ((size_t)t * hq + h) * d;
        for (int c = 0; c < d; ++c) ot[c] = 0.0;
        FOR_KEYS({
          const uint16_t* ku = k + ((size_t)u * hkv + kh) * d;
          const uint16_t* vu = v + ((size_t)u * hkv + kh) * d;
          double a = 0.0;
          for (int c = 0; c < d; ++c) a += bf(qt[c]) * bf(ku[c]);
          const double p = exp(a * scale - mx);
          z += p;
          for (int c = 0; c < d; ++c) ot[c] += p * bf(vu[c]);
        })
        for (int c = 0; c < d; ++c) ot[c] /= z;
        lse[(size_t)h * total + t] = mx + log(z);
      }
  }
}

void orc_sparse_attn_bwd(const uint16_t* q, const uint16_t* k, const uint16_t* v,
                         const double* o, const uint16_t* d_o, const double* lse,
                         const int32_t* cu, const int32_t* blk_off, int nseq, int total, int hq,
                         int hkv, int d, int bsz, const int32_t* idx, const int32_t* cnt,
                         int hsel, int k_max, double scale, double* dq, double* dk, double* dv) {
  const int grp = hq / hkv;
  const int sgrp = hq / hsel;
  const int nbt = blk_off[nseq];
  const size_t kv_elems = (size_t)total * hkv * d;
  memset(dq, 0, sizeof(double) * (size_t)total * hq * d);
  memset(dk, 0, sizeof(double) * kv_elems);
  memset(dv, 0, sizeof(double) * kv_elems);
  const int nth = omp_get_max_threads();
  /* Thread-private dK/dV partials reduced in thread order afterwards: parallel over every
   * (head, query row) without races; deterministic for a fixed thread count. */
  double* part = (double*)calloc((size_t)nth * 2 * kv_elems, sizeof(double));
#pragma omp parallel
  {
    double* pdk = part + (size_t)omp_get_thread_num() * 2 * kv_elems;
    double* pdv = pdk + kv_elems;
#pragma omp for collapse(2) schedule(dynamic, 16)
    for (int h = 0; h < hq; ++h)
      for (int t = 0; t < total; ++t) {
        int s = 0;
        while (cu[s + 1] <= t) ++s;
        const int kh = h / grp;
        const int i = (t - cu[s]) / bsz;
        const int gi = blk_off[s] + i;
        const int32_t* sel = idx + ((size_t)(h / sgrp) * nbt + gi) * k_max;
        const int n = cnt[(size_t)(h / sgrp) * nbt + gi];
        const uint16_t* qt = q + ((size_t)t * hq + h) * d;
        const uint16_t* dot = d_o + ((size_t)t * hq + h) * d;
        const double* ot = o + ((size_t)t * hq + h) * d;
        double* dqt = dq + ((size_t)t * hq + h) * d;
        double D = 0.0;
        for (int c = 0; c < d; ++c) D += bf(dot[c]) * ot[c];
        const double L = lse[(size_t)h * total + t];
        FOR_KEYS({
          const uint16_t* ku = k + ((size_t)u * hkv + kh) * d;
          const uint16_t* vu = v + ((size_t)u * hkv + kh) * d;
          double a = 0.0, dp = 0.0;
          for (int c = 0; c < d; ++c) {
            a += bf(qt[c]) * bf(ku[c]);
            dp += bf(dot[c]) * bf(vu[c]);
          }
          const double p = exp(a * scale - L);
          const double ds = p * (dp - D);
          double* dku = pdk + ((size_t)u * hkv + kh) * d;
          double* dvu = pdv + ((size_t)u * hkv + kh) * d;
          for (int c = 0; c < d; ++c) {
            dqt[c] += scale * ds * bf(ku[c]);
            dku[c] += scale * ds * bf(qt[c]);
            dvu[c] += p * bf(dot[c]);
          }
        })
      }
  }
  for (int th = 0; th < nth; ++th) {
    const double* pdk = part + (size_t)th * 2 * kv_elems;
    const double* pdv = pdk + kv_elems;
    for (size_t e = 0; e < kv_elems; ++e) {
      dk[e] += pdk[e];
      dv[e] += pdv[e];
    }
  }
  free(part);
}
