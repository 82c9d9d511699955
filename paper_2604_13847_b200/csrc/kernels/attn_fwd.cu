// K5: varlen block-sparse attention forward on tcgen05 / TMEM (Eq. 2).
//
// Persistent kernel: one CTA per SM walks a longest-first list of work items (one item = one
// q block x q head: a 128-row Q tile -- for B=64 the block plus 64 rows computed and
// discarded -- and the selected key blocks of its selection row). The CTA runs TWO
// independent item streams (rounds s, s + 2, ... of its snake order, s = 0, 1), so each SM
// sub-partition holds two softmax warps and the tensor core works on one stream while the
// other one's softmax runs (the single-stream kernel was paced by its one softmax warp per
// sub-partition: 1.229 vs 1.162 ms on C2). Per stream s:
//   producer warp (2s)      TMA of Q (per item) and K_j, V_j of every selected block (each a
//                           contiguous B x D slab: plain tensor-map boxes, no gather).
//   issuer warp (2s + 1)    single-thread UMMA: S = Q K_j^T (SS, M=128 N=B K=D) into S_s,
//                           then O_s += P_j V_j (TS, A = P_j from TMEM over S_s, B = V_j
//                           MN-major), in the order QK_j, PV_j, QK_{j+1}.
//   softmax warpgroup 1+s   one TMEM lane (= query row) per thread; online softmax in the
//                           log2 domain with lazy O rescaling (only when the row max grows by
//                           > 8); 3/8 of the exponentials on the FMA pipe (fastmath.cuh); P
//                           written back over S as packed bf16; epilogue O / l -> bf16 through
//                           a TMA store and LSE.
// TMEM: S0 | S1 | O0 | O1. Masking (keys past the sequence end, causal upper triangle of the
// diagonal block) patches S in TMEM (mask_diag_tmem), so all blocks run one softmax path.
#include "common.cuh"
#include "fastmath.cuh"
#include "sb_kernels.h"
#include "sched.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

namespace sbk {
namespace {

using namespace sm100;

constexpr int kM = 128;                 // UMMA M / Q tile rows
constexpr float kRescaleThresh = 8.0f;  // log2 units: lazily rescale O only on a 256x max jump

struct Item {
  int h, i, seq0, seq_len, n, first;
  const int32_t* list;
};

// Item of a prefetched schedule record (sched::q_records_kernel): register arithmetic only.
__device__ __forceinline__ Item from_rec(const sched::ItemRec& r, int nbt, const int32_t* idx, int k_max) {
  Item w;
  w.h = r.it / nbt;
  w.i = r.loc;
  w.seq0 = r.seq0;
  w.seq_len = r.seq_len;
  w.n = r.n;
  w.first = r.first;
  w.list = idx + static_cast<size_t>(r.base) * k_max;
  return w;
}

// Diagonal block (causal + sequence end: columns >= lim masked): the masked columns of S are
// overwritten with -inf in TMEM, 32 columns at a time from the warp's first partial chunk, so
// every block then runs the one unmasked softmax below. This path runs once per item and its
// code is cold in the instruction cache; an unrolled masked softmax variant (~1100
// instructions) cost ~3000 cycles per item in instruction fetch alone, this loop is ~60.
// P of a masked column is 0 from the SFU lanes and <= 2^-126 from the FMA-pipe exp2 lanes
// (fastmath.cuh clamps at -126): below any bf16 / fp32 tolerance.
template <int B>
__device__ __forceinline__ void mask_diag_tmem(uint32_t t_s, int lim) {
  const int first = __reduce_min_sync(0xffffffffu, lim) >> 5;  // first chunk with a masked column
  for (int ch = first; ch < B / 32; ++ch) {
    uint32_t v[32];
    tmem_ld32(t_s + ch * 32, v);
    tmem_wait_ld();
#pragma unroll
    for (int e = 0; e < 32; ++e) v[e] = ch * 32 + e < lim ? v[e] : 0xff800000u;
    tmem_st32(t_s + ch * 32, v);
  }
  tmem_wait_st();
}

// One key block of one query row (this thread's TMEM lane): row max (FMNMX3), lazy rescale
// decision, P = 2^(S*scale_log2 - m) with packed FFMA2 / FADD2 and the SFU/FMA exp2 split,
// packed bf16 P written back over the first B/2 columns of S.
template <int B>
__device__ __forceinline__ void softmax_block(const uint32_t (&sv)[B / 32][32], float scale_log2, float m_run,
                                              uint32_t t_s, float& m_use, float& alpha, float& sum, bool& rescale,
                                              unsigned long long* dbg) {
  float xs[B];
#pragma unroll
  for (int c = 0; c < B; ++c) xs[c] = __uint_as_float(sv[c / 32][c % 32]);
  float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
#pragma unroll
  for (int c = 0; c < B; c += 8) {
    m0 = fmax3(m0, xs[c], xs[c + 1]);
    m1 = fmax3(m1, xs[c + 2], xs[c + 3]);
    m2 = fmax3(m2, xs[c + 4], xs[c + 5]);
    m3 = fmax3(m3, xs[c + 6], xs[c + 7]);
  }
  const float m_new = fmaxf(m_run, fmax3(m0, m1, fmaxf(m2, m3)) * scale_log2);
  if (dbg) dbg[1] = clock64();
  rescale = m_new > m_run + kRescaleThresh;
  m_use = rescale ? m_new : m_run;
  alpha = rescale ? ex2_sfu(m_run - m_use) : 1.0f;
  const f2 sc = mk2(scale_log2, scale_log2), nm = mk2(-m_use, -m_use);
  f2 acc[4] = {mk2(0.f, 0.f), mk2(0.f, 0.f), mk2(0.f, 0.f), mk2(0.f, 0.f)};
#pragma unroll
  for (int c2 = 0; c2 < B / 64; ++c2) {
    uint32_t pw[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      const int pe = c2 * 32 + e;  // column pair (2pe, 2pe+1)
      const f2 p = ex2_pair(ffma2(mk2(xs[2 * pe], xs[2 * pe + 1]), sc, nm), pe);
      acc[e & 3] = fadd2(acc[e & 3], p);
      pw[e] = pack_bf16x2(p.x, p.y);
    }
    tmem_st32(t_s + c2 * 32, pw);  // P (packed bf16) over the first B/2 columns of S
    if (dbg && c2 < 2) dbg[2 + c2] = clock64();
  }
  const f2 a01 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
  sum = a01.x + a01.y;
}

// ------------------------------------------------------------------ two-stream kernel
// Warps 0..3 (WG0): producer / issuer of stream 0, producer / issuer of stream 1 (their
// waits spin: a sleeping try_wait added 300-700 cycles to each PV / QK issue); warps 4..7
// and 8..11: softmax of stream 0 / 1. Per stream, s_full(j) implies PV_{j-1} completed (same
// issuer, in order), so a lazy O rescale needs no wait. setmaxnreg: WG0 56, softmax 224.
constexpr int kThreads2 = 384;

template <int D, int B>
struct Fwd2Cfg {
  static constexpr int kChunks = D / 64;
  static constexpr int kQBytes = kChunks * kM * 128;
  static constexpr int kKVBytes = kChunks * B * 128;
  static constexpr int kStageBytes = B * 128;  // one 64-column chunk of a stream's O tile (TMA store)
  static constexpr int kSmemTiles = 2 * kQBytes + 4 * kKVBytes + 2 * kStageBytes;  // per stream: Q, K, V, stage
  static constexpr int kTmemO = 2 * B;                          // S_s at s * B, O_s at 2B + s * D
  static constexpr uint32_t kTmemCols = (2 * B + 2 * D) <= 256 ? 256 : 512;
  static constexpr int kSmemBytes = kSmemTiles + 1024 + 1024;  // + alignment slack + Fwd2Bars
};

// Items are claimed dynamically, per stream: stream s of CTA c starts at its snake slot of round
// s (c, or 2G - 1 - c), and every later item comes from a global cursor (reset by
// q_records_kernel) in the head-major, longest-first order. The stream's producer claims one item
// ahead and publishes the 32-byte record in a shared-memory ring that the stream's issuer and
// softmax warps read in order. The static snake left C2's per-CTA busy spans 1.08x apart.
constexpr int kFwdRing = 8;
constexpr int kFwdRingReaders = 5;  // the stream's issuer warp and its 4 softmax warps

struct Fwd2Bars {
  uint64_t q_full[2], q_empty[2], k_full[2], k_empty[2], v_full[2], v_empty[2];
  uint64_t s_full[2], p_full[2], o_done[2], o_free[2];
  uint64_t sched_full[2][kFwdRing], sched_empty[2][kFwdRing];
  int4 sched_rec[2][kFwdRing][2];  // sched::ItemRec of round k in slot k % kFwdRing
  uint32_t tmem_base;
};
static_assert(sizeof(Fwd2Bars) <= 1024, "Fwd2Bars fits the reserved tail of the forward's shared memory");

template <int D, int B>
__global__ void __launch_bounds__(kThreads2, 1) attn_fwd2_kernel(
    const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
    const __grid_constant__ CUtensorMap tm_ores, const int32_t* __restrict__ blk_off, int nseq, int total_tokens,
    int hq, int hkv, const int32_t* __restrict__ idx, int k_max, float scale_log2, uint16_t* __restrict__ out,
    uint16_t* __restrict__ ores, float* __restrict__ lse, const sched::ItemRec* __restrict__ recs, int n_items,
    unsigned long long* __restrict__ trace) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  using C = Fwd2Cfg<D, B>;
  if (trace != nullptr && threadIdx.x == 0) trace[8192 + 2 * blockIdx.x] = globaltimer_ns();  // per-CTA span
  // Debug timeline: CTA 0, per stream s and block g < 256: [s][g][slot] (slots: 0 QK issued,
  // 1 PV issued, 2 S seen by softmax warp 0, 3 P arrived, 4 epilogue start, 5 end, 6 k_full seen).
  // An L2 prefetch of block j+1's K / V one block early was measured 4% slower.
  auto tr2 = [&](int st, int g, int slot) {
    if (trace != nullptr && blockIdx.x == 0 && g < 256) trace[(st * 256 + g) * 8 + slot] = clock64();
  };
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* q_smem = smem;                         // [stream]
  uint8_t* k_smem = smem + 2 * C::kQBytes;        // [stream]
  uint8_t* v_smem = k_smem + 2 * C::kKVBytes;     // [stream]
  uint8_t* o_stage = v_smem + 2 * C::kKVBytes;    // [stream]: SW128 chunk of O for the TMA store
  Fwd2Bars* bars = reinterpret_cast<Fwd2Bars*>(smem + C::kSmemTiles);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nbt = blk_off[nseq];
  const int grid = gridDim.x, cta = blockIdx.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars->q_full[s], 1);
      mbar_init(&bars->q_empty[s], 1);
      mbar_init(&bars->k_full[s], 1);
      mbar_init(&bars->k_empty[s], 1);
      mbar_init(&bars->v_full[s], 1);
      mbar_init(&bars->v_empty[s], 1);
      mbar_init(&bars->s_full[s], 1);
      mbar_init(&bars->p_full[s], 128);
      mbar_init(&bars->o_done[s], 1);
      mbar_init(&bars->o_free[s], 128);
      for (int i = 0; i < kFwdRing; ++i) {
        mbar_init(&bars->sched_full[s][i], 1);
        mbar_init(&bars->sched_empty[s][i], kFwdRingReaders);
      }
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  int* cursor = const_cast<int*>(reinterpret_cast<const int*>(recs + n_items));  // sched::rec_workspace_bytes slack
  // Round k of stream s: claimed and published by the stream's producer (lane 0) ...
  auto claim = [&](int s, int k) {
    const int slot = k % kFwdRing;
    if (k >= kFwdRing) mbar_wait_spin(&bars->sched_empty[s][slot], ((k / kFwdRing) & 1) ^ 1);
    const int pos = k == 0 ? (s == 0 ? cta : 2 * grid - 1 - cta) : 2 * grid + atomicAdd(cursor, 1);
    int4 a = make_int4(-1, 0, 0, 0), b = make_int4(0, 0, 0, 0);
    if (pos < n_items) {
      a = __ldg(reinterpret_cast<const int4*>(recs + pos));
      b = __ldg(reinterpret_cast<const int4*>(recs + pos) + 1);
    }
    bars->sched_rec[s][slot][0] = a;
    bars->sched_rec[s][slot][1] = b;
    mbar_arrive(&bars->sched_full[s][slot]);  // release: the record is visible to the waiters
    return sched::ItemRec{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  };
  // ... and read, in round order, by each of its issuer and softmax warps (whole warp).
  auto take = [&](int s, int k) {
    const int slot = k % kFwdRing;
    mbar_wait_spin(&bars->sched_full[s][slot], (k / kFwdRing) & 1);
    const int4 a = bars->sched_rec[s][slot][0], b = bars->sched_rec[s][slot][1];
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars->sched_empty[s][slot]);
    return sched::ItemRec{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  };

  if (warp < 4) {
    setmaxnreg_dec<56>();
    const int s = warp >> 1;  // warps 0, 1: stream 0; warps 2, 3: stream 1
    if ((warp & 1) == 0) {
      // -------------------------------------------------------- TMA producer of stream s
      if (lane == 0) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        uint8_t* qs = q_smem + s * C::kQBytes;
        uint8_t* ks = k_smem + s * C::kKVBytes;
        uint8_t* vs = v_smem + s * C::kKVBytes;
        int g = 0, q = 0;
        sched::ItemRec nr = claim(s, 0);
        for (int k = 0;; ++k) {
          const sched::ItemRec rec = nr;
          if (rec.it < 0) break;
          nr = claim(s, k + 1);
          const Item w = from_rec(rec, nbt, idx, k_max);
          if (w.n <= 0) continue;
          const int hk = w.h / (hq / hkv);
          if (nr.it >= 0 && nr.n > 0) {
            // L2 prefetch of this stream's next item's Q tile: its load waits for this item's last
            // QK, so with few blocks per item a DRAM round trip would sit on the stream's chain
            for (int c = 0; c < C::kChunks; ++c)
              tma_prefetch_l2_3d(&tm_q, c * 64, nr.it / nbt, nr.seq0 + nr.loc * B);
          }
          mbar_wait_spin(&bars->q_empty[s], (q & 1) ^ 1);
          mbar_expect_tx(&bars->q_full[s], C::kQBytes);
          for (int c = 0; c < C::kChunks; ++c)
            tma_load_3d(qs + c * kM * 128, &tm_q, &bars->q_full[s], c * 64, w.h, w.seq0 + w.i * B);
          for (int j = 0; j < w.n; ++j, ++g) {
            const int kv_row = w.seq0 + __ldg(w.list + j) * B;
            mbar_wait_spin(&bars->k_empty[s], (g & 1) ^ 1);
            mbar_expect_tx(&bars->k_full[s], C::kKVBytes);
            for (int c = 0; c < C::kChunks; ++c)
              tma_load_3d(ks + c * B * 128, &tm_k, &bars->k_full[s], c * 64, hk, kv_row);
            mbar_wait_spin(&bars->v_empty[s], (g & 1) ^ 1);
            mbar_expect_tx(&bars->v_full[s], C::kKVBytes);
            for (int c = 0; c < C::kChunks; ++c)
              tma_load_3d(vs + c * B * 128, &tm_v, &bars->v_full[s], c * 64, hk, kv_row);
          }
          ++q;
        }
      }
    } else {
      // -------------------------------------------------------- UMMA issuer of stream s
      const uint32_t leader = elect_one();
      constexpr uint32_t idesc_qk = idesc_bf16_f32(kM, B, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(kM, D, false, true);
      const uint32_t q_addr = smem_u32(q_smem + s * C::kQBytes);
      const uint32_t k_addr = smem_u32(k_smem + s * C::kKVBytes), v_addr = smem_u32(v_smem + s * C::kKVBytes);
      const uint32_t d_s = tmem + s * B, d_o = tmem + C::kTmemO + s * D;
      int g = 0, q = 0;
      for (int k = 0;; ++k) {
        const sched::ItemRec rec = take(s, k);
        if (rec.it < 0) break;
        const int n = rec.n;
        if (n <= 0) continue;
        mbar_wait_spin(&bars->q_full[s], q & 1);
        for (int j = 0; j < n; ++j, ++g) {
          mbar_wait_spin(&bars->k_full[s], g & 1);
          if (lane == 0) tr2(s, g, 6);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t koff = (kk & 3) * 32;
            const uint64_t a = desc_sw128(q_addr + (kk >> 2) * (kM * 128) + koff, 16, 1024);
            const uint64_t b = desc_sw128(k_addr + (kk >> 2) * (B * 128) + koff, 16, 1024);
            mma_ss(d_s, a, b, idesc_qk, kk > 0 ? 1u : 0u, leader);
          }
          tc_commit(&bars->s_full[s], leader);
          tc_commit(&bars->k_empty[s], leader);
          if (lane == 0) tr2(s, g, 0);
          if (j == n - 1) tc_commit(&bars->q_empty[s], leader);
          mbar_wait_spin(&bars->v_full[s], g & 1);
          mbar_wait_spin(&bars->p_full[s], g & 1);
          if (j == 0) mbar_wait_spin(&bars->o_free[s], (q & 1) ^ 1);  // epilogue of the stream's previous item
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < B / 16; ++kk) {
            const uint64_t b = desc_sw128(v_addr + kk * 2048, B * 128, 1024);
            mma_ts(d_o, d_s + kk * 8, b, idesc_pv, (j > 0 || kk > 0) ? 1u : 0u, leader);
          }
          tc_commit(&bars->v_empty[s], leader);
          if (lane == 0) tr2(s, g, 1);
          if (j == n - 1) tc_commit(&bars->o_done[s], leader);
        }
        ++q;
      }
    }
  } else {
    setmaxnreg_inc<224>();
    // ---------------------------------------------------------- softmax / epilogue of stream s
    const int s = (warp >> 2) - 1;
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t lane_field = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t t_s = tmem + lane_field + s * B, t_o = tmem + lane_field + C::kTmemO + s * D;
    int g = 0, q = 0;
    for (int k = 0;; ++k) {
      const sched::ItemRec rec = take(s, k);
      if (rec.it < 0) break;
      const Item w = from_rec(rec, nbt, idx, k_max);
      const int row0 = w.seq0 + w.i * B;
      const int nrows = min(B, w.seq_len - w.i * B);
      const bool store = r < nrows;
      if (w.n <= 0) {  // nothing selected: zero output, LSE = -inf
        if (store) {
          uint4* dst = reinterpret_cast<uint4*>(out + (static_cast<size_t>(row0 + r) * hq + w.h) * D);
          for (int e = 0; e < D / 8; ++e) dst[e] = make_uint4(0, 0, 0, 0);
          if (ores != nullptr) {
            uint4* dr = reinterpret_cast<uint4*>(ores + (static_cast<size_t>(row0 + r) * hq + w.h) * D);
            for (int e = 0; e < D / 8; ++e) dr[e] = make_uint4(0, 0, 0, 0);
          }
          lse[static_cast<size_t>(w.h) * total_tokens + row0 + r] = -INFINITY;
        }
        continue;
      }
      float m_run = -INFINITY, l_run = 0.f;
      int jb_next = w.first;
      for (int j = 0; j < w.n; ++j, ++g) {
        const int jb = jb_next;
        if (j + 1 < w.n) jb_next = __ldg(w.list + j + 1);
        mbar_wait_spin(&bars->s_full[s], g & 1);
        if (r == 0) tr2(s, g, 2);
        tc_fence_after();
        if (jb == w.i) mask_diag_tmem<B>(t_s, min(min(B, w.seq_len - jb * B), r + 1));
        uint32_t sv[B / 32][32];
#pragma unroll
        for (int c = 0; c < B / 32; ++c) tmem_ld32(t_s + c * 32, sv[c]);
        tmem_wait_ld();
        float m_use, alpha, sum;
        bool rescale;
        softmax_block<B>(sv, scale_log2, m_run, t_s, m_use, alpha, sum, rescale, nullptr);
        l_run = l_run * alpha + sum;
        tmem_wait_st();
        // PV_{j-1} completed before S_j was committed (same issuer, in order): O is final.
        if (j > 0 && __any_sync(0xffffffffu, rescale)) {
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t v[32];
            tmem_ld32(t_o + c * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(__uint_as_float(v[e]) * alpha);
            tmem_st32(t_o + c * 32, v);
          }
          tmem_wait_st();
        }
        m_run = m_use;
        tc_fence_before();
        if (r == 0) tr2(s, g, 3);
        mbar_arrive(&bars->p_full[s]);
      }
      // Epilogue: the item's last PV, O / l -> bf16 rows; LSE (natural log).
      if (r == 0) tr2(s, g - 1, 4);
      mbar_wait(&bars->o_done[s], q & 1);
      tc_fence_after();
      const float inv_l = l_run > 0.f ? 1.0f / l_run : 0.f;
      uint32_t v[D / 32][32];
#pragma unroll
      for (int c = 0; c < D / 32; ++c) tmem_ld32(t_o + c * 32, v[c]);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&bars->o_free[s]);  // O may be overwritten by the stream's next item
      // O (and, when ores != nullptr, its bf16 rounding residual bf16(O - bf16(O)), from which the
      // backward forms D = rowsum(dO * O) to ~2^-16 instead of bf16 precision).
      const int parts = ores != nullptr ? 2 : 1;
      if (nrows == B) {
        // Full tile: 32-column boxes (64-byte rows, 64B swizzle) through two halves of the
        // stream's staging slot, double-buffered: round n writes half n & 1 once the store of
        // round n - 2 has read it (wait_group.read 1), so the O / O-residual stores pipeline
        // instead of waiting out each store's shared-memory read (6000 -> ~2000 cycles per
        // item with the residual). Thread r == 0 issues; named barrier 1 + s syncs the stream.
        uint8_t* stg = o_stage + s * C::kStageBytes;
        int n = 0;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          for (int part = 0; part < parts; ++part, ++n) {
            uint8_t* buf = stg + (n & 1) * (B * 64);
            if (r == 0) bulk_wait_read<1>();
            named_bar_sync(1 + s, 128);
            if (r < B) {
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int d0 = c * 32 + u * 8;
                float x[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                  x[e] = __uint_as_float(v[(d0 + e) / 32][(d0 + e) % 32]) * inv_l;
                  if (part) x[e] -= __bfloat162float(__float2bfloat16_rn(x[e]));
                }
                *reinterpret_cast<uint4*>(buf + r * 64 + ((u ^ ((r >> 1) & 3)) << 4)) =
                    make_uint4(pack_bf16x2(x[0], x[1]), pack_bf16x2(x[2], x[3]), pack_bf16x2(x[4], x[5]),
                               pack_bf16x2(x[6], x[7]));
              }
            }
            fence_proxy_async_smem();
            named_bar_sync(1 + s, 128);
            if (r == 0) {
              tma_store_3d(part ? &tm_ores : &tm_o, buf, c * 32, w.h, row0);
              bulk_commit();
            }
          }
        }
        if (store) lse[static_cast<size_t>(w.h) * total_tokens + row0 + r] = (m_run + log2f(l_run)) * 0.69314718055994531f;
      } else if (store) {  // the last (partial) tile of a sequence: a box would cross into the next
        SB_DCHECK(row0 + r < total_tokens);
        for (int part = 0; part < parts; ++part) {
          uint16_t* orow = (part ? ores : out) + (static_cast<size_t>(row0 + r) * hq + w.h) * D;
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t w16[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              float a = __uint_as_float(v[c][2 * e]) * inv_l, b = __uint_as_float(v[c][2 * e + 1]) * inv_l;
              if (part) {
                a -= __bfloat162float(__float2bfloat16_rn(a));
                b -= __bfloat162float(__float2bfloat16_rn(b));
              }
              w16[e] = pack_bf16x2(a, b);
            }
            store_64B(orow + c * 32, w16);
          }
        }
        lse[static_cast<size_t>(w.h) * total_tokens + row0 + r] = (m_run + log2f(l_run)) * 0.69314718055994531f;
      }
      if (r == 0) tr2(s, g - 1, 5);
      ++q;
    }
    if (r == 0) bulk_wait_all();  // the stream's outstanding O stores read smem and reach global
  }
  tc_fence_before();
  __syncthreads();
  if (trace != nullptr && threadIdx.x == 0) trace[8192 + 2 * blockIdx.x + 1] = globaltimer_ns();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem);
  }
}

unsigned long long* g_trace = nullptr;  // debug timeline buffer (sb_debug_set_trace)

template <int D, int B>
void launch_fwd(const uint16_t* q, const uint16_t* k, const uint16_t* v, const int32_t* cu, const int32_t* blk_off,
                int nseq, int total, int nb_total, int hq, int hkv, const int32_t* idx, const int32_t* cnt, int hsel,
                int k_max, float scale, uint16_t* o, uint16_t* ores, float* lse, void* ws, cudaStream_t st) {
  const int n_items = hq * nb_total;
  auto* recs = reinterpret_cast<sched::ItemRec*>(
      (reinterpret_cast<uintptr_t>(ws) + sched::order_workspace_bytes(n_items, hq * (k_max + 1)) + 255) & ~uintptr_t(255));
  sched::build_q_schedule(sched::CostFromCnt{cnt, k_max, hq, hsel, nb_total}, n_items, ws, recs, cu, blk_off, nseq,
                          idx, k_max, st, "sb_sparse_attn_fwd/order");
  const CUtensorMap tq = make_thd_map(q, total, hq, D, kM);
  const CUtensorMap tk = make_thd_map(k, total, hkv, D, B);
  const CUtensorMap tv = make_thd_map(v, total, hkv, D, B);
  const CUtensorMap to = make_thd_map(o, total, hq, D, B, 32);
  const CUtensorMap tores = make_thd_map(ores != nullptr ? ores : o, total, hq, D, B, 32);
  const int grid = std::min(n_items, sched::num_sms());
  using C2 = Fwd2Cfg<D, B>;
  auto k2 = attn_fwd2_kernel<D, B>;
  set_smem_once(k2, C2::kSmemBytes, "sb_sparse_attn_fwd: smem attribute");
  launch(k2, grid, kThreads2, C2::kSmemBytes, st, tq, tk, tv, to, tores, blk_off, nseq, total, hq, hkv, idx, k_max,
                                              scale * 1.4426950408889634f, o, ores, lse, recs, n_items, g_trace);
  launched("sb_sparse_attn_fwd");
}

}  // namespace
}  // namespace sbk

// Debug only: device buffer of 2 x 256 x 8 uint64 for CTA 0's per-stream timeline (NULL disables).
SB_API void sb_debug_set_trace(unsigned long long* buf) { sbk::g_trace = buf; }

SB_API size_t sb_sparse_attn_fwd_workspace_size(int nb_total, int hq, int k_max) {
  return sbk::sched::order_workspace_bytes(nb_total * hq, hq * (k_max + 1)) + 256 +
         sbk::sched::rec_workspace_bytes(nb_total * hq);
}

SB_API size_t sb_sparse_attn_fwd_workspace_size_ex(int nseq, int nb_total, int hq, int hsel, int k_max, int block_size) {
  if (block_size != 256) return sb_sparse_attn_fwd_workspace_size(nb_total, hq, k_max);
  return sbk::expand256_workspace_bytes(nseq, nb_total, hsel, k_max) +
         sb_sparse_attn_fwd_workspace_size(2 * nb_total, hq, 2 * k_max);
}

SB_API int sb_sparse_attn_fwd_ex(const uint16_t* q, const uint16_t* k, const uint16_t* v, const int32_t* cu_seqlens,
                                 const int32_t* blk_off, int nseq, int total_tokens, int nb_total, int hq, int hkv,
                                 int head_dim, int block_size, const int32_t* idx, const int32_t* cnt, int hsel,
                                 int k_max, float scale, uint16_t* o, uint16_t* o_res, float* lse, void* workspace,
                                 void* stream) {
  return sbk::abi_call([&] {
    sbk::require(head_dim == 64 || head_dim == 128, "head_dim must be 64 or 128");
    sbk::require(block_size == 64 || block_size == 128 || block_size == 256, "block_size must be 64, 128 or 256");
    sbk::require(hq >= 1 && hkv >= 1 && hq % hkv == 0, "hq must be a positive multiple of hkv");
    sbk::require(hsel >= hkv && hq % hsel == 0 && hsel % hkv == 0,
                 "hsel must divide hq and be a multiple of hkv (each selection row maps to one kv head)");
    sbk::require(k_max >= 1, "k_max must be >= 1");
    if (nseq == 0 || nb_total == 0 || total_tokens == 0) return;
    sbk::require(q && k && v && cu_seqlens && blk_off && idx && cnt && o && lse && workspace, "null pointer");
    if (block_size == 256) {  // workspace: sb_sparse_attn_fwd_workspace_size_ex
      const cudaStream_t st256 = static_cast<cudaStream_t>(stream);
      const sbk::Expanded256 e = sbk::expand_selection_256(cu_seqlens, blk_off, nseq, nb_total, hsel, idx, cnt, k_max,
                                                           static_cast<uint8_t*>(workspace), st256);
      void* ws128 = static_cast<uint8_t*>(workspace) + e.used;
      if (head_dim == 128)
        return sbk::launch_fwd<128, 128>(q, k, v, cu_seqlens, e.blk_off, nseq, total_tokens, e.nb_total, hq, hkv,
                                         e.idx, e.cnt, hsel, e.k_max, scale, o, o_res, lse, ws128, st256);
      return sbk::launch_fwd<64, 128>(q, k, v, cu_seqlens, e.blk_off, nseq, total_tokens, e.nb_total, hq, hkv, e.idx,
                                      e.cnt, hsel, e.k_max, scale, o, o_res, lse, ws128, st256);
    }
    sbk::require((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v) |
                  reinterpret_cast<uintptr_t>(o) | reinterpret_cast<uintptr_t>(o_res)) % 16 == 0,
                 "q/k/v/o/o_res must be 16-byte aligned");
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
#define SB_FWD_CASE(DD, BB)                                                                                      \
  if (head_dim == DD && block_size == BB)                                                                        \
    return sbk::launch_fwd<DD, BB>(q, k, v, cu_seqlens, blk_off, nseq, total_tokens, nb_total, hq, hkv, idx, cnt, \
                                   hsel, k_max, scale, o, o_res, lse, workspace, st);
    SB_FWD_CASE(128, 128)
    SB_FWD_CASE(128, 64)
    SB_FWD_CASE(64, 128)
    SB_FWD_CASE(64, 64)
#undef SB_FWD_CASE
  });
}

SB_API int sb_sparse_attn_fwd(const uint16_t* q, const uint16_t* k, const uint16_t* v, const int32_t* cu_seqlens,
                              const int32_t* blk_off, int nseq, int total_tokens, int nb_total, int hq, int hkv,
                              int head_dim, int block_size, const int32_t* idx, const int32_t* cnt, int hsel,
                              int k_max, float scale, uint16_t* o, float* lse, void* workspace, void* stream) {
  return sb_sparse_attn_fwd_ex(q, k, v, cu_seqlens, blk_off, nseq, total_tokens, nb_total, hq, hkv, head_dim,
                               block_size, idx, cnt, hsel, k_max, scale, o, nullptr, lse, workspace, stream);
}
