// K5: varlen block-sparse attention forward on tcgen05 / TMEM (Eq. 2).
//
// Persistent kernel: one CTA per SM walks a longest-first list of work items (one item = one
// q block x q head: a 128-row Q tile -- for B=64 the block plus 64 rows computed and
// discarded -- and the selected key blocks of its selection row). Warp roles:
//   warp 0      TMA producer: Q of each item (2 buffers, so the next item's Q arrives while
//               the current one runs) and K_j / V_j of every selected block into a 2-stage
//               ring (each selected block is a contiguous B x D slab -> plain tensor-map
//               boxes, no element gather).
//   warp 1      TMEM allocator + single-thread UMMA issuer over the CTA's global block
//               stream g (all items back to back):
//                 S_g = Q K_g^T   (SS, M=128 N=B K=D)          -> TMEM S[g % 2]
//                 O  += P_g V_g   (TS, A = P_g from TMEM, B = V_g MN-major in smem)
//               issue order QK_0, QK_1, QK_2, PV_0, QK_3, PV_1, ... (QK_g before PV_{g-2})
//               across item boundaries. S is triple-buffered (TMEM: S0 | S1 | S2 | O): P_g
//               aliases S_g, so with two buffers QK_{g+1} had to wait for PV_{g-1} and the
//               chain P_{g-1} -> PV_{g-1} -> QK_{g+1} -> S_{g+1} (~1650 cycles) paced the
//               softmax; with three the softmax has two blocks of slack. O is single: the
//               same softmax warps run the epilogue before producing the next item's P_0, so
//               a second O buffer could never be used early.
//   warps 2..5  softmax: one TMEM lane (= query row) per thread; online softmax in the log2
//               domain with lazy O rescaling (only when the row max grows by > 8); 3/8 of the
//               exponentials on the FMA pipe (fastmath.cuh); P written back into TMEM as packed
//               bf16 over S; epilogue O / l -> bf16 rows and LSE.
// Masking: keys past the sequence end and the causal upper triangle of the diagonal block.
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
constexpr int kStages = 2;              // K ring depth
constexpr int kSBufs = 3;               // S / P buffers in TMEM
constexpr int kVStages = 2;             // V ring depth (3 measured no faster; the slot holds the O staging tile)
constexpr int kThreads = 224;           // 7 warps: Q/K producer, UMMA, 4 softmax, V producer
constexpr float kRescaleThresh = 8.0f;  // log2 units: lazily rescale O only on a 256x max jump

template <int D, int B>
struct FwdCfg {
  static constexpr int kChunks = D / 64;              // 128-byte swizzle atoms along D
  static constexpr int kQBytes = kChunks * kM * 128;  // one Q tile
  static constexpr int kKVBytes = kChunks * B * 128;  // one K or V block
  static constexpr int kStageBytes = kChunks * B * 128;  // bf16 O tile staged for the TMA store
  static constexpr int kSmemTiles = 2 * kQBytes + (kStages + kVStages) * kKVBytes + kStageBytes;
  static constexpr int kTmemO = kSBufs * B;  // S_b at column b * B
  static constexpr uint32_t kTmemCols = (kSBufs * B + D) <= 256 ? 256 : 512;
  static constexpr int kSmemBytes = kSmemTiles + 1024 /*align slack*/ + 256 /*barriers*/;
};

struct FwdBars {
  uint64_t q_full[2], q_empty[2];
  uint64_t k_full[kStages], k_empty[kStages];
  uint64_t v_full[kVStages], v_empty[kVStages];
  uint64_t s_full[kSBufs], p_full[kSBufs];
  uint64_t o_done[kSBufs], o_free;  // o_done[b]: PV of the blocks g with g % kSBufs == b
  uint32_t tmem_base;
};

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

template <int D, int B>
__global__ void __launch_bounds__(kThreads, 1) attn_fwd_kernel(
    const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o, const int32_t* __restrict__ cu, const int32_t* __restrict__ blk_off,
    int nseq, int total_tokens, int hq, int hkv, const int32_t* __restrict__ idx, const int32_t* __restrict__ cnt,
    int hsel, int k_max, float scale_log2, uint16_t* __restrict__ out, float* __restrict__ lse,
    const sched::ItemRec* __restrict__ recs, int n_items, unsigned long long* __restrict__ trace) {
  using C = FwdCfg<D, B>;
  // Debug timeline (sb_debug_set_trace): CTA 0 records clock64 at phase boundaries.
  auto tr = [&](int slot, int g) {
    if (trace != nullptr && blockIdx.x == 0 && g < 256 && (threadIdx.x & 31) == 0) trace[g * 8 + slot] = clock64();
  };
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* q_smem = smem;                                // [2]
  uint8_t* k_smem = smem + 2 * C::kQBytes;               // [kStages]
  uint8_t* v_smem = k_smem + kStages * C::kKVBytes;      // [kVStages]
  uint8_t* o_stage = v_smem + kVStages * C::kKVBytes;    // O tile for the TMA store (SW128, [chunk][row])
  FwdBars* bars = reinterpret_cast<FwdBars*>(smem + C::kSmemTiles);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nbt = blk_off[nseq];
  const int grid = gridDim.x, cta = blockIdx.x;

  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars->q_full[b], 1);
      mbar_init(&bars->q_empty[b], 1);
    }
    for (int b = 0; b < kSBufs; ++b) {
      mbar_init(&bars->s_full[b], 1);
      mbar_init(&bars->p_full[b], 128);
      mbar_init(&bars->o_done[b], 1);
    }
    mbar_init(&bars->o_free, 128);
    for (int st = 0; st < kStages; ++st) {
      mbar_init(&bars->k_full[st], 1);
      mbar_init(&bars->k_empty[st], 1);
    }
    for (int st = 0; st < kVStages; ++st) {
      mbar_init(&bars->v_full[st], 1);
      mbar_init(&bars->v_empty[st], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  // TMA producer over the CTA's item stream: Q + K (v_stream = false) or V (v_stream = true).
  auto produce = [&](bool v_stream) {
    if (lane != 0) return;
    if (v_stream) {
      tma_prefetch(&tm_v);
    } else {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
    }
    int g = 0, q = 0;
    for (sched::RecCursor cur(recs, n_items, grid, cta);;) {
      const sched::ItemRec rec = cur.next();
      if (rec.it < 0) break;
      const Item w = from_rec(rec, nbt, idx, k_max);
      if (w.n <= 0) continue;
      const int hk = w.h / (hq / hkv);
      if (!v_stream) {
        const int qb = q & 1;
        mbar_wait(&bars->q_empty[qb], ((q >> 1) & 1) ^ 1);
        mbar_expect_tx(&bars->q_full[qb], C::kQBytes);
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d(q_smem + qb * C::kQBytes + c * kM * 128, &tm_q, &bars->q_full[qb], c * 64, w.h,
                      w.seq0 + w.i * B);
      }
      for (int j = 0; j < w.n; ++j, ++g) {
        const int kv_row = w.seq0 + __ldg(w.list + j) * B;
        if (!v_stream) {
          const int st = g % kStages;
          mbar_wait(&bars->k_empty[st], ((g / kStages) & 1) ^ 1);
          mbar_expect_tx(&bars->k_full[st], C::kKVBytes);
          for (int c = 0; c < C::kChunks; ++c)
            tma_load_3d(k_smem + st * C::kKVBytes + c * B * 128, &tm_k, &bars->k_full[st], c * 64, hk, kv_row);
        } else {
          const int vs = g % kVStages;
          mbar_wait(&bars->v_empty[vs], ((g / kVStages) & 1) ^ 1);
          mbar_expect_tx(&bars->v_full[vs], C::kKVBytes);
          for (int c = 0; c < C::kChunks; ++c)
            tma_load_3d(v_smem + vs * C::kKVBytes + c * B * 128, &tm_v, &bars->v_full[vs], c * 64, hk, kv_row);
        }
      }
      ++q;
    }
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producers
    // Warp 0 streams Q + K, warp 6 streams V: separate warps, so neither ring's wait blocks
    // the other (divergent lanes of one warp would serialise on each other's sleeps).
    produce(false);
  } else if (warp == 1) {
    // ------------------------------------------------------------ UMMA issuer
    {  // whole warp, converged; `leader` issues
      const uint32_t leader = elect_one();
      constexpr uint32_t idesc_qk = idesc_bf16_f32(kM, B, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(kM, D, false, true);
      const uint32_t k_addr = smem_u32(k_smem), v_addr = smem_u32(v_smem);
      // Pending PVs (the two previous global blocks), issued two QKs late: a ring of 2.
      int pv_g[2] = {-1, -1}, pv_j[2] = {0, 0}, pv_q[2] = {0, 0}, pv_n = 0, pv_h = 0;
      auto issue_pv = [&]() {
        const int g = pv_g[pv_h], j = pv_j[pv_h], q = pv_q[pv_h];
        pv_h ^= 1;
        --pv_n;
        const int st = g % kVStages;
        mbar_wait(&bars->v_full[st], (g / kVStages) & 1);
        tr(2, g);
        mbar_wait(&bars->p_full[g % kSBufs], (g / kSBufs) & 1);
        tr(3, g);
        if (j == 0) mbar_wait(&bars->o_free, (q & 1) ^ 1);  // epilogue of item q-1 read O
        tc_fence_after();
        const uint32_t p_tmem = tmem + (g % kSBufs) * B;
        const uint32_t o_tmem = tmem + C::kTmemO;
#pragma unroll
        for (int kk = 0; kk < B / 16; ++kk) {
          const uint64_t b = desc_sw128(v_addr + st * C::kKVBytes + kk * 2048, B * 128, 1024);
          mma_ts(o_tmem, p_tmem + kk * 8, b, idesc_pv, (j > 0 || kk > 0) ? 1u : 0u, leader);
        }
        tc_commit(&bars->v_empty[st], leader);
        tc_commit(&bars->o_done[g % kSBufs], leader);
      };
      int g = 0, q = 0;
      for (sched::RecCursor cur(recs, n_items, grid, cta);;) {
        const sched::ItemRec rec = cur.next();
        if (rec.it < 0) break;
        const Item w = from_rec(rec, nbt, idx, k_max);
        if (w.n <= 0) continue;
        const int qb = q & 1;
        const uint32_t q_addr = smem_u32(q_smem + qb * C::kQBytes);
        mbar_wait(&bars->q_full[qb], (q >> 1) & 1);
        for (int j = 0; j < w.n; ++j, ++g) {
          const int st = g % kStages;
          tr(0, g);
          mbar_wait(&bars->k_full[st], (g / kStages) & 1);
          tr(1, g);
          tc_fence_after();
          const uint32_t d_s = tmem + (g % kSBufs) * B;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t koff = (kk & 3) * 32;  // 16 bf16 = 32 B inside the swizzle atom
            const uint64_t a = desc_sw128(q_addr + (kk >> 2) * (kM * 128) + koff, 16, 1024);
            const uint64_t b = desc_sw128(k_addr + st * C::kKVBytes + (kk >> 2) * (B * 128) + koff, 16, 1024);
            mma_ss(d_s, a, b, idesc_qk, kk > 0 ? 1u : 0u, leader);
          }
          tc_commit(&bars->s_full[g % kSBufs], leader);
          tc_commit(&bars->k_empty[st], leader);
          if (j == w.n - 1) tc_commit(&bars->q_empty[qb], leader);
          if (pv_n == 2) issue_pv();
          const int t = (pv_h + pv_n) & 1;
          pv_g[t] = g;
          pv_j[t] = j;
          pv_q[t] = q;
          ++pv_n;
        }
        ++q;
      }
      while (pv_n > 0) issue_pv();
    }
  } else if (warp == 6) {
    produce(true);
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int r = quarter * 32 + lane;
    const uint32_t lane_field = static_cast<uint32_t>(quarter * 32) << 16;
    int g = 0, q = 0;
    for (sched::RecCursor cur(recs, n_items, grid, cta);;) {
      const sched::ItemRec rec = cur.next();
      if (rec.it < 0) break;
      const Item w = from_rec(rec, nbt, idx, k_max);
      const int row0 = w.seq0 + w.i * B;
      const int nrows = min(B, w.seq_len - w.i * B);
      const bool store = r < nrows;
      if (w.n <= 0) {  // nothing selected: zero output, LSE = -inf
        if (store) {
          uint4* dst = reinterpret_cast<uint4*>(out + (static_cast<size_t>(row0 + r) * hq + w.h) * D);
          for (int e = 0; e < D / 8; ++e) dst[e] = make_uint4(0, 0, 0, 0);
          lse[static_cast<size_t>(w.h) * total_tokens + row0 + r] = -INFINITY;
        }
        continue;
      }
      const uint32_t t_o = tmem + lane_field + C::kTmemO;
      float m_run = -INFINITY, l_run = 0.f;
      // Key block ids are loaded one block ahead: a global load consumed right after the
      // s_full wait put its L2 latency (~300 cycles) on every block when S was already ready.
      int jb_next = w.first;
      for (int j = 0; j < w.n; ++j, ++g) {
        const int b = g % kSBufs;
        const uint32_t t_s = tmem + lane_field + b * B;
        const int jb = jb_next;
        if (j + 1 < w.n) jb_next = __ldg(w.list + j + 1);
        mbar_wait_spin(&bars->s_full[b], (g / kSBufs) & 1);
        if (threadIdx.x == 64) tr(4, g);
        if (trace != nullptr && blockIdx.x == 0 && g < 256 && lane == 0)  // per-warp S seen (debug)
          trace[3072 + g * 4 + (warp - 2)] = clock64();
        tc_fence_after();
        // Keys of off-diagonal blocks are all valid (earlier blocks of a sequence are full);
        // the diagonal block masks the causal upper triangle and keys past the sequence end.
        if (jb == w.i) mask_diag_tmem<B>(t_s, min(min(B, w.seq_len - jb * B), r + 1));
        uint32_t sv[B / 32][32];
#pragma unroll
        for (int c = 0; c < B / 32; ++c) tmem_ld32(t_s + c * 32, sv[c]);
        tmem_wait_ld();
        unsigned long long* dbg =
            (trace != nullptr && blockIdx.x == 0 && g < 256 && threadIdx.x == 64) ? trace + 5120 + g * 4 : nullptr;
        if (dbg) dbg[0] = clock64();
        float m_use, alpha, sum;
        bool rescale;
        softmax_block<B>(sv, scale_log2, m_run, t_s, m_use, alpha, sum, rescale, dbg);
        if (threadIdx.x == 64) tr(7, g);
        const float sum0 = sum, sum1 = 0.f;
        l_run = l_run * alpha + (sum0 + sum1);
        tmem_wait_st();
        if (threadIdx.x == 64) tr(5, g);
        // Rescale O only when a lane's max jumped; only then wait for PV_{g-1} (same item) to
        // finish writing O. Skipping the wait is safe with per-slot barriers: s_full(g) implies
        // PV_{g-2} completed (in-order pipe, QK_g issued after PV_{g-2}), so o_done[(g-1) % 3]
        // has completed either PV_{g-4} or PV_{g-1} and the parity test is unambiguous.
        if (j > 0 && __any_sync(0xffffffffu, rescale)) {
          mbar_wait(&bars->o_done[(g - 1) % kSBufs], ((g - 1) / kSBufs) & 1);
          if (threadIdx.x == 64) tr(6, g);
          tc_fence_after();
          {
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
        }
        m_run = m_use;
        tc_fence_before();
        if (trace != nullptr && blockIdx.x == 0 && g < 256 && lane == 0)  // per-warp arrival (debug)
          trace[2048 + g * 4 + (warp - 2)] = clock64();
        mbar_arrive(&bars->p_full[b]);
      }
      // Epilogue: wait for the item's last PV, O / l -> bf16 rows; LSE (natural log).
      auto tre = [&](int slot) {  // debug: per-item epilogue stamps of warp 2
        if (trace != nullptr && blockIdx.x == 0 && q < 256 && threadIdx.x == 64) trace[4096 + q * 4 + slot] = clock64();
      };
      tre(0);
      mbar_wait(&bars->o_done[(g - 1) % kSBufs], ((g - 1) / kSBufs) & 1);
      tre(1);
      tc_fence_after();
      const float inv_l = l_run > 0.f ? 1.0f / l_run : 0.f;
      uint16_t* orow = out + (static_cast<size_t>(row0 + r) * hq + w.h) * D;
      uint32_t v[D / 32][32];
#pragma unroll
      for (int c = 0; c < D / 32; ++c) tmem_ld32(t_o + c * 32, v[c]);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&bars->o_free);  // O may be overwritten by item q + 1
      tre(2);
      if (nrows == B) {
        // Full tile: rows -> SW128 staging tile -> one TMA store per 64-column chunk, issued by
        // one thread and completed asynchronously. Row-per-thread global stores put 32 rows
        // (8 KB apart) in every warp store: ~1000 LSU cycles per item, 4% of the kernel.
        if (threadIdx.x == 64) bulk_wait_read();  // the previous item's store has read the tile
        named_bar_sync(1, 128);
        if (r < B) {
#pragma unroll
          for (int c = 0; c < D / 64; ++c) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int d0 = c * 64 + u * 8;
              uint4 q4;
              q4.x = pack_bf16x2(__uint_as_float(v[d0 / 32][d0 % 32]) * inv_l,
                                 __uint_as_float(v[d0 / 32][d0 % 32 + 1]) * inv_l);
              q4.y = pack_bf16x2(__uint_as_float(v[d0 / 32][d0 % 32 + 2]) * inv_l,
                                 __uint_as_float(v[d0 / 32][d0 % 32 + 3]) * inv_l);
              q4.z = pack_bf16x2(__uint_as_float(v[d0 / 32][d0 % 32 + 4]) * inv_l,
                                 __uint_as_float(v[d0 / 32][d0 % 32 + 5]) * inv_l);
              q4.w = pack_bf16x2(__uint_as_float(v[d0 / 32][d0 % 32 + 6]) * inv_l,
                                 __uint_as_float(v[d0 / 32][d0 % 32 + 7]) * inv_l);
              *reinterpret_cast<uint4*>(o_stage + c * (B * 128) + r * 128 + ((u ^ (r & 7)) << 4)) = q4;
            }
          }
        }
        fence_proxy_async_smem();
        named_bar_sync(1, 128);
        if (threadIdx.x == 64) {
#pragma unroll
          for (int c = 0; c < D / 64; ++c) tma_store_3d(&tm_o, o_stage + c * (B * 128), c * 64, w.h, row0);
          bulk_commit();
        }
      } else if (store) {  // the last (partial) tile of a sequence: the box would cross into the next
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t w16[16];
#pragma unroll
          for (int e = 0; e < 16; ++e)
            w16[e] = pack_bf16x2(__uint_as_float(v[c][2 * e]) * inv_l, __uint_as_float(v[c][2 * e + 1]) * inv_l);
          store_64B(orow + c * 32, w16);
        }
      }
      if (store) lse[static_cast<size_t>(w.h) * total_tokens + row0 + r] = (m_run + log2f(l_run)) * 0.69314718055994531f;
      tre(3);
      ++q;
    }
    if (threadIdx.x == 64) bulk_wait_all();  // outstanding O stores read smem and reach global
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem);
  }
}

// ------------------------------------------------------------------ two-stream variant
// The single-stream kernel above is paced by its softmax: one softmax warp per SM
// sub-partition, ~1300 busy cycles per key block plus ~300 cycles of fixed latency (TMEM
// load, P store wait, barrier) against a 1024-cycle MMA floor. Here each CTA runs TWO
// independent item streams (rounds k = s, s + 2, ... of its snake order), each with its own
// Q / K / V slots, S and O in TMEM (S0 | S1 | O0 | O1), producer warp, UMMA issuer warp and
// softmax warpgroup, so every sub-partition holds two softmax warps and the tensor core works
// on one stream while the other one's softmax runs. Per stream the order is QK_j, PV_j,
// QK_{j+1} (P_j aliases S_j): s_full(j) therefore implies PV_{j-1} completed and a lazy O
// rescale needs no wait. Registers: WG0 (producers, issuers) drops to 56, the softmax
// warpgroups rise to 224 (setmaxnreg).
constexpr int kThreads2 = 384;

template <int D, int B>
struct Fwd2Cfg {
  static constexpr int kChunks = D / 64;
  static constexpr int kQBytes = kChunks * kM * 128;
  static constexpr int kKVBytes = kChunks * B * 128;
  static constexpr int kSmemTiles = 2 * kQBytes + 4 * kKVBytes;  // per stream: Q, K, V
  static constexpr int kTmemO = 2 * B;                          // S_s at s * B, O_s at 2B + s * D
  static constexpr uint32_t kTmemCols = (2 * B + 2 * D) <= 256 ? 256 : 512;
  static constexpr int kSmemBytes = kSmemTiles + 1024 + 256;
};

struct Fwd2Bars {
  uint64_t q_full[2], q_empty[2], k_full[2], k_empty[2], v_full[2], v_empty[2];
  uint64_t s_full[2], p_full[2], o_done[2], o_free[2];
  uint32_t tmem_base;
};

template <int D, int B>
__global__ void __launch_bounds__(kThreads2, 1) attn_fwd2_kernel(
    const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
    const __grid_constant__ CUtensorMap tm_v, const int32_t* __restrict__ blk_off, int nseq, int total_tokens,
    int hq, int hkv, const int32_t* __restrict__ idx, int k_max, float scale_log2, uint16_t* __restrict__ out,
    float* __restrict__ lse, const sched::ItemRec* __restrict__ recs, int n_items,
    unsigned long long* __restrict__ trace) {
  using C = Fwd2Cfg<D, B>;
  // Debug timeline: CTA 0, per stream s and block g < 256: [s][g][slot] (slots: 0 k_full seen
  // + QK issued, 1 PV issued, 2 S seen by softmax warp 0, 3 P arrived, 4 epilogue start, 5 end).
  auto tr2 = [&](int st, int g, int slot) {
    if (trace != nullptr && blockIdx.x == 0 && g < 256) trace[(st * 256 + g) * 8 + slot] = clock64();
  };
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* q_smem = smem;                         // [stream]
  uint8_t* k_smem = smem + 2 * C::kQBytes;        // [stream]
  uint8_t* v_smem = k_smem + 2 * C::kKVBytes;     // [stream]
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
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

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
        for (sched::RecCursor cur(recs, n_items, grid, cta, s, 2);;) {
          const sched::ItemRec rec = cur.next();
          if (rec.it < 0) break;
          const Item w = from_rec(rec, nbt, idx, k_max);
          if (w.n <= 0) continue;
          const int hk = w.h / (hq / hkv);
          mbar_wait(&bars->q_empty[s], (q & 1) ^ 1);
          mbar_expect_tx(&bars->q_full[s], C::kQBytes);
          for (int c = 0; c < C::kChunks; ++c)
            tma_load_3d(qs + c * kM * 128, &tm_q, &bars->q_full[s], c * 64, w.h, w.seq0 + w.i * B);
          for (int j = 0; j < w.n; ++j, ++g) {
            const int kv_row = w.seq0 + __ldg(w.list + j) * B;
            mbar_wait(&bars->k_empty[s], (g & 1) ^ 1);
            mbar_expect_tx(&bars->k_full[s], C::kKVBytes);
            for (int c = 0; c < C::kChunks; ++c)
              tma_load_3d(ks + c * B * 128, &tm_k, &bars->k_full[s], c * 64, hk, kv_row);
            mbar_wait(&bars->v_empty[s], (g & 1) ^ 1);
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
      for (sched::RecCursor cur(recs, n_items, grid, cta, s, 2);;) {
        const sched::ItemRec rec = cur.next();
        if (rec.it < 0) break;
        const int n = rec.n;
        if (n <= 0) continue;
        mbar_wait(&bars->q_full[s], q & 1);
        for (int j = 0; j < n; ++j, ++g) {
          mbar_wait(&bars->k_full[s], g & 1);
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
          mbar_wait(&bars->v_full[s], g & 1);
          mbar_wait(&bars->p_full[s], g & 1);
          if (j == 0) mbar_wait(&bars->o_free[s], (q & 1) ^ 1);  // epilogue of the stream's previous item
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
    for (sched::RecCursor cur(recs, n_items, grid, cta, s, 2);;) {
      const sched::ItemRec rec = cur.next();
      if (rec.it < 0) break;
      const Item w = from_rec(rec, nbt, idx, k_max);
      const int row0 = w.seq0 + w.i * B;
      const int nrows = min(B, w.seq_len - w.i * B);
      const bool store = r < nrows;
      if (w.n <= 0) {  // nothing selected: zero output, LSE = -inf
        if (store) {
          uint4* dst = reinterpret_cast<uint4*>(out + (static_cast<size_t>(row0 + r) * hq + w.h) * D);
          for (int e = 0; e < D / 8; ++e) dst[e] = make_uint4(0, 0, 0, 0);
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
      if (store) {
        uint16_t* orow = out + (static_cast<size_t>(row0 + r) * hq + w.h) * D;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t w16[16];
#pragma unroll
          for (int e = 0; e < 16; ++e)
            w16[e] = pack_bf16x2(__uint_as_float(v[c][2 * e]) * inv_l, __uint_as_float(v[c][2 * e + 1]) * inv_l);
          store_64B(orow + c * 32, w16);
        }
        lse[static_cast<size_t>(w.h) * total_tokens + row0 + r] = (m_run + log2f(l_run)) * 0.69314718055994531f;
      }
      if (r == 0) tr2(s, g - 1, 5);
      ++q;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem);
  }
}

unsigned long long* g_trace = nullptr;  // debug timeline buffer (sb_debug_set_trace)

template <int D, int B>
void launch_fwd(const uint16_t* q, const uint16_t* k, const uint16_t* v, const int32_t* cu, const int32_t* blk_off,
                int nseq, int total, int nb_total, int hq, int hkv, const int32_t* idx, const int32_t* cnt, int hsel,
                int k_max, float scale, uint16_t* o, float* lse, void* ws, cudaStream_t st) {
  using C = FwdCfg<D, B>;
  const int n_items = hq * nb_total;
  const int32_t* order = sched::build_order(sched::CostFromCnt{cnt, k_max, hq, hsel, nb_total}, n_items, ws, st,
                                            "sb_sparse_attn_fwd/order");
  auto* recs = reinterpret_cast<sched::ItemRec*>(
      (reinterpret_cast<uintptr_t>(ws) + sched::order_workspace_bytes(n_items, hq * (k_max + 1)) + 255) & ~uintptr_t(255));
  sched::q_records_kernel<<<(n_items + 255) / 256, 256, 0, st>>>(order, n_items, cu, blk_off, nseq, nb_total, hq, hsel,
                                                                 idx, cnt, k_max, recs);
  launched("sb_sparse_attn_fwd/records");
  const CUtensorMap tq = make_thd_map(q, total, hq, D, kM);
  const CUtensorMap tk = make_thd_map(k, total, hkv, D, B);
  const CUtensorMap tv = make_thd_map(v, total, hkv, D, B);
  const CUtensorMap to = make_thd_map(o, total, hq, D, B);
  auto kern = attn_fwd_kernel<D, B>;
  cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes),
             "sb_sparse_attn_fwd: smem attribute");
  const int grid = std::min(n_items, sched::num_sms());
  static const bool two = [] {
    const char* e = std::getenv("SB_FWD_STREAMS");
    return !(e && e[0] == '1');
  }();
  if (two) {
    using C2 = Fwd2Cfg<D, B>;
    auto k2 = attn_fwd2_kernel<D, B>;
    cuda_check(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, C2::kSmemBytes),
               "sb_sparse_attn_fwd: smem attribute");
    k2<<<grid, kThreads2, C2::kSmemBytes, st>>>(tq, tk, tv, blk_off, nseq, total, hq, hkv, idx, k_max,
                                                scale * 1.4426950408889634f, o, lse, recs, n_items, g_trace);
    launched("sb_sparse_attn_fwd");
    return;
  }
  kern<<<grid, kThreads, C::kSmemBytes, st>>>(tq, tk, tv, to, cu, blk_off, nseq, total, hq, hkv, idx, cnt, hsel, k_max,
                                              scale * 1.4426950408889634f, o, lse, recs, n_items, g_trace);
  launched("sb_sparse_attn_fwd");
}

}  // namespace
}  // namespace sbk

// Debug only: device buffer of 256 x 32 uint64 for CTA 0's phase timeline (NULL disables).
SB_API void sb_debug_set_trace(unsigned long long* buf) { sbk::g_trace = buf; }

SB_API size_t sb_sparse_attn_fwd_workspace_size(int nb_total, int hq, int k_max) {
  return sbk::sched::order_workspace_bytes(nb_total * hq, hq * (k_max + 1)) + 256 +
         sbk::sched::rec_workspace_bytes(nb_total * hq);
}

SB_API int sb_sparse_attn_fwd(const uint16_t* q, const uint16_t* k, const uint16_t* v, const int32_t* cu_seqlens,
                              const int32_t* blk_off, int nseq, int total_tokens, int nb_total, int hq, int hkv,
                              int head_dim, int block_size, const int32_t* idx, const int32_t* cnt, int hsel,
                              int k_max, float scale, uint16_t* o, float* lse, void* workspace, void* stream) {
  return sbk::abi_call([&] {
    sbk::require(head_dim == 64 || head_dim == 128, "head_dim must be 64 or 128");
    sbk::require(block_size == 64 || block_size == 128, "block_size must be 64 or 128");
    sbk::require(hq >= 1 && hkv >= 1 && hq % hkv == 0, "hq must be a positive multiple of hkv");
    sbk::require(hsel >= 1 && hq % hsel == 0, "hsel must divide hq");
    sbk::require(k_max >= 1, "k_max must be >= 1");
    if (nseq == 0 || nb_total == 0 || total_tokens == 0) return;
    sbk::require(q && k && v && cu_seqlens && blk_off && idx && cnt && o && lse && workspace, "null pointer");
    sbk::require((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) % 16 == 0,
                 "q/k/v must be 16-byte aligned");
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
#define SB_FWD_CASE(DD, BB)                                                                                      \
  if (head_dim == DD && block_size == BB)                                                                        \
    return sbk::launch_fwd<DD, BB>(q, k, v, cu_seqlens, blk_off, nseq, total_tokens, nb_total, hq, hkv, idx, cnt, \
                                   hsel, k_max, scale, o, lse, workspace, st);
    SB_FWD_CASE(128, 128)
    SB_FWD_CASE(128, 64)
    SB_FWD_CASE(64, 128)
    SB_FWD_CASE(64, 64)
#undef SB_FWD_CASE
  });
}
