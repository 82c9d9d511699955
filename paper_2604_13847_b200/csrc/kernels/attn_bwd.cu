// K6 (+K7): varlen block-sparse attention backward on tcgen05 / TMEM.
//
// Deterministic two-pass design (no floating-point atomics):
//   prep      lse2 = LSE * log2(e) and D = rowsum(dO * O) into a padded [Hq][Tp] workspace.
//   K7        transposed selection: for every (kv head, key block) the ordered list of the
//             selection rows (head, q block) that selected it (count pass, scan, fill pass;
//             each list is enumerated in a fixed order by one warp, so it is deterministic).
//   dkv pass  one CTA per (key block, kv head), 128 TMEM lanes = key rows; for every
//             (q head, q block) in its list:  S^T = K Q^T, dP^T = V dO^T  (SS UMMA),
//             P^T = exp2(S^T * scale*log2e - lse2), dS^T = P^T (dP^T - D) written back to TMEM
//             as bf16, then dV += P^T dO and dK += dS^T Q (TS UMMA, A operand from TMEM).
//   dq pass   one CTA per (q block, q head), TMEM lanes = query rows; for every selected key
//             block: S = Q K^T, dP = dO V^T, dS = P (dP - D) -> TMEM bf16, dQ += dS K.
// Warp roles as in the forward kernel: warp 0 TMA producer, warp 1 TMEM allocator + UMMA
// issuer, warps 2..5 the elementwise softmax-gradient math (one TMEM lane per thread).
#include "common.cuh"
#include "sb_kernels.h"
#include "sm100.cuh"
#include "tmap.cuh"

namespace sbk {
namespace {

using namespace sm100;

constexpr int kM = 128;
constexpr int kStages = 2;
constexpr int kThreads = 192;
constexpr float kLog2e = 1.4426950408889634f;

__host__ __device__ constexpr uint32_t pow2_cols(int c) { return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512; }

// ------------------------------------------------------------------------------------ prep
__global__ void bwd_prep_kernel(const uint16_t* __restrict__ o, const uint16_t* __restrict__ d_o,
                                const float* __restrict__ lse, int total, int hq, int d, int tp,
                                float* __restrict__ lse2, float* __restrict__ dvec) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int per_lane = d / 32;  // 2 or 4 bf16
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < total * hq; row += warps) {
    const int t = row / hq, h = row - t * hq;
    const uint16_t* a = o + static_cast<size_t>(row) * d + lane * per_lane;
    const uint16_t* b = d_o + static_cast<size_t>(row) * d + lane * per_lane;
    float acc = 0.f;
    for (int e = 0; e < per_lane; ++e) acc += bf2f(a[e]) * bf2f(b[e]);
#pragma unroll
    for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) {
      dvec[static_cast<size_t>(h) * tp + t] = acc;
      lse2[static_cast<size_t>(h) * tp + t] = lse[static_cast<size_t>(h) * total + t] * kLog2e;
    }
  }
  // Padding columns [total, tp): never read for valid rows, but keep them finite.
  const int pad = tp - total;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < hq * pad; e += gridDim.x * blockDim.x) {
    const int h = e / pad, t = total + e % pad;
    dvec[static_cast<size_t>(h) * tp + t] = 0.f;
    lse2[static_cast<size_t>(h) * tp + t] = 0.f;
  }
}

// ------------------------------------------------------------------------------------ K7
// Warp w = hk * NB + gj enumerates candidate selection rows (hs in hk's range, q block i >= j of
// the same sequence) in (hs, i) order and finds key block j by binary search in the row's
// ascending index list. pass 0 writes the count, pass 1 the entries (hs * NB + gi).
__global__ void transpose_sel_kernel(const int32_t* __restrict__ idx, const int32_t* __restrict__ cnt,
                                     const int32_t* __restrict__ blk_off, int nseq, int hkv, int rows_per_kv,
                                     int k_max, int pass, int32_t* __restrict__ tr_cnt,
                                     const int32_t* __restrict__ tr_off, int32_t* __restrict__ tr_ent) {
  const int nbt = blk_off[nseq];
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= hkv * nbt) return;
  const int hk = w / nbt, gj = w - hk * nbt;
  const int s = seq_of_block(blk_off, nseq, gj);
  const int j = gj - blk_off[s];
  const int nb = blk_off[s + 1] - blk_off[s];
  const int span = nb - j;
  const int total = rows_per_kv * span;
  int found = 0;
  int32_t* dst = pass ? tr_ent + tr_off[w] : nullptr;
  for (int c0 = 0; c0 < total; c0 += 32) {
    const int c = c0 + lane;
    bool hit = false;
    int key = 0;
    if (c < total) {
      const int hs = hk * rows_per_kv + c / span;
      const int gi = blk_off[s] + j + c % span;
      const size_t row = static_cast<size_t>(hs) * nbt + gi;
      const int32_t* list = idx + row * k_max;
      int lo = 0, hi = cnt[row];  // ascending list
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (list[mid] < j) lo = mid + 1; else hi = mid;
      }
      hit = lo < cnt[row] && list[lo] == j;
      key = hs * nbt + gi;
    }
    const uint32_t m = __ballot_sync(0xffffffffu, hit);
    if (pass && hit) dst[found + __popc(m & ((1u << lane) - 1u))] = key;
    found += __popc(m);
  }
  if (!pass && lane == 0) tr_cnt[w] = found;
}

// Exclusive scan of n ints (single CTA of 1024 threads).
__global__ void __launch_bounds__(1024) scan_kernel(const int32_t* __restrict__ in, int n, int32_t* __restrict__ out) {
  __shared__ int warp_sum[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int base = 0; base < n; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < n ? in[i] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int ws = warp_sum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, ws, o);
        if (lane >= o) ws += y;
      }
      warp_sum[lane] = ws;
    }
    __syncthreads();
    const int excl = carry + (warp ? warp_sum[warp - 1] : 0) + x - v;
    if (i < n) out[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = carry;
}

// ------------------------------------------------------------------------------------ dkv
template <int D, int B>
struct DkvCfg {
  static constexpr int kChunks = D / 64;
  static constexpr int kTileBytes = kChunks * kM * 128;  // K or V (128 key rows)
  static constexpr int kQBytes = kChunks * B * 128;      // Q_i or dO_i (B query rows)
  static constexpr int kVecBytes = 2 * B * 4;            // lse2 + D for B rows
  static constexpr int kSmemTiles = 2 * kTileBytes + kStages * (2 * kQBytes) + kStages * kVecBytes;
  static constexpr int kSt = 0, kDPt = B, kDV = 2 * B, kDK = 2 * B + D;
  static constexpr uint32_t kCols = pow2_cols(2 * B + 2 * D);
  static constexpr int kSmemBytes = kSmemTiles + 1024 + 256;
};

struct DkvBars {
  uint64_t kv_full;
  uint64_t q_full[kStages], q_empty[kStages];
  uint64_t s_full, p_full, done;
  uint32_t tmem_base;
};

template <int D, int B>
__global__ void __launch_bounds__(kThreads, 1) attn_bwd_dkv_kernel(
    const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
    const int32_t* __restrict__ cu, const int32_t* __restrict__ blk_off, int nseq, int hq, int hkv, int hsel,
    const int32_t* __restrict__ tr_off, const int32_t* __restrict__ tr_ent, const float* __restrict__ lse2,
    const float* __restrict__ dvec, int tp, float scale, float scale_log2, uint16_t* __restrict__ dk,
    uint16_t* __restrict__ dv) {
  using C = DkvCfg<D, B>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* k_smem = smem;
  uint8_t* v_smem = smem + C::kTileBytes;
  uint8_t* q_smem = smem + 2 * C::kTileBytes;            // [stage]
  uint8_t* do_smem = q_smem + kStages * C::kQBytes;      // [stage]
  float* vec_smem = reinterpret_cast<float*>(do_smem + kStages * C::kQBytes);  // [stage][2][B]
  DkvBars* bars = reinterpret_cast<DkvBars*>(smem + C::kSmemTiles);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gj = blockIdx.x, hk = blockIdx.y;
  const int nbt = blk_off[nseq];
  const int s = seq_of_block(blk_off, nseq, gj);
  const int jl = gj - blk_off[s];
  const int seq0 = cu[s], seq_len = cu[s + 1] - seq0;
  const int kv0 = seq0 + jl * B;
  const int nkv = min(B, seq_len - jl * B);
  const int w = hk * nbt + gj;
  const int e0 = tr_off[w], ne = tr_off[w + 1] - e0;
  const int sg = hq / hsel;          // q heads per selection row
  const int items = ne * sg;

  if (threadIdx.x == 0) {
    mbar_init(&bars->kv_full, 1);
    for (int st = 0; st < kStages; ++st) {
      mbar_init(&bars->q_full[st], 2);  // TMA expect_tx arrive + vector-copy arrive
      mbar_init(&bars->q_empty[st], 1);
    }
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->p_full, 128);
    mbar_init(&bars->done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kCols>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  auto item_head = [&](int m, int& h, int& gi) {
    const int ent = __ldg(tr_ent + e0 + m / sg);
    const int hs = ent / nbt;
    gi = ent - hs * nbt;
    h = hs * sg + m % sg;
  };

  if (warp == 0) {
    if (items > 0) {
      if (lane == 0) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        tma_prefetch(&tm_do);
        mbar_expect_tx(&bars->kv_full, 2 * C::kTileBytes);
        for (int c = 0; c < C::kChunks; ++c) {
          tma_load_3d(k_smem + c * kM * 128, &tm_k, &bars->kv_full, c * 64, hk, kv0);
          tma_load_3d(v_smem + c * kM * 128, &tm_v, &bars->kv_full, c * 64, hk, kv0);
        }
      }
      for (int m = 0; m < items; ++m) {
        const int st = m % kStages;
        const uint32_t ph = (m / kStages) & 1;
        int h, gi;
        item_head(m, h, gi);
        const int q0 = seq0 + (gi - blk_off[s]) * B;
        const int nq = min(B, seq_len - (gi - blk_off[s]) * B);
        mbar_wait(&bars->q_empty[st], ph ^ 1);
        if (lane == 0) {
          mbar_expect_tx(&bars->q_full[st], 2 * C::kQBytes);
          for (int c = 0; c < C::kChunks; ++c) {
            tma_load_3d(q_smem + st * C::kQBytes + c * B * 128, &tm_q, &bars->q_full[st], c * 64, h, q0);
            tma_load_3d(do_smem + st * C::kQBytes + c * B * 128, &tm_do, &bars->q_full[st], c * 64, h, q0);
          }
        }
        float* vs = vec_smem + st * 2 * B;
        for (int r = lane; r < B; r += 32) {
          const bool ok = r < nq;
          vs[r] = ok ? __ldg(lse2 + static_cast<size_t>(h) * tp + q0 + r) : 0.f;
          vs[B + r] = ok ? __ldg(dvec + static_cast<size_t>(h) * tp + q0 + r) : 0.f;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->q_full[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && items > 0) {
      constexpr uint32_t idesc_t = idesc_bf16_f32(kM, B, false, false);
      constexpr uint32_t idesc_acc = idesc_bf16_f32(kM, D, false, true);
      const uint32_t k_addr = smem_u32(k_smem), v_addr = smem_u32(v_smem);
      mbar_wait(&bars->kv_full, 0);
      for (int m = 0; m < items; ++m) {
        const int st = m % kStages;
        mbar_wait(&bars->q_full[st], (m / kStages) & 1);
        tc_fence_after();
        const uint32_t qa = smem_u32(q_smem + st * C::kQBytes), da = smem_u32(do_smem + st * C::kQBytes);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off_m = (kk >> 2) * (kM * 128) + (kk & 3) * 32;
          const uint32_t off_n = (kk >> 2) * (B * 128) + (kk & 3) * 32;
          mma_ss(tmem + C::kSt, desc_sw128(k_addr + off_m, 16, 1024), desc_sw128(qa + off_n, 16, 1024), idesc_t,
                 kk > 0);
          mma_ss(tmem + C::kDPt, desc_sw128(v_addr + off_m, 16, 1024), desc_sw128(da + off_n, 16, 1024), idesc_t,
                 kk > 0);
        }
        tc_commit(&bars->s_full);
        mbar_wait(&bars->p_full, m & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < B / 16; ++kk) {
          const uint32_t acc = (m > 0 || kk > 0) ? 1u : 0u;
          mma_ts(tmem + C::kDV, tmem + C::kSt + kk * 8, desc_sw128(da + kk * 2048, B * 128, 1024), idesc_acc, acc);
          mma_ts(tmem + C::kDK, tmem + C::kDPt + kk * 8, desc_sw128(qa + kk * 2048, B * 128, 1024), idesc_acc, acc);
        }
        tc_commit(&bars->q_empty[st]);
      }
      tc_commit(&bars->done);
    }
  } else {
    const int quarter = warp & 3;
    const int c = quarter * 32 + lane;  // key row
    const uint32_t lf = static_cast<uint32_t>(quarter * 32) << 16;
    for (int m = 0; m < items; ++m) {
      const int st = m % kStages;
      int h, gi;
      item_head(m, h, gi);
      const int il = gi - blk_off[s];
      const int nq = min(B, seq_len - il * B);
      const bool diag = il == jl;
      const float* vs = vec_smem + st * 2 * B;
      mbar_wait(&bars->q_full[st], (m / kStages) & 1);  // producer's plain smem writes of vs
      mbar_wait(&bars->s_full, m & 1);
      tc_fence_after();
#pragma unroll
      for (int c2 = 0; c2 < B / 32; ++c2) {
        uint32_t sv[32], pv[32];
        tmem_ld32(tmem + lf + C::kSt + c2 * 32, sv);
        tmem_ld32(tmem + lf + C::kDPt + c2 * 32, pv);
        tmem_wait_ld();
        uint32_t pp[16], dd[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          float p[2], ds[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int r = c2 * 32 + e + u;
            const bool ok = r < nq && (!diag || c <= r);
            p[u] = ok ? exp2f(__uint_as_float(sv[e + u]) * scale_log2 - vs[r]) : 0.f;
            ds[u] = p[u] * (__uint_as_float(pv[e + u]) - vs[B + r]);
          }
          pp[e / 2] = pack_bf16x2(p[0], p[1]);
          dd[e / 2] = pack_bf16x2(ds[0], ds[1]);
        }
        tmem_st16(tmem + lf + C::kSt + c2 * 16, pp);
        tmem_st16(tmem + lf + C::kDPt + c2 * 16, dd);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&bars->p_full);
    }
    if (items > 0) {
      mbar_wait(&bars->done, 0);
      tc_fence_after();
    }
    const bool store = c < nkv;
    uint16_t* dv_row = dv + (static_cast<size_t>(kv0 + c) * hkv + hk) * D;
    uint16_t* dk_row = dk + (static_cast<size_t>(kv0 + c) * hkv + hk) * D;
#pragma unroll
    for (int part = 0; part < 2; ++part) {
      const uint32_t col = part == 0 ? C::kDV : C::kDK;
      const float mul = part == 0 ? 1.0f : scale;
      uint16_t* row = part == 0 ? dv_row : dk_row;
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t v[32];
        if (items > 0) {
          tmem_ld32(tmem + lf + col + cc * 32, v);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = 0u;
        }
        if (store) {
          uint4* dst = reinterpret_cast<uint4*>(row + cc * 32);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            uint4 q4;
            q4.x = pack_bf16x2(__uint_as_float(v[8 * e + 0]) * mul, __uint_as_float(v[8 * e + 1]) * mul);
            q4.y = pack_bf16x2(__uint_as_float(v[8 * e + 2]) * mul, __uint_as_float(v[8 * e + 3]) * mul);
            q4.z = pack_bf16x2(__uint_as_float(v[8 * e + 4]) * mul, __uint_as_float(v[8 * e + 5]) * mul);
            q4.w = pack_bf16x2(__uint_as_float(v[8 * e + 6]) * mul, __uint_as_float(v[8 * e + 7]) * mul);
            dst[e] = q4;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kCols>(tmem);
  }
}

// ------------------------------------------------------------------------------------ dq
template <int D, int B>
struct DqCfg {
  static constexpr int kChunks = D / 64;
  static constexpr int kQBytes = kChunks * kM * 128;   // Q or dO tile (128 rows)
  static constexpr int kKVBytes = kChunks * B * 128;   // K_j or V_j
  static constexpr int kSmemTiles = 2 * kQBytes + 2 * kStages * kKVBytes;
  static constexpr int kS = 0, kDP = B, kDQ = 2 * B;
  static constexpr uint32_t kCols = pow2_cols(2 * B + D);
  static constexpr int kSmemBytes = kSmemTiles + 1024 + 256;
};

struct DqBars {
  uint64_t qdo_full;
  uint64_t k_full[kStages], k_empty[kStages], v_full[kStages], v_empty[kStages];
  uint64_t s_full, ds_full, done;
  uint32_t tmem_base;
};

template <int D, int B>
__global__ void __launch_bounds__(kThreads, 1) attn_bwd_dq_kernel(
    const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
    const int32_t* __restrict__ cu, const int32_t* __restrict__ blk_off, int nseq, int hq, int hkv,
    const int32_t* __restrict__ idx, const int32_t* __restrict__ cnt, int hsel, int k_max,
    const float* __restrict__ lse2, const float* __restrict__ dvec, int tp, float scale, float scale_log2,
    uint16_t* __restrict__ dq) {
  using C = DqCfg<D, B>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* q_smem = smem;
  uint8_t* do_smem = smem + C::kQBytes;
  uint8_t* k_smem = smem + 2 * C::kQBytes;
  uint8_t* v_smem = k_smem + kStages * C::kKVBytes;
  DqBars* bars = reinterpret_cast<DqBars*>(smem + C::kSmemTiles);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gi = blockIdx.x, h = blockIdx.y;
  const int nbt = blk_off[nseq];
  const int s = seq_of_block(blk_off, nseq, gi);
  const int i = gi - blk_off[s];
  const int seq0 = cu[s], seq_len = cu[s + 1] - seq0;
  const int row0 = seq0 + i * B;
  const int nrows = min(B, seq_len - i * B);
  const int hk = h / (hq / hkv);
  const int srow = h / (hq / hsel);
  const int32_t* list = idx + (static_cast<size_t>(srow) * nbt + gi) * k_max;
  const int n = cnt[static_cast<size_t>(srow) * nbt + gi];

  if (threadIdx.x == 0) {
    mbar_init(&bars->qdo_full, 1);
    for (int st = 0; st < kStages; ++st) {
      mbar_init(&bars->k_full[st], 1);
      mbar_init(&bars->k_empty[st], 1);
      mbar_init(&bars->v_full[st], 1);
      mbar_init(&bars->v_empty[st], 1);
    }
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->ds_full, 128);
    mbar_init(&bars->done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kCols>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0) {
    if (lane == 0 && n > 0) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
      tma_prefetch(&tm_do);
      mbar_expect_tx(&bars->qdo_full, 2 * C::kQBytes);
      for (int c = 0; c < C::kChunks; ++c) {
        tma_load_3d(q_smem + c * kM * 128, &tm_q, &bars->qdo_full, c * 64, h, row0);
        tma_load_3d(do_smem + c * kM * 128, &tm_do, &bars->qdo_full, c * 64, h, row0);
      }
      for (int j = 0; j < n; ++j) {
        const int st = j % kStages;
        const uint32_t ph = (j / kStages) & 1;
        const int kv_row = seq0 + __ldg(list + j) * B;
        mbar_wait(&bars->k_empty[st], ph ^ 1);
        mbar_expect_tx(&bars->k_full[st], C::kKVBytes);
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d(k_smem + st * C::kKVBytes + c * B * 128, &tm_k, &bars->k_full[st], c * 64, hk, kv_row);
        mbar_wait(&bars->v_empty[st], ph ^ 1);
        mbar_expect_tx(&bars->v_full[st], C::kKVBytes);
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d(v_smem + st * C::kKVBytes + c * B * 128, &tm_v, &bars->v_full[st], c * 64, hk, kv_row);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && n > 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(kM, B, false, false);
      constexpr uint32_t idesc_dq = idesc_bf16_f32(kM, D, false, true);
      const uint32_t q_addr = smem_u32(q_smem), do_addr = smem_u32(do_smem);
      const uint32_t k_addr = smem_u32(k_smem), v_addr = smem_u32(v_smem);
      mbar_wait(&bars->qdo_full, 0);
      auto issue_dq = [&](int jj) {
        const int st = jj % kStages;
        mbar_wait(&bars->ds_full, jj & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < B / 16; ++kk)
          mma_ts(tmem + C::kDQ, tmem + C::kS + kk * 8, desc_sw128(k_addr + st * C::kKVBytes + kk * 2048, B * 128, 1024),
                 idesc_dq, (jj > 0 || kk > 0) ? 1u : 0u);
        tc_commit(&bars->k_empty[st]);
      };
      for (int j = 0; j < n; ++j) {
        const int st = j % kStages;
        mbar_wait(&bars->k_full[st], (j / kStages) & 1);
        mbar_wait(&bars->v_full[st], (j / kStages) & 1);
        tc_fence_after();
        if (j > 0) issue_dq(j - 1);  // frees S (dS alias) before S_j overwrites it (in-order pipe)
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off_m = (kk >> 2) * (kM * 128) + (kk & 3) * 32;
          const uint32_t off_n = (kk >> 2) * (B * 128) + (kk & 3) * 32;
          mma_ss(tmem + C::kS, desc_sw128(q_addr + off_m, 16, 1024),
                 desc_sw128(k_addr + st * C::kKVBytes + off_n, 16, 1024), idesc_s, kk > 0);
          mma_ss(tmem + C::kDP, desc_sw128(do_addr + off_m, 16, 1024),
                 desc_sw128(v_addr + st * C::kKVBytes + off_n, 16, 1024), idesc_s, kk > 0);
        }
        tc_commit(&bars->v_empty[st]);
        tc_commit(&bars->s_full);
      }
      issue_dq(n - 1);
      tc_commit(&bars->done);
    }
  } else {
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t lf = static_cast<uint32_t>(quarter * 32) << 16;
    const bool valid = r < nrows;
    const float l2 = valid ? __ldg(lse2 + static_cast<size_t>(h) * tp + row0 + r) : 0.f;
    const float dd = valid ? __ldg(dvec + static_cast<size_t>(h) * tp + row0 + r) : 0.f;
    for (int j = 0; j < n; ++j) {
      const int jb = __ldg(list + j);
      const int key_lim = min(B, seq_len - jb * B);
      const int lim = valid ? min(key_lim, jb == i ? r + 1 : B) : 0;
      mbar_wait(&bars->s_full, j & 1);
      tc_fence_after();
#pragma unroll
      for (int c2 = 0; c2 < B / 32; ++c2) {
        uint32_t sv[32], pv[32];
        tmem_ld32(tmem + lf + C::kS + c2 * 32, sv);
        tmem_ld32(tmem + lf + C::kDP + c2 * 32, pv);
        tmem_wait_ld();
        uint32_t dsp[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          float ds[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int col = c2 * 32 + e + u;
            const float p = col < lim ? exp2f(__uint_as_float(sv[e + u]) * scale_log2 - l2) : 0.f;
            ds[u] = p * (__uint_as_float(pv[e + u]) - dd);
          }
          dsp[e / 2] = pack_bf16x2(ds[0], ds[1]);
        }
        tmem_st16(tmem + lf + C::kS + c2 * 16, dsp);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&bars->ds_full);
    }
    if (n > 0) {
      mbar_wait(&bars->done, 0);
      tc_fence_after();
    }
    uint16_t* row = dq + (static_cast<size_t>(row0 + r) * hq + h) * D;
#pragma unroll
    for (int cc = 0; cc < D / 32; ++cc) {
      uint32_t v[32];
      if (n > 0) {
        tmem_ld32(tmem + lf + C::kDQ + cc * 32, v);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = 0u;
      }
      if (valid) {
        uint4* dst = reinterpret_cast<uint4*>(row + cc * 32);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          uint4 q4;
          q4.x = pack_bf16x2(__uint_as_float(v[8 * e + 0]) * scale, __uint_as_float(v[8 * e + 1]) * scale);
          q4.y = pack_bf16x2(__uint_as_float(v[8 * e + 2]) * scale, __uint_as_float(v[8 * e + 3]) * scale);
          q4.z = pack_bf16x2(__uint_as_float(v[8 * e + 4]) * scale, __uint_as_float(v[8 * e + 5]) * scale);
          q4.w = pack_bf16x2(__uint_as_float(v[8 * e + 6]) * scale, __uint_as_float(v[8 * e + 7]) * scale);
          dst[e] = q4;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kCols>(tmem);
  }
}

// ------------------------------------------------------------------------------------ host
struct BwdWorkspace {
  size_t lse2, dvec, tr_cnt, tr_off, tr_ent, total;
  int tp;
};

inline size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

BwdWorkspace bwd_layout(int total, int nb_total, int hq, int hkv, int hsel, int k_max) {
  BwdWorkspace w;
  w.tp = ((total + 3) / 4) * 4 + 128;
  size_t off = 0;
  w.lse2 = off;
  off = align256(off + static_cast<size_t>(hq) * w.tp * 4);
  w.dvec = off;
  off = align256(off + static_cast<size_t>(hq) * w.tp * 4);
  w.tr_cnt = off;
  off = align256(off + static_cast<size_t>(hkv) * nb_total * 4);
  w.tr_off = off;
  off = align256(off + (static_cast<size_t>(hkv) * nb_total + 1) * 4);
  w.tr_ent = off;
  off = align256(off + static_cast<size_t>(hsel) * nb_total * k_max * 4);
  w.total = off;
  return w;
}

template <int D, int B>
void launch_bwd(const uint16_t* q, const uint16_t* k, const uint16_t* v, const uint16_t* o, const uint16_t* d_o,
                const float* lse, const int32_t* cu, const int32_t* blk_off, int nseq, int total, int nb_total, int hq,
                int hkv, const int32_t* idx, const int32_t* cnt, int hsel, int k_max, float scale, uint16_t* dq,
                uint16_t* dk, uint16_t* dv, uint8_t* ws, cudaStream_t st) {
  const BwdWorkspace w = bwd_layout(total, nb_total, hq, hkv, hsel, k_max);
  float* lse2 = reinterpret_cast<float*>(ws + w.lse2);
  float* dvec = reinterpret_cast<float*>(ws + w.dvec);
  int32_t* tr_cnt = reinterpret_cast<int32_t*>(ws + w.tr_cnt);
  int32_t* tr_off = reinterpret_cast<int32_t*>(ws + w.tr_off);
  int32_t* tr_ent = reinterpret_cast<int32_t*>(ws + w.tr_ent);
  const float scale_log2 = scale * kLog2e;

  bwd_prep_kernel<<<592, 256, 0, st>>>(o, d_o, lse, total, hq, D, w.tp, lse2, dvec);
  launched("sb_sparse_attn_bwd/prep");
  const int warps = hkv * nb_total;
  const int rows_per_kv = hsel / hkv;
  transpose_sel_kernel<<<(warps + 3) / 4, 128, 0, st>>>(idx, cnt, blk_off, nseq, hkv, rows_per_kv, k_max, 0, tr_cnt,
                                                         nullptr, nullptr);
  launched("sb_sparse_attn_bwd/transpose_count");
  scan_kernel<<<1, 1024, 0, st>>>(tr_cnt, warps, tr_off);
  launched("sb_sparse_attn_bwd/scan");
  transpose_sel_kernel<<<(warps + 3) / 4, 128, 0, st>>>(idx, cnt, blk_off, nseq, hkv, rows_per_kv, k_max, 1, tr_cnt,
                                                         tr_off, tr_ent);
  launched("sb_sparse_attn_bwd/transpose_fill");

  // dK / dV: key tiles are 128 rows (UMMA M); query tiles are B rows (UMMA N).
  {
    using C = DkvCfg<D, B>;
    const CUtensorMap tq = make_thd_map(q, total, hq, D, B);
    const CUtensorMap tdo = make_thd_map(d_o, total, hq, D, B);
    const CUtensorMap tk = make_thd_map(k, total, hkv, D, kM);
    const CUtensorMap tv = make_thd_map(v, total, hkv, D, kM);
    auto kern = attn_bwd_dkv_kernel<D, B>;
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes),
               "sb_sparse_attn_bwd: smem attribute (dkv)");
    kern<<<dim3(nb_total, hkv), kThreads, C::kSmemBytes, st>>>(tq, tk, tv, tdo, cu, blk_off, nseq, hq, hkv, hsel,
                                                               tr_off, tr_ent, lse2, dvec, w.tp, scale, scale_log2,
                                                               dk, dv);
    launched("sb_sparse_attn_bwd/dkv");
  }
  {
    using C = DqCfg<D, B>;
    const CUtensorMap tq = make_thd_map(q, total, hq, D, kM);
    const CUtensorMap tdo = make_thd_map(d_o, total, hq, D, kM);
    const CUtensorMap tk = make_thd_map(k, total, hkv, D, B);
    const CUtensorMap tv = make_thd_map(v, total, hkv, D, B);
    auto kern = attn_bwd_dq_kernel<D, B>;
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes),
               "sb_sparse_attn_bwd: smem attribute (dq)");
    kern<<<dim3(nb_total, hq), kThreads, C::kSmemBytes, st>>>(tq, tk, tv, tdo, cu, blk_off, nseq, hq, hkv, idx, cnt,
                                                              hsel, k_max, lse2, dvec, w.tp, scale, scale_log2, dq);
    launched("sb_sparse_attn_bwd/dq");
  }
}

}  // namespace
}  // namespace sbk

SB_API size_t sb_sparse_attn_bwd_workspace_size(int total_tokens, int nb_total, int hq, int hkv, int head_dim, int hsel,
                                                int k_max) {
  (void)head_dim;
  return sbk::bwd_layout(total_tokens, nb_total, hq, hkv, hsel, k_max).total;
}

SB_API int sb_sparse_attn_bwd(const uint16_t* q, const uint16_t* k, const uint16_t* v, const uint16_t* o,
                              const uint16_t* d_o, const float* lse, const int32_t* cu_seqlens, const int32_t* blk_off,
                              int nseq, int total_tokens, int nb_total, int hq, int hkv, int head_dim, int block_size,
                              const int32_t* idx, const int32_t* cnt, int hsel, int k_max, float scale, uint16_t* dq,
                              uint16_t* dk, uint16_t* dv, void* workspace, void* stream) {
  return sbk::abi_call([&] {
    sbk::require(head_dim == 64 || head_dim == 128, "head_dim must be 64 or 128");
    sbk::require(block_size == 64 || block_size == 128, "block_size must be 64 or 128");
    sbk::require(hq >= 1 && hkv >= 1 && hq % hkv == 0, "hq must be a positive multiple of hkv");
    sbk::require(hsel >= hkv && hq % hsel == 0 && hsel % hkv == 0,
                 "hsel must divide hq and be a multiple of hkv (each selection row maps to one kv head)");
    sbk::require(k_max >= 1, "k_max must be >= 1");
    if (nseq == 0 || nb_total == 0 || total_tokens == 0) return;
    sbk::require(q && k && v && o && d_o && lse && cu_seqlens && blk_off && idx && cnt && dq && dk && dv && workspace,
                 "null pointer");
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint8_t* ws = static_cast<uint8_t*>(workspace);
#define SB_BWD_CASE(DD, BB)                                                                                     \
  if (head_dim == DD && block_size == BB)                                                                       \
    return sbk::launch_bwd<DD, BB>(q, k, v, o, d_o, lse, cu_seqlens, blk_off, nseq, total_tokens, nb_total, hq, \
                                   hkv, idx, cnt, hsel, k_max, scale, dq, dk, dv, ws, st);
    SB_BWD_CASE(128, 128)
    SB_BWD_CASE(128, 64)
    SB_BWD_CASE(64, 128)
    SB_BWD_CASE(64, 64)
#undef SB_BWD_CASE
  });
}
