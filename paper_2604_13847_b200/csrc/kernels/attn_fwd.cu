// K5: varlen block-sparse attention forward on tcgen05 / TMEM (Eq. 2).
//
// One CTA owns one (q block, q head) work item: a 128-row Q tile (B=128: the block; B=64:
// the block plus 64 rows that are computed and discarded) and the list of selected key
// blocks of its selection row. Warp roles:
//   warp 0      TMA producer: Q once, then K_j / V_j of every selected block j into a
//               2-stage ring (each selected block is a contiguous B x D slab -> plain
//               tensor-map boxes, no element gather).
//   warp 1      TMEM allocator + single-thread UMMA issuer:
//                 S_j = Q K_j^T   (SS, M=128 N=B K=D)         -> TMEM S[j % 2]
//                 O  += P_j V_j   (TS, A = P_j from TMEM, B = V_j MN-major smem)
//               issue order QK_0, QK_1, PV_0, QK_2, PV_1, ... so QK_{j+1} overlaps softmax_j.
//   warps 2..5  softmax: one TMEM lane (= query row) per thread; online softmax in the
//               log2 domain with lazy O rescaling (only when the row max grows by > 8),
//               P_j written back into TMEM as packed bf16 over S_j, final O / l and LSE.
// Masking: keys past the sequence end and the causal upper triangle of the diagonal block.
#include "common.cuh"
#include "sb_kernels.h"
#include "sm100.cuh"
#include "tmap.cuh"

namespace sbk {
namespace {

using namespace sm100;

constexpr int kM = 128;            // UMMA M / Q tile rows
constexpr int kStages = 2;         // K and V ring depth
constexpr int kThreads = 192;      // 6 warps
constexpr float kRescaleThresh = 8.0f;  // log2 units: lazily rescale O only on a 256x max jump

template <int D, int B>
struct FwdCfg {
  static constexpr int kChunks = D / 64;                 // 128-byte swizzle atoms along D
  static constexpr int kQBytes = kChunks * kM * 128;     // Q tile
  static constexpr int kKVBytes = kChunks * B * 128;     // one K or V block
  static constexpr int kSmemTiles = kQBytes + 2 * kStages * kKVBytes;
  static constexpr int kTmemS0 = 0, kTmemS1 = B, kTmemO = 2 * B;
  static constexpr uint32_t kTmemCols = (2 * B + D) <= 256 ? 256 : 512;
  static constexpr int kSmemBytes = kSmemTiles + 1024 /*align slack*/ + 256 /*barriers*/;
};

struct FwdBars {
  uint64_t q_full;
  uint64_t k_full[kStages], k_empty[kStages];
  uint64_t v_full[kStages], v_empty[kStages];
  uint64_t s_full[2], p_full[2];
  uint64_t o_done;
  uint32_t tmem_base;
};

template <int D, int B>
__global__ void __launch_bounds__(kThreads, 1) attn_fwd_kernel(
    const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
    const __grid_constant__ CUtensorMap tm_v, const int32_t* __restrict__ cu, const int32_t* __restrict__ blk_off,
    int nseq, int total_tokens, int hq, int hkv, const int32_t* __restrict__ idx, const int32_t* __restrict__ cnt,
    int hsel, int k_max, float scale_log2, uint16_t* __restrict__ out, float* __restrict__ lse) {
  using C = FwdCfg<D, B>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* q_smem = smem;
  uint8_t* k_smem = smem + C::kQBytes;
  uint8_t* v_smem = k_smem + kStages * C::kKVBytes;
  FwdBars* bars = reinterpret_cast<FwdBars*>(smem + C::kSmemTiles);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gi = blockIdx.x, h = blockIdx.y;
  const int nbt = blk_off[nseq];
  const int s = seq_of_block(blk_off, nseq, gi);
  const int i = gi - blk_off[s];
  const int seq0 = cu[s];
  const int seq_len = cu[s + 1] - seq0;
  const int row0 = seq0 + i * B;
  const int nrows = min(B, seq_len - i * B);
  const int hk = h / (hq / hkv);
  const int srow = h / (hq / hsel);
  const int32_t* list = idx + (static_cast<size_t>(srow) * nbt + gi) * k_max;
  const int n = cnt[static_cast<size_t>(srow) * nbt + gi];

  if (threadIdx.x == 0) {
    mbar_init(&bars->q_full, 1);
    for (int st = 0; st < kStages; ++st) {
      mbar_init(&bars->k_full[st], 1);
      mbar_init(&bars->k_empty[st], 1);
      mbar_init(&bars->v_full[st], 1);
      mbar_init(&bars->v_empty[st], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars->s_full[b], 1);
      mbar_init(&bars->p_full[b], 128);
    }
    mbar_init(&bars->o_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && n > 0) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
      mbar_expect_tx(&bars->q_full, C::kQBytes);
      for (int c = 0; c < C::kChunks; ++c) tma_load_3d(q_smem + c * kM * 128, &tm_q, &bars->q_full, c * 64, h, row0);
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
    // ------------------------------------------------------------ UMMA issuer
    if (lane == 0 && n > 0) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(kM, B, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(kM, D, false, true);
      const uint32_t q_addr = smem_u32(q_smem), k_addr = smem_u32(k_smem), v_addr = smem_u32(v_smem);
      mbar_wait(&bars->q_full, 0);
      tc_fence_after();
      for (int j = 0; j <= n; ++j) {
        if (j < n) {
          const int st = j % kStages;
          mbar_wait(&bars->k_full[st], (j / kStages) & 1);
          tc_fence_after();
          const uint32_t d_s = tmem + ((j & 1) ? C::kTmemS1 : C::kTmemS0);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t koff = (kk & 3) * 32;  // 16 bf16 = 32 B inside the swizzle atom
            const uint64_t a = desc_sw128(q_addr + (kk >> 2) * (kM * 128) + koff, 16, 1024);
            const uint64_t b = desc_sw128(k_addr + st * C::kKVBytes + (kk >> 2) * (B * 128) + koff, 16, 1024);
            mma_ss(d_s, a, b, idesc_qk, kk > 0 ? 1u : 0u);
          }
          tc_commit(&bars->s_full[j & 1]);
          tc_commit(&bars->k_empty[st]);
        }
        if (j >= 1) {
          const int jj = j - 1;
          const int st = jj % kStages;
          mbar_wait(&bars->v_full[st], (jj / kStages) & 1);
          mbar_wait(&bars->p_full[jj & 1], (jj >> 1) & 1);
          tc_fence_after();
          const uint32_t p_tmem = tmem + ((jj & 1) ? C::kTmemS1 : C::kTmemS0);
#pragma unroll
          for (int kk = 0; kk < B / 16; ++kk) {
            const uint64_t b = desc_sw128(v_addr + st * C::kKVBytes + kk * 2048, B * 128, 1024);
            mma_ts(tmem + C::kTmemO, p_tmem + kk * 8, b, idesc_pv, (jj > 0 || kk > 0) ? 1u : 0u);
          }
          tc_commit(&bars->v_empty[st]);
          tc_commit(&bars->o_done);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int r = quarter * 32 + lane;
    const uint32_t lane_field = static_cast<uint32_t>(quarter * 32) << 16;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < n; ++j) {
      const int b = j & 1;
      const uint32_t t_s = tmem + lane_field + (b ? C::kTmemS1 : C::kTmemS0);
      const int jb = __ldg(list + j);
      mbar_wait(&bars->s_full[b], (j >> 1) & 1);
      tc_fence_after();
      float x[B];
#pragma unroll
      for (int c = 0; c < B / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(t_s + c * 32, v);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e) x[c * 32 + e] = __uint_as_float(v[e]);
      }
      // Valid keys: inside the sequence, and causal on the diagonal block.
      const int key_lim = min(B, seq_len - jb * B);
      const int causal_lim = (jb == i) ? r + 1 : B;
      const int lim = min(key_lim, causal_lim);
      float mblk = -INFINITY;
#pragma unroll
      for (int c = 0; c < B; ++c) {
        x[c] = (c < lim) ? x[c] * scale_log2 : -INFINITY;
        mblk = fmaxf(mblk, x[c]);
      }
      const float m_new = fmaxf(m_run, mblk);
      const bool rescale = m_new > m_run + kRescaleThresh;
      const float m_use = rescale ? m_new : m_run;
      const float alpha = rescale ? exp2f(m_run - m_use) : 1.0f;
      float sum = 0.f;
#pragma unroll
      for (int c = 0; c < B / 64; ++c) {
        uint32_t w[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float p0 = exp2f(x[c * 64 + 2 * e] - m_use), p1 = exp2f(x[c * 64 + 2 * e + 1] - m_use);
          sum += p0 + p1;
          w[e] = pack_bf16x2(p0, p1);
        }
        tmem_st32(t_s + c * 32, w);  // P_j (packed bf16) over the first B/2 columns of S_j
      }
      l_run = l_run * alpha + sum;
      tmem_wait_st();
      if (j > 0) {
        mbar_wait(&bars->o_done, (j - 1) & 1);  // PV_{j-1} finished writing O
        tc_fence_after();
        if (__any_sync(0xffffffffu, rescale)) {
          const uint32_t t_o = tmem + lane_field + C::kTmemO;
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
      mbar_arrive(&bars->p_full[b]);
    }
    // Epilogue: O / l -> bf16 rows; LSE (natural log).
    if (n > 0) {
      mbar_wait(&bars->o_done, (n - 1) & 1);
      tc_fence_after();
    }
    const float inv_l = (n > 0 && l_run > 0.f) ? 1.0f / l_run : 0.f;
    const bool store = r < nrows;
    uint16_t* orow = out + (static_cast<size_t>(row0 + r) * hq + h) * D;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t v[32];
      if (n > 0) {
        tmem_ld32(tmem + lane_field + C::kTmemO + c * 32, v);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = 0u;
      }
      if (store) {
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          uint4 w;
          w.x = pack_bf16x2(__uint_as_float(v[8 * e + 0]) * inv_l, __uint_as_float(v[8 * e + 1]) * inv_l);
          w.y = pack_bf16x2(__uint_as_float(v[8 * e + 2]) * inv_l, __uint_as_float(v[8 * e + 3]) * inv_l);
          w.z = pack_bf16x2(__uint_as_float(v[8 * e + 4]) * inv_l, __uint_as_float(v[8 * e + 5]) * inv_l);
          w.w = pack_bf16x2(__uint_as_float(v[8 * e + 6]) * inv_l, __uint_as_float(v[8 * e + 7]) * inv_l);
          dst[e] = w;
        }
      }
    }
    if (store)
      lse[static_cast<size_t>(h) * total_tokens + row0 + r] =
          (n > 0) ? (m_run + log2f(l_run)) * 0.69314718055994531f : -INFINITY;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem);
  }
}

template <int D, int B>
void launch_fwd(const uint16_t* q, const uint16_t* k, const uint16_t* v, const int32_t* cu, const int32_t* blk_off,
                int nseq, int total, int nb_total, int hq, int hkv, const int32_t* idx, const int32_t* cnt, int hsel,
                int k_max, float scale, uint16_t* o, float* lse, cudaStream_t st) {
  using C = FwdCfg<D, B>;
  const CUtensorMap tq = make_thd_map(q, total, hq, D, kM);
  const CUtensorMap tk = make_thd_map(k, total, hkv, D, B);
  const CUtensorMap tv = make_thd_map(v, total, hkv, D, B);
  auto kern = attn_fwd_kernel<D, B>;
  cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes),
             "sb_sparse_attn_fwd: smem attribute");
  dim3 grid(nb_total, hq);
  kern<<<grid, kThreads, C::kSmemBytes, st>>>(tq, tk, tv, cu, blk_off, nseq, total, hq, hkv, idx, cnt, hsel, k_max,
                                              scale * 1.4426950408889634f, o, lse);
  launched("sb_sparse_attn_fwd");
}

}  // namespace
}  // namespace sbk

SB_API size_t sb_sparse_attn_fwd_workspace_size(int nb_total, int hq) {
  (void)nb_total;
  (void)hq;
  return 0;
}

SB_API int sb_sparse_attn_fwd(const uint16_t* q, const uint16_t* k, const uint16_t* v, const int32_t* cu_seqlens,
                              const int32_t* blk_off, int nseq, int total_tokens, int nb_total, int hq, int hkv,
                              int head_dim, int block_size, const int32_t* idx, const int32_t* cnt, int hsel,
                              int k_max, float scale, uint16_t* o, float* lse, void* workspace, void* stream) {
  (void)workspace;
  return sbk::abi_call([&] {
    sbk::require(head_dim == 64 || head_dim == 128, "head_dim must be 64 or 128");
    sbk::require(block_size == 64 || block_size == 128, "block_size must be 64 or 128");
    sbk::require(hq >= 1 && hkv >= 1 && hq % hkv == 0, "hq must be a positive multiple of hkv");
    sbk::require(hsel >= 1 && hq % hsel == 0, "hsel must divide hq");
    sbk::require(k_max >= 1, "k_max must be >= 1");
    sbk::require(hq <= 65535, "hq too large");
    if (nseq == 0 || nb_total == 0 || total_tokens == 0) return;
    sbk::require(q && k && v && cu_seqlens && blk_off && idx && cnt && o && lse, "null pointer");
    sbk::require((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) % 16 == 0,
                 "q/k/v must be 16-byte aligned");
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
#define SB_FWD_CASE(DD, BB)                                                                                      \
  if (head_dim == DD && block_size == BB)                                                                        \
    return sbk::launch_fwd<DD, BB>(q, k, v, cu_seqlens, blk_off, nseq, total_tokens, nb_total, hq, hkv, idx, cnt, \
                                   hsel, k_max, scale, o, lse, st);
    SB_FWD_CASE(128, 128)
    SB_FWD_CASE(128, 64)
    SB_FWD_CASE(64, 128)
    SB_FWD_CASE(64, 64)
#undef SB_FWD_CASE
  });
}
