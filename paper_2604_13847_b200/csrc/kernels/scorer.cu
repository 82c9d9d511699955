// K1 block mean-pool and K2 block scorer (MoBA gate: PAPER.md:119).
//
// K1 streams X [T][H][D] once with 128-bit coalesced loads (CTAs split each block's
// contiguous B x H x D slab by columns) and writes the fp32 block means: HBM-bound.
// K2 forms the per-sequence lower-triangular score matrix S = scale * Qbar Kbar^T (64 rows per
// CTA, 8 per thread, Kbar staged through shared memory in 32-key chunks).
#include "common.cuh"
#include "sb_kernels.h"

namespace sbk {
namespace {

constexpr int kPoolThreads = 128;
constexpr int kPoolRows = 8;  // rows in flight per thread

// CTA (gi, y): block gi, 16-byte column chunks [128 y, 128 y + 128) of the flattened [H*D]
// row, one chunk per thread, the block's valid rows accumulated in fp32 in row order (the
// same per-element sum as the one-CTA-per-block kernel this replaced). Splitting the columns
// over grid.y gives C2 1024 CTAs (~7 per SM, no 1-vs-2 CTA imbalance across SMs) instead of
// 256 whole-slab CTAs.
__global__ void __launch_bounds__(kPoolThreads) block_pool_kernel(
    const uint16_t* __restrict__ x, const int32_t* __restrict__ cu, const int32_t* __restrict__ blk_off,
    int nseq, int row_elems, int block_size, float* __restrict__ xbar) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  const int gi = blockIdx.x;
  const int ch = blockIdx.y * kPoolThreads + threadIdx.x;
  const int chunks = row_elems >> 3;
  if (ch >= chunks) return;
  const int s = seq_of_block(blk_off, nseq, gi);
  const int i = gi - blk_off[s];
  const int t0 = cu[s] + i * block_size;
  const int rows = min(t0 + block_size, cu[s + 1]) - t0;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  const uint4* base = reinterpret_cast<const uint4*>(x + static_cast<size_t>(t0) * row_elems) + ch;
  auto add = [&](const uint4& v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      acc[2 * e] += __uint_as_float(w[e] << 16);
      acc[2 * e + 1] += __uint_as_float(w[e] & 0xffff0000u);
    }
  };
  int r = 0;
  for (; r + kPoolRows <= rows; r += kPoolRows) {
    uint4 v[kPoolRows];
#pragma unroll
    for (int u = 0; u < kPoolRows; ++u) v[u] = __ldg(base + static_cast<size_t>(r + u) * chunks);
#pragma unroll
    for (int u = 0; u < kPoolRows; ++u) add(v[u]);
  }
  for (; r < rows; ++r) add(__ldg(base + static_cast<size_t>(r) * chunks));
  const float inv = 1.0f / static_cast<float>(rows);
  float4* out = reinterpret_cast<float4*>(xbar + static_cast<size_t>(gi) * row_elems);
  out[2 * ch] = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
  out[2 * ch + 1] = make_float4(acc[4] * inv, acc[5] * inv, acc[6] * inv, acc[7] * inv);
}

constexpr int kRowsPerCta = 64;  // score rows per CTA
constexpr int kColsPerCta = 64;  // keys per CTA (two 32-key chunks)
constexpr int kRowsPerThread = 8;

// Scores of 64 consecutive rows i x 64 consecutive keys j of sequence s, q head h (CTA x = one
// lower-triangular (row tile, column tile) pair, so a long sequence's rows are not one CTA's
// serial chain of key chunks). The rows' Qbar are staged once,
// transposed ([d][row]); Kbar goes through shared memory in 32-key chunks ([d][key]).
// Thread (warp w, lane l) computes rows i0 + 8w .. i0 + 8w + 7 against key j0 + l: per d one
// 4-byte load of Kbar and two broadcast float4 loads of Qbar feed 8 FMAs. The one-warp-per-row
// kernel this replaced (one 4-byte load per FMA) was shared-memory bound: 66 us per C3 layer.
// Every score is still acc = fma over d = 0..D-1 in order from 0, times scale: bit-identical.
template <int D>
__global__ void __launch_bounds__(256) block_scores_kernel(
    const float* __restrict__ qbar, const float* __restrict__ kbar, const int32_t* __restrict__ blk_off,
    const int64_t* __restrict__ tri_off, int nseq, int hq, int hkv, float scale, int tiles,
    float* __restrict__ scores) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  constexpr int kV = D / 4;  // float4 per row
  const int s = blockIdx.y, h = blockIdx.z;
  const int nb = blk_off[s + 1] - blk_off[s];
  // blockIdx.x enumerates the lower-triangular (row tile, column tile) pairs: x = rt (rt + 1) / 2 + ct.
  int rt = static_cast<int>((sqrtf(8.0f * blockIdx.x + 1.0f) - 1.0f) * 0.5f);
  while ((rt + 1) * (rt + 2) / 2 <= static_cast<int>(blockIdx.x)) ++rt;
  while (rt * (rt + 1) / 2 > static_cast<int>(blockIdx.x)) --rt;
  const int ct = blockIdx.x - rt * (rt + 1) / 2;
  (void)tiles;
  const int i0 = rt * kRowsPerCta, jt0 = ct * kColsPerCta;
  if (i0 >= nb) return;
  const int b0 = blk_off[s];
  const int hk = h / (hq / hkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = warp * kRowsPerThread;
  const int i_last = min(i0 + kRowsPerCta - 1, nb - 1);
  __shared__ __align__(16) float qt[D][kRowsPerCta];
  __shared__ float kt[D][32];
  {  // all loads in flight before the transposed stores (consecutive threads: consecutive rows)
    constexpr int kQ = kRowsPerCta * kV / 256;
    float4 x[kQ];
#pragma unroll
    for (int u = 0; u < kQ; ++u) {
      const int e = threadIdx.x + u * 256, r = e % kRowsPerCta, c = e / kRowsPerCta;
      x[u] = i0 + r < nb ? __ldg(reinterpret_cast<const float4*>(qbar + (static_cast<size_t>(b0 + i0 + r) * hq + h) * D) + c)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < kQ; ++u) {
      const int e = threadIdx.x + u * 256, r = e % kRowsPerCta, c = e / kRowsPerCta;
      qt[4 * c][r] = x[u].x;
      qt[4 * c + 1][r] = x[u].y;
      qt[4 * c + 2][r] = x[u].z;
      qt[4 * c + 3][r] = x[u].w;
    }
  }
  float* sbase = scores + static_cast<size_t>(h) * tri_off[nseq] + tri_off[s];
  for (int j0 = jt0; j0 <= i_last && j0 < jt0 + kColsPerCta; j0 += 32) {
    __syncthreads();  // the previous chunk is consumed (first pass: qt is written)
    {
      constexpr int kK = 32 * kV / 256;
      float4 x[kK];
#pragma unroll
      for (int u = 0; u < kK; ++u) {
        const int e = threadIdx.x + u * 256, jr = e % 32, c = e / 32;  // consecutive threads: consecutive keys
        const int j = j0 + jr;
        x[u] = j <= i_last ? __ldg(reinterpret_cast<const float4*>(kbar + (static_cast<size_t>(b0 + j) * hkv + hk) * D) + c)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kK; ++u) {
        const int e = threadIdx.x + u * 256, jr = e % 32, c = e / 32;
        kt[4 * c][jr] = x[u].x;
        kt[4 * c + 1][jr] = x[u].y;
        kt[4 * c + 2][jr] = x[u].z;
        kt[4 * c + 3][jr] = x[u].w;
      }
    }
    __syncthreads();
    if (i0 + r0 + kRowsPerThread - 1 < j0 || i0 + r0 > i_last) continue;  // this warp's rows: all above the chunk
    float acc[kRowsPerThread];
#pragma unroll
    for (int u = 0; u < kRowsPerThread; ++u) acc[u] = 0.f;
#pragma unroll 8
    for (int d = 0; d < D; ++d) {
      const float kv = kt[d][lane];
      const float4 qa = *reinterpret_cast<const float4*>(&qt[d][r0]);
      const float4 qb = *reinterpret_cast<const float4*>(&qt[d][r0 + 4]);
      acc[0] = fmaf(qa.x, kv, acc[0]);
      acc[1] = fmaf(qa.y, kv, acc[1]);
      acc[2] = fmaf(qa.z, kv, acc[2]);
      acc[3] = fmaf(qa.w, kv, acc[3]);
      acc[4] = fmaf(qb.x, kv, acc[4]);
      acc[5] = fmaf(qb.y, kv, acc[5]);
      acc[6] = fmaf(qb.z, kv, acc[6]);
      acc[7] = fmaf(qb.w, kv, acc[7]);
    }
    const int j = j0 + lane;
#pragma unroll
    for (int u = 0; u < kRowsPerThread; ++u) {
      const int i = i0 + r0 + u;
      if (i <= i_last && j <= i) sbase[static_cast<int64_t>(i) * (i + 1) / 2 + j] = acc[u] * scale;
    }
  }
}

}  // namespace
}  // namespace sbk

SB_API int sb_block_pool(const uint16_t* x, const int32_t* cu_seqlens, const int32_t* blk_off, int nseq,
                         int nb_total, int heads, int head_dim, int block_size, float* xbar, void* stream) {
  return sbk::abi_call([&] {
    sbk::require(heads >= 1 && (head_dim == 64 || head_dim == 128), "heads >= 1 and head_dim in {64,128}");
    sbk::require(block_size == 64 || block_size == 128 || block_size == 256, "block_size must be 64, 128 or 256");
    if (nb_total == 0 || nseq == 0) return;
    sbk::require(x && cu_seqlens && blk_off && xbar, "null pointer");
    const dim3 grid(nb_total, (heads * head_dim / 8 + sbk::kPoolThreads - 1) / sbk::kPoolThreads);
    sbk::launch(sbk::block_pool_kernel, grid, sbk::kPoolThreads, 0, static_cast<cudaStream_t>(stream), 
        x, cu_seqlens, blk_off, nseq, heads * head_dim, block_size, xbar);
    sbk::launched("sb_block_pool");
  });
}

SB_API int sb_block_scores(const float* qbar, const float* kbar, const int32_t* blk_off, const int64_t* tri_off,
                           int nseq, int nb_max, int hq, int hkv, int head_dim, float scale, float* scores,
                           void* stream) {
  return sbk::abi_call([&] {
    sbk::require(hq >= 1 && hkv >= 1 && hq % hkv == 0, "hq must be a positive multiple of hkv");
    sbk::require(head_dim == 64 || head_dim == 128, "head_dim must be 64 or 128");
    if (nseq == 0 || nb_max == 0) return;
    sbk::require(qbar && kbar && blk_off && tri_off && scores, "null pointer");
    sbk::require(nseq <= 65535 && hq <= 65535, "nseq and hq must be <= 65535");
    const int tiles = (nb_max + sbk::kRowsPerCta - 1) / sbk::kRowsPerCta;
    sbk::require(static_cast<long long>(tiles) * (tiles + 1) / 2 < (1ll << 31), "nb_max too large");
    dim3 grid(tiles * (tiles + 1) / 2, nseq, hq);  // lower-triangular tile pairs
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (head_dim == 128) {
      sbk::launch(sbk::block_scores_kernel<128>, grid, 256, 0, st, qbar, kbar, blk_off, tri_off, nseq, hq, hkv, scale, tiles, scores);
    } else {
      sbk::launch(sbk::block_scores_kernel<64>, grid, 256, 0, st, qbar, kbar, blk_off, tri_off, nseq, hq, hkv, scale, tiles, scores);
    }
    sbk::launched("sb_block_scores");
  });
}
