// K1 block mean-pool and K2 block scorer (MoBA gate: PAPER.md:119).
//
// K1 streams X [T][H][D] once with 128-bit coalesced loads (one CTA per block covers the
// whole contiguous B x H x D slab) and writes the fp32 block means: HBM-bound.
// K2 forms the per-sequence lower-triangular score matrix S = scale * Qbar Kbar^T as a
// tiled fp32 GEMM (64 x 64 tiles, only tiles on/below the diagonal launch work).
#include "common.cuh"
#include "sb_kernels.h"

namespace sbk {
namespace {

constexpr int kPoolThreads = 256;
constexpr int kPoolMaxChunks = 4;  // (H*D/8) / 256 <= 4  ->  H*D <= 8192

// One CTA per global block. Thread c owns 16-byte column chunk(s) c, c+256, ... of the
// flattened [H*D] row and accumulates the block's valid rows in fp32.
__global__ void __launch_bounds__(kPoolThreads) block_pool_kernel(
    const uint16_t* __restrict__ x, const int32_t* __restrict__ cu, const int32_t* __restrict__ blk_off,
    int nseq, int row_elems, int block_size, float* __restrict__ xbar) {
  const int gi = blockIdx.x;
  const int s = seq_of_block(blk_off, nseq, gi);
  const int i = gi - blk_off[s];
  const int t0 = cu[s] + i * block_size;
  const int t1 = min(t0 + block_size, cu[s + 1]);
  const int chunks = row_elems >> 3;
  float acc[kPoolMaxChunks][8];
#pragma unroll
  for (int c = 0; c < kPoolMaxChunks; ++c)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[c][e] = 0.f;

  const uint4* base = reinterpret_cast<const uint4*>(x + static_cast<size_t>(t0) * row_elems);
  const int rows = t1 - t0;
  int r = 0;
  // Four rows in flight per iteration for memory-level parallelism.
  for (; r + 4 <= rows; r += 4) {
    uint4 v[4][kPoolMaxChunks];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c = 0; c < kPoolMaxChunks; ++c) {
        const int ch = threadIdx.x + c * kPoolThreads;
        if (ch < chunks) v[u][c] = __ldg(base + static_cast<size_t>(r + u) * chunks + ch);
      }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c = 0; c < kPoolMaxChunks; ++c) {
        const int ch = threadIdx.x + c * kPoolThreads;
        if (ch < chunks) {
          const uint32_t w[4] = {v[u][c].x, v[u][c].y, v[u][c].z, v[u][c].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            acc[c][2 * e] += __uint_as_float(w[e] << 16);
            acc[c][2 * e + 1] += __uint_as_float(w[e] & 0xffff0000u);
          }
        }
      }
  }
  for (; r < rows; ++r) {
#pragma unroll
    for (int c = 0; c < kPoolMaxChunks; ++c) {
      const int ch = threadIdx.x + c * kPoolThreads;
      if (ch < chunks) {
        const uint4 vv = __ldg(base + static_cast<size_t>(r) * chunks + ch);
        const uint32_t w[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          acc[c][2 * e] += __uint_as_float(w[e] << 16);
          acc[c][2 * e + 1] += __uint_as_float(w[e] & 0xffff0000u);
        }
      }
    }
  }
  const float inv = 1.0f / static_cast<float>(rows);
  float4* out = reinterpret_cast<float4*>(xbar + static_cast<size_t>(gi) * row_elems);
#pragma unroll
  for (int c = 0; c < kPoolMaxChunks; ++c) {
    const int ch = threadIdx.x + c * kPoolThreads;
    if (ch < chunks) {
      out[2 * ch] = make_float4(acc[c][0] * inv, acc[c][1] * inv, acc[c][2] * inv, acc[c][3] * inv);
      out[2 * ch + 1] = make_float4(acc[c][4] * inv, acc[c][5] * inv, acc[c][6] * inv, acc[c][7] * inv);
    }
  }
}

constexpr int kRowsPerCta = 8;  // one warp per score row

// Scores of 8 consecutive rows i of sequence s, q head h (one warp per row): the rows' Qbar
// and 32-key chunks of Kbar (transposed, conflict-free) are staged in shared memory and lane
// l computes S[i][j0 + l] for j0 + l <= i. Every score is acc = fma over d = 0..D-1 in order
// from 0, times scale -- the same operation sequence as the 64x64-tile kernel this replaced
// (bit-identical output), which launched mostly-empty CTAs and ran four latency-bound rounds
// each (36 us on C2).
template <int D>
__global__ void __launch_bounds__(256) block_scores_kernel(
    const float* __restrict__ qbar, const float* __restrict__ kbar, const int32_t* __restrict__ blk_off,
    const int64_t* __restrict__ tri_off, int nseq, int hq, int hkv, float scale, float* __restrict__ scores) {
  constexpr int kV = D / 4;  // float4 per row
  const int s = blockIdx.y, h = blockIdx.z;
  const int nb = blk_off[s + 1] - blk_off[s];
  const int i0 = blockIdx.x * kRowsPerCta;
  if (i0 >= nb) return;
  const int b0 = blk_off[s];
  const int hk = h / (hq / hkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = i0 + warp;
  const int i_last = min(i0 + kRowsPerCta - 1, nb - 1);
  __shared__ float4 qs[kRowsPerCta][kV];
  __shared__ float kt[D][33];
  for (int e = threadIdx.x; e < kRowsPerCta * kV; e += blockDim.x) {
    const int r = e / kV, c = e % kV;
    qs[r][c] = i0 + r < nb ? reinterpret_cast<const float4*>(qbar + (static_cast<size_t>(b0 + i0 + r) * hq + h) * D)[c]
                           : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float* srow = scores + static_cast<size_t>(h) * tri_off[nseq] + tri_off[s] + static_cast<int64_t>(i) * (i + 1) / 2;
  for (int j0 = 0; j0 <= i_last; j0 += 32) {
    __syncthreads();  // the previous chunk is consumed (first pass: qs is written)
    for (int e = threadIdx.x; e < 32 * kV; e += blockDim.x) {
      const int jr = e / kV, c = e % kV;
      const int j = j0 + jr;
      const float4 x = j <= i_last ? reinterpret_cast<const float4*>(kbar + (static_cast<size_t>(b0 + j) * hkv + hk) * D)[c]
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
      kt[4 * c][jr] = x.x;
      kt[4 * c + 1][jr] = x.y;
      kt[4 * c + 2][jr] = x.z;
      kt[4 * c + 3][jr] = x.w;
    }
    __syncthreads();
    const int j = j0 + lane;
    if (i <= i_last && j <= i) {
      float acc = 0.f;
#pragma unroll
      for (int c = 0; c < kV; ++c) {
        const float4 qv = qs[warp][c];
        acc = fmaf(qv.x, kt[4 * c][lane], acc);
        acc = fmaf(qv.y, kt[4 * c + 1][lane], acc);
        acc = fmaf(qv.z, kt[4 * c + 2][lane], acc);
        acc = fmaf(qv.w, kt[4 * c + 3][lane], acc);
      }
      srow[j] = acc * scale;
    }
  }
}

}  // namespace
}  // namespace sbk

SB_API int sb_block_pool(const uint16_t* x, const int32_t* cu_seqlens, const int32_t* blk_off, int nseq,
                         int nb_total, int heads, int head_dim, int block_size, float* xbar, void* stream) {
  return sbk::abi_call([&] {
    sbk::require(heads >= 1 && (head_dim == 64 || head_dim == 128), "heads >= 1 and head_dim in {64,128}");
    sbk::require(heads * head_dim <= 8 * 256 * 4, "heads * head_dim must be <= 8192");
    sbk::require(block_size == 64 || block_size == 128, "block_size must be 64 or 128");
    if (nb_total == 0 || nseq == 0) return;
    sbk::require(x && cu_seqlens && blk_off && xbar, "null pointer");
    sbk::block_pool_kernel<<<nb_total, sbk::kPoolThreads, 0, static_cast<cudaStream_t>(stream)>>>(
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
    dim3 grid((nb_max + sbk::kRowsPerCta - 1) / sbk::kRowsPerCta, nseq, hq);
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (head_dim == 128) {
      sbk::block_scores_kernel<128><<<grid, 256, 0, st>>>(qbar, kbar, blk_off, tri_off, nseq, hq, hkv, scale, scores);
    } else {
      sbk::block_scores_kernel<64><<<grid, 256, 0, st>>>(qbar, kbar, blk_off, tri_off, nseq, hq, hkv, scale, scores);
    }
    sbk::launched("sb_block_scores");
  });
}
