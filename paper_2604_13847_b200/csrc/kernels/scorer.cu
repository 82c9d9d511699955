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

constexpr int kTile = 64;
constexpr int kTk = 32;

// S tile (ti, tj) of sequence s, q head h: rows i in [64 ti, 64 ti + 64), cols j in
// [64 tj, ...), only j <= i < nb_s written. 256 threads, 4x4 outputs per thread.
__global__ void __launch_bounds__(256) block_scores_kernel(
    const float* __restrict__ qbar, const float* __restrict__ kbar, const int32_t* __restrict__ blk_off,
    const int64_t* __restrict__ tri_off, int nseq, int hq, int hkv, int d, float scale,
    float* __restrict__ scores) {
  const int ti = blockIdx.x, tj = blockIdx.y;
  if (tj > ti) return;
  const int s = blockIdx.z / hq;
  const int h = blockIdx.z % hq;
  const int nb = blk_off[s + 1] - blk_off[s];
  if (ti * kTile >= nb) return;
  const int hk = h / (hq / hkv);
  const int b0 = blk_off[s];

  __shared__ float qs[kTk][kTile + 4];
  __shared__ float ks[kTk][kTile + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int c0 = 0; c0 < d; c0 += kTk) {
    // Load 64 rows x 32 cols of Qbar and Kbar (transposed into [col][row]).
    for (int e = threadIdx.x; e < kTile * kTk; e += 256) {
      const int row = e / kTk, col = e % kTk;
      const int qi = ti * kTile + row, kj = tj * kTile + row;
      qs[col][row] = qi < nb ? qbar[(static_cast<size_t>(b0 + qi) * hq + h) * d + c0 + col] : 0.f;
      ks[col][row] = kj < nb ? kbar[(static_cast<size_t>(b0 + kj) * hkv + hk) * d + c0 + col] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int c = 0; c < kTk; ++c) {
      float a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = qs[c][ty + 16 * u];
        b[u] = ks[c][tx + 16 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int w = 0; w < 4; ++w) acc[u][w] = fmaf(a[u], b[w], acc[u][w]);
    }
    __syncthreads();
  }
  const int64_t tri_total = tri_off[nseq];
  float* srow = scores + static_cast<size_t>(h) * tri_total + tri_off[s];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int i = ti * kTile + ty + 16 * u;
    if (i >= nb) continue;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int j = tj * kTile + tx + 16 * w;
      if (j <= i) srow[static_cast<int64_t>(i) * (i + 1) / 2 + j] = acc[u][w] * scale;
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
    sbk::require(head_dim % sbk::kTk == 0 && head_dim > 0, "head_dim must be a multiple of 32");
    if (nseq == 0 || nb_max == 0) return;
    sbk::require(qbar && kbar && blk_off && tri_off && scores, "null pointer");
    const int tiles = (nb_max + sbk::kTile - 1) / sbk::kTile;
    sbk::require(static_cast<int64_t>(nseq) * hq <= 65535, "nseq * hq must be <= 65535");
    dim3 grid(tiles, tiles, nseq * hq);
    sbk::block_scores_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        qbar, kbar, blk_off, tri_off, nseq, hq, hkv, head_dim, scale, scores);
    sbk::launched("sb_block_scores");
  });
}
