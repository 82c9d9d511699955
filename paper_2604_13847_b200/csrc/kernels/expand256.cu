// Block size 256 (the paper's MoBA setting; the reference default, config.hpp:21)
// on the B = 128 attention kernels. A selected 256-key block is two 128-key sub-blocks, and a
// 256-row query block is two 128-row query tiles, so the B = 256 selection maps exactly onto a
// B = 128 selection over a PADDED 128 layout in which every 256 block owns two 128 slots
// (blk_off128[s] = 2 * blk_off256[s]; a second slot past the sequence end is a ghost with no rows
// and no selection). For q tile a = 2i + half of parent row i with parent list j_0 < ... < j_{n-1}:
//   j < i  -> children 2j, 2j + 1 (the second only if it holds keys);
//   j == i -> half 0: child 2i (the diagonal; 2i + 1 lies wholly in the future of these rows);
//             half 1: children 2i (all keys in the past) and 2i + 1 (the diagonal).
// Children come out ascending because parents are. The key sets per query row, and hence the
// attention outputs and gradients, are identical to B = 256 semantics; the tensor cores run
// M = N = 128 tiles, whose TMEM budget the two-stream forward and the backward are built for.
#include <algorithm>

#include "common.cuh"
#include "sb_kernels.h"

namespace sbk {
namespace {

__global__ void blk_off_2x_kernel(const int32_t* __restrict__ blk_off256, int nseq, int32_t* __restrict__ blk_off128) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s <= nseq; s += gridDim.x * blockDim.x)
    blk_off128[s] = 2 * blk_off256[s];
}

// One thread per (selection head, 128 slot).
__global__ void expand_kernel(const int32_t* __restrict__ cu, const int32_t* __restrict__ blk_off256, int nseq,
                              int nb256, int hsel, const int32_t* __restrict__ idx, const int32_t* __restrict__ cnt,
                              int k_max, int32_t* __restrict__ idx128, int32_t* __restrict__ cnt128) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  const int nb128 = 2 * nb256;
  const long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (t >= static_cast<long long>(hsel) * nb128) return;
  const int hs = static_cast<int>(t / nb128);
  const int ga = static_cast<int>(t - static_cast<long long>(hs) * nb128);
  const int gi = ga >> 1, half = ga & 1;
  const int s = seq_of_block(blk_off256, nseq, gi);
  const int i = gi - blk_off256[s];
  const int len = cu[s + 1] - cu[s];
  const int a = 2 * i + half;  // local 128 slot
  int32_t* out = idx128 + (static_cast<size_t>(hs) * nb128 + ga) * (2 * k_max);
  int n = 0;
  if (a * 128 < len) {  // ghost slots (past the sequence end) keep an empty selection
    const size_t row = static_cast<size_t>(hs) * nb256 + gi;
    const int32_t* list = idx + row * k_max;
    const int c = cnt[row];
    for (int e = 0; e < c; ++e) {
      const int j = list[e];
      if (j < i) {
        out[n++] = 2 * j;
        if ((2 * j + 1) * 128 < len) out[n++] = 2 * j + 1;
      } else if (j == i) {
        out[n++] = 2 * i;
        if (half == 1) out[n++] = 2 * i + 1;
      }
    }
  }
  SB_DCHECK(n <= 2 * k_max);
  cnt128[static_cast<size_t>(hs) * nb128 + ga] = n;
  for (int e = n; e < 2 * k_max; ++e) out[e] = -1;
}

}  // namespace

size_t expand256_workspace_bytes(int nseq, int nb256, int hsel, int k_max) {
  const size_t a = (static_cast<size_t>(nseq + 1) * 4 + 255) & ~size_t(255);
  const size_t b = (static_cast<size_t>(hsel) * 2 * nb256 * 2 * k_max * 4 + 255) & ~size_t(255);
  const size_t c = (static_cast<size_t>(hsel) * 2 * nb256 * 4 + 255) & ~size_t(255);
  return a + b + c;
}

Expanded256 expand_selection_256(const int32_t* cu, const int32_t* blk_off256, int nseq, int nb256, int hsel,
                                 const int32_t* idx, const int32_t* cnt, int k_max, uint8_t* ws, cudaStream_t st) {
  Expanded256 e;
  e.blk_off = reinterpret_cast<int32_t*>(ws);
  const size_t a = (static_cast<size_t>(nseq + 1) * 4 + 255) & ~size_t(255);
  e.idx = reinterpret_cast<int32_t*>(ws + a);
  const size_t b = (static_cast<size_t>(hsel) * 2 * nb256 * 2 * k_max * 4 + 255) & ~size_t(255);
  e.cnt = reinterpret_cast<int32_t*>(ws + a + b);
  const size_t c = (static_cast<size_t>(hsel) * 2 * nb256 * 4 + 255) & ~size_t(255);
  e.used = a + b + c;
  e.nb_total = 2 * nb256;
  e.k_max = 2 * k_max;
  launch(blk_off_2x_kernel, std::max(1, std::min(64, (nseq + 256) / 256)), 256, 0, st, blk_off256, nseq, e.blk_off);
  launched("expand256/blk_off");
  const long long n = static_cast<long long>(hsel) * 2 * nb256;
  launch(expand_kernel, static_cast<unsigned>((n + 255) / 256), 256, 0, st, cu, blk_off256, nseq, nb256, hsel, idx, cnt,
                                                                          k_max, e.idx, e.cnt);
  launched("expand256/selection");
  return e;
}

}  // namespace sbk
