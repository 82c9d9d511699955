// K3 per-query-block top-k block selector and K4 coverage profile / coverage-at-grid.
//
// Selector: rows of up to 256 candidates (sequences up to 32K tokens at B=128) take one WARP
// per row: 8 candidates per lane in registers, the k-th largest 32-bit order key found by a
// 32-step bitwise radix select on warp ballots (no shared memory, no block barriers), ties at
// the threshold resolved to the lowest block index with ordered ballot prefix counts. Longer
// rows take one CTA: candidates in registers, a 4-pass 8-bit radix select over shared-memory
// histograms and block-wide ordered ballot scans. Both produce exactly "score descending,
// index ascending", already in ascending index order without a sort.
// Profile: per-row softmax masses sorted descending (bitonic sort in shared memory), then a
// deterministic per-(sequence, rank) fp64 reduction over (head, row).
#include "common.cuh"
#include "sb_kernels.h"

namespace sbk {
namespace {

constexpr int kSelThreads = 128;
constexpr int kSelPerThread = 32;  // candidates per row <= 4096
constexpr int kMaxRow = kSelThreads * kSelPerThread;

// Order-preserving float -> uint32 key after canonicalisation (NaN -> -inf, -0 -> +0).
__device__ __forceinline__ uint32_t order_key(float v) {
  if (v != v) v = -INFINITY;
  if (v == 0.0f) v = 0.0f;
  const uint32_t u = __float_as_uint(v);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Block-wide exclusive prefix over one flag per thread, threads ordered by index.
// Returns this thread's prefix; *total gets the block total. Uses warp ballots.
__device__ __forceinline__ int block_excl_scan(bool flag, int* warp_tot, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t b = __ballot_sync(0xffffffffu, flag);
  if (lane == 0) warp_tot[warp] = __popc(b);
  __syncthreads();
  int before = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kSelThreads / 32; ++w) {
    const int c = warp_tot[w];
    before += (w < warp) ? c : 0;
    tot += c;
  }
  __syncthreads();
  *total = tot;
  return before + __popc(b & ((1u << lane) - 1u));
}

constexpr int kWarpRow = 256;  // rows up to this many candidates: one warp per row
constexpr int kArgmaxRounds = 8;  // keep counts up to this: iterated warp argmax instead of the radix select

__global__ void __launch_bounds__(256) topk_select_warp_kernel(
    const float* __restrict__ scores, const int32_t* __restrict__ blk_off, const int64_t* __restrict__ tri_off,
    int nseq, int nbt, int group, const int32_t* __restrict__ k_seq, int k_max, int force_diag,
    int32_t* __restrict__ idx, int32_t* __restrict__ cnt) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int gi = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int g = blockIdx.y;
  if (gi >= nbt) return;
  const int s = seq_of_block(blk_off, nseq, gi);
  const int i = gi - blk_off[s];
  const int n = i + 1;
  if (n > kWarpRow) return;  // long rows: topk_select_kernel
  const int64_t tri = tri_off[nseq];
  // k_seq is clamped to the row length and to the idx row stride k_max (a caller passing
  // k_seq > k_max gets k_max blocks, never writes past its row).
  const int k = max(1, min(min(k_seq[s], n), k_max));
  int32_t* out = idx + (static_cast<size_t>(g) * nbt + gi) * k_max;
  SB_DCHECK(k >= 1 && k <= k_max && gi < nbt);
  if (lane == 0) cnt[static_cast<size_t>(g) * nbt + gi] = k;
  const int m = force_diag ? n - 1 : n;     // candidate count
  const int want = force_diag ? k - 1 : k;  // candidates to keep
  if (want >= m) {
    for (int r = lane; r < k_max; r += 32) out[r] = r < n ? r : -1;
    return;
  }
  if (want == 0) {
    for (int r = lane; r < k_max; r += 32) out[r] = r == 0 ? i : -1;
    return;
  }
  const int64_t row_off = tri_off[s] + static_cast<int64_t>(i) * (i + 1) / 2;
  const float* base = scores + static_cast<size_t>(g) * group * tri + row_off;
  uint32_t key[kWarpRow / 32];
#pragma unroll
  for (int r = 0; r < kWarpRow / 32; ++r) {
    const int j = r * 32 + lane;
    float v = -INFINITY;
    if (j < m) {
      v = __ldg(base + j);
      for (int q = 1; q < group; ++q) v += __ldg(base + static_cast<size_t>(q) * tri + j);
    }
    key[r] = j < m ? order_key(v) : 0u;
  }
  const int slots = (m + 31) >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  if (want <= kArgmaxRounds) {
    // Few to keep (C3: k = 5): `want` rounds of a warp argmax over (key, ~index), i.e. score
    // descending, index ascending -- the same set as the radix select below in ~1/3 of its
    // instructions. Valid keys are > 0 (order_key(-inf) = 0x007FFFFF), so 0 marks taken / past m.
    uint32_t taken = 0;  // bit r: candidate r * 32 + lane is kept
#pragma unroll 1
    for (int t = 0; t < want; ++t) {
      unsigned long long best = 0ull;
#pragma unroll
      for (int r = 0; r < kWarpRow / 32; ++r) {
        if (r >= slots) break;
        const int j = r * 32 + lane;
        const unsigned long long c =
            (j < m && !((taken >> r) & 1u)) ? (static_cast<unsigned long long>(key[r]) << 32) | static_cast<uint32_t>(~j)
                                            : 0ull;
        best = c > best ? c : best;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, best, o);
        best = x > best ? x : best;
      }
      const int jw = static_cast<int>(~static_cast<uint32_t>(best));
      if ((jw & 31) == lane) taken |= 1u << (jw >> 5);
    }
    int kept_before = 0;
#pragma unroll
    for (int r = 0; r < kWarpRow / 32; ++r) {
      if (r >= slots) break;
      const bool keep = (taken >> r) & 1u;
      const uint32_t kb = __ballot_sync(0xffffffffu, keep);
      if (keep) out[kept_before + __popc(kb & lt)] = r * 32 + lane;
      kept_before += __popc(kb);
    }
    for (int r = lane; r < k_max; r += 32) {
      if (r == want && force_diag) out[r] = i;
      else if (r >= k) out[r] = -1;
    }
    return;
  }
  // Bitwise radix select of the want-th largest key among the m candidates.
  uint32_t prefix = 0;
  int remaining = want;
#pragma unroll 1
  for (int bit = 31; bit >= 0; --bit) {
    const uint32_t hi_mask = bit == 31 ? 0u : (0xffffffffu << (bit + 1));
    int c = 0;
#pragma unroll
    for (int r = 0; r < kWarpRow / 32; ++r) {
      if (r >= slots) break;
      const int j = r * 32 + lane;
      const bool hit = j < m && (key[r] & hi_mask) == prefix && ((key[r] >> bit) & 1u);
      c += __popc(__ballot_sync(0xffffffffu, hit));
    }
    if (c >= remaining) {
      prefix |= 1u << bit;
    } else {
      remaining -= c;
    }
  }
  const uint32_t thresh = prefix;  // keys > thresh all kept; `remaining` of the == thresh kept
  int ties_before = 0, kept_before = 0;
#pragma unroll
  for (int r = 0; r < kWarpRow / 32; ++r) {
    if (r >= slots) break;
    const int j = r * 32 + lane;
    const bool valid = j < m;
    const bool tie = valid && key[r] == thresh;
    const uint32_t tb = __ballot_sync(0xffffffffu, tie);
    const bool keep = valid && (key[r] > thresh || (tie && ties_before + __popc(tb & lt) < remaining));
    const uint32_t kb = __ballot_sync(0xffffffffu, keep);
    if (keep) out[kept_before + __popc(kb & lt)] = j;
    ties_before += __popc(tb);
    kept_before += __popc(kb);
  }
  for (int r = lane; r < k_max; r += 32) {
    if (r == want && force_diag) out[r] = i;
    else if (r >= k) out[r] = -1;
  }
}

__global__ void __launch_bounds__(kSelThreads) topk_select_kernel(
    const float* __restrict__ scores, const int32_t* __restrict__ blk_off, const int64_t* __restrict__ tri_off,
    int nseq, int group, const int32_t* __restrict__ k_seq, int k_max, int force_diag,
    int32_t* __restrict__ idx, int32_t* __restrict__ cnt) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  const int gi = blockIdx.x;
  const int g = blockIdx.y;
  const int nbt = blk_off[nseq];
  const int64_t tri = tri_off[nseq];
  const int s = seq_of_block(blk_off, nseq, gi);
  const int i = gi - blk_off[s];
  const int n = i + 1;
  if (n <= kWarpRow) return;  // short rows: topk_select_warp_kernel
  const int k = max(1, min(min(k_seq[s], n), k_max));  // clamped as in topk_select_warp_kernel
  int32_t* out = idx + (static_cast<size_t>(g) * nbt + gi) * k_max;
  SB_DCHECK(k >= 1 && k <= k_max && gi < nbt);
  if (threadIdx.x == 0) cnt[static_cast<size_t>(g) * nbt + gi] = k;

  const int m = force_diag ? n - 1 : n;   // candidate count
  const int want = force_diag ? k - 1 : k;  // candidates to keep
  if (want >= m) {  // dense row: every block
    for (int r = threadIdx.x; r < k_max; r += kSelThreads) out[r] = r < n ? r : -1;
    return;
  }
  if (want == 0) {  // k = 1 with the forced diagonal: block i only
    for (int r = threadIdx.x; r < k_max; r += kSelThreads) out[r] = r == 0 ? i : -1;
    return;
  }

  __shared__ int hist[256];
  __shared__ int warp_tot[kSelThreads / 32];
  __shared__ int sh_digit, sh_remaining;

  const int64_t row_off = tri_off[s] + static_cast<int64_t>(i) * (i + 1) / 2;
  uint32_t key[kSelPerThread];
#pragma unroll
  for (int r = 0; r < kSelPerThread; ++r) {
    const int j = threadIdx.x + r * kSelThreads;
    float v = -INFINITY;
    if (j < m) {
      const float* base = scores + static_cast<size_t>(g) * group * tri + row_off + j;
      v = __ldg(base);
      for (int q = 1; q < group; ++q) v += __ldg(base + static_cast<size_t>(q) * tri);
    }
    key[r] = j < m ? order_key(v) : 0u;  // padding never selected (want < m real keys)
  }

  // Radix select: find the want-th largest key (prefix) and how many of its ties to keep.
  uint32_t prefix = 0, mask = 0;
  int remaining = want;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int b = threadIdx.x; b < 256; b += kSelThreads) hist[b] = 0;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kSelPerThread; ++r) {
      const int j = threadIdx.x + r * kSelThreads;
      if (j < m && (key[r] & mask) == prefix) atomicAdd(&hist[(key[r] >> shift) & 0xffu], 1);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      // Warp 0 scans the 256 bins from the top: lane l owns bins 255-8l .. 248-8l.
      const int lane = threadIdx.x;
      int local = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) local += hist[255 - 8 * lane - b];
      int incl = local;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const int excl = incl - local;
      // The lane whose range crosses `remaining` resolves the digit.
      if (excl < remaining && incl >= remaining) {
        int run = excl;
        for (int b = 0; b < 8; ++b) {
          const int bin = 255 - 8 * lane - b;
          const int c = hist[bin];
          if (run + c >= remaining) {
            sh_digit = bin;
            sh_remaining = remaining - run;
            break;
          }
          run += c;
        }
      }
    }
    __syncthreads();
    prefix |= static_cast<uint32_t>(sh_digit) << shift;
    mask |= 0xffu << shift;
    remaining = sh_remaining;
    __syncthreads();
  }
  const uint32_t thresh = prefix;  // keys > thresh all kept; `remaining` of the == thresh kept

  // Ordered pass over j: keep key > thresh, or key == thresh among the first `remaining` ties.
  int ties_before = 0, kept_before = 0;
#pragma unroll 1
  for (int r = 0; r < kSelPerThread; ++r) {
    if (r * kSelThreads >= m) break;
    const int j = threadIdx.x + r * kSelThreads;
    const bool valid = j < m;
    const bool tie = valid && key[r] == thresh;
    int tie_total;
    const int tie_rank = ties_before + block_excl_scan(tie, warp_tot, &tie_total);
    const bool keep = valid && (key[r] > thresh || (tie && tie_rank < remaining));
    int keep_total;
    const int pos = kept_before + block_excl_scan(keep, warp_tot, &keep_total);
    if (keep) out[pos] = j;
    ties_before += tie_total;
    kept_before += keep_total;
  }
  // Diagonal block (largest index) goes last; pad.
  for (int r = threadIdx.x; r < k_max; r += kSelThreads) {
    if (r == want && force_diag) out[r] = i;
    else if (r >= k) out[r] = -1;
  }
}

// ---- K4a: sorted softmax masses per row -> workspace, then per-(s, r) fp64 mean ----

// Rows of at most 32 * E blocks: one warp per row, element e of lane l is column e * 32 + l,
// so register e's lane butterfly is the block kernel's warp-e reduction and summing the
// registers in order is its sum over warps -- max, exponentials, z, the normalised values and
// the sorted output are bit-identical to row_sorted_mass_kernel, without its ~30 CTA-wide
// barriers per row (bitonic network in registers: shuffles for strides < 32, register pairs
// above; the compare-exchange keeps the block kernel's predicate, NaNs included).
// One row's softmax masses sorted descending, E values per lane (rows of n <= 32 * E). The sum
// over e adds exact zeros for slots past the row, so z, the masses and the sorted output are
// bit-identical for any E that covers the row.
template <int E>
__device__ __forceinline__ void sorted_mass_row(const float* __restrict__ row, int n, int lane, float* __restrict__ dst) {
  float v[E];
  float mx = -INFINITY;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int j = e * 32 + lane;
    v[e] = j < n ? row[j] : 0.f;
    if (j < n) mx = fmaxf(mx, v[e]);
  }
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float z = 0.f;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int j = e * 32 + lane;
    float t = 0.f;
    if (j < n) {
      v[e] = __expf(v[e] - mx);
      t = v[e];
    }
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    z += t;
  }
  const float inv = 1.0f / z;
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = e * 32 + lane < n ? v[e] * inv : -1.0f;
  // Bitonic sort of 32 * E values, descending (element x = e * 32 + lane).
#pragma unroll
  for (int size = 2; size <= 32 * E; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= 32) {
        const int rs = stride >> 5;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if (e & rs) continue;
          const bool desc = ((e * 32 + lane) & size) == 0;
          const float a = v[e], b = v[e + rs];
          if ((a < b) == desc) {
            v[e] = b;
            v[e + rs] = a;
          }
        }
      } else {
        const bool is_lo = (lane & stride) == 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const float other = __shfl_xor_sync(0xffffffffu, v[e], stride);
          const int x_lo = (e * 32 + lane) & ~stride;
          const bool desc = (x_lo & size) == 0;
          const float a = is_lo ? v[e] : other, b = is_lo ? other : v[e];
          const bool swap = (a < b) == desc;
          v[e] = is_lo ? (swap ? b : a) : (swap ? a : b);
        }
      }
    }
  }
  
#pragma unroll
  for (int e = 0; e < E; ++e)
    if (e * 32 + lane < n) dst[e * 32 + lane] = v[e];
}

template <int E>
__global__ void __launch_bounds__(256) row_sorted_mass_warp_kernel(const float* __restrict__ scores,
                                                                   const int32_t* __restrict__ blk_off,
                                                                   const int64_t* __restrict__ tri_off, int nseq,
                                                                   int nb_total, float* __restrict__ sorted) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  const int gi = blockIdx.x * 8 + (threadIdx.x >> 5), h = blockIdx.y, lane = threadIdx.x & 31;
  if (gi >= nb_total) return;
  const int64_t tri = tri_off[nseq];
  const int s = seq_of_block(blk_off, nseq, gi);
  const int i = gi - blk_off[s];
  const int n = i + 1;
  if (n > 32 * E) return;  // the block kernel's rows
  const size_t off = static_cast<size_t>(h) * tri + tri_off[s] + static_cast<int64_t>(i) * (i + 1) / 2;
  const float* row = scores + off;
  float* dst = sorted + off;
  // The smallest bitonic width that covers this row (C3: most rows are far shorter than the
  // longest, whose width E the host picked).
  if (E >= 8 && n > 128) {
    sorted_mass_row<E>(row, n, lane, dst);
  } else if (E >= 4 && n > 64) {
    sorted_mass_row<(E < 4 ? E : 4)>(row, n, lane, dst);
  } else if (E >= 2 && n > 32) {
    sorted_mass_row<(E < 2 ? E : 2)>(row, n, lane, dst);
  } else {
    sorted_mass_row<1>(row, n, lane, dst);
  }
}

__global__ void row_sorted_mass_kernel(const float* __restrict__ scores, const int32_t* __restrict__ blk_off,
                                       const int64_t* __restrict__ tri_off, int nseq, int pow2, int min_n,
                                       float* __restrict__ sorted) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  extern __shared__ float buf[];
  __shared__ float red[32];
  const int gi = blockIdx.x, h = blockIdx.y;
  const int64_t tri = tri_off[nseq];
  const int s = seq_of_block(blk_off, nseq, gi);
  const int i = gi - blk_off[s];
  const int n = i + 1;
  if (n <= min_n) return;  // the warp kernel's rows
  int p2 = 1;
  while (p2 < n) p2 <<= 1;
  const float* row = scores + static_cast<size_t>(h) * tri + tri_off[s] + static_cast<int64_t>(i) * (i + 1) / 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;

  float mx = -INFINITY;
  for (int j = threadIdx.x; j < n; j += blockDim.x) mx = fmaxf(mx, row[j]);
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = -INFINITY;
  for (int w = 0; w < nw; ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float z = 0.f;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const float e = __expf(row[j] - mx);
    buf[j] = e;
    z += e;
  }
  for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
  if (lane == 0) red[warp] = z;
  __syncthreads();
  z = 0.f;
  for (int w = 0; w < nw; ++w) z += red[w];
  const float inv = 1.0f / z;
  for (int j = threadIdx.x; j < p2; j += blockDim.x) buf[j] = j < n ? buf[j] * inv : -1.0f;
  __syncthreads();
  // Bitonic sort, descending.
  for (int size = 2; size <= p2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < (p2 >> 1); t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool desc = (lo & size) == 0;
        const float a = buf[lo], b = buf[hi];
        if ((a < b) == desc) {
          buf[lo] = b;
          buf[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  float* dst = sorted + static_cast<size_t>(h) * tri + tri_off[s] + static_cast<int64_t>(i) * (i + 1) / 2;
  for (int j = threadIdx.x; j < n; j += blockDim.x) dst[j] = buf[j];
}

// Partial sums per (sequence, rank r, head h) over the rows i >= r of that head, then a fixed
// order sum over heads: deterministic and parallel over (s, r, h).
__global__ void profile_partial_kernel(const float* __restrict__ sorted, const int32_t* __restrict__ blk_off,
                                       const int64_t* __restrict__ tri_off, int nseq, int nb_max,
                                       double* __restrict__ partial) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  const int s = blockIdx.y, h = blockIdx.z;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nb_max) return;
  const int nb = blk_off[s + 1] - blk_off[s];
  const int64_t tri = tri_off[nseq];
  double acc = 0.0;
  const float* base = sorted + static_cast<size_t>(h) * tri + tri_off[s];
  // Same summation order (i ascending); 16 loads in flight per step instead of one per add.
  int i = r;
  for (; i + 16 <= nb; i += 16) {
    float v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = __ldg(base + static_cast<int64_t>(i + u) * (i + u + 1) / 2 + r);
#pragma unroll
    for (int u = 0; u < 16; ++u) acc = __dadd_rn(acc, static_cast<double>(v[u]));
  }
  for (; i < nb; ++i) acc = __dadd_rn(acc, static_cast<double>(base[static_cast<int64_t>(i) * (i + 1) / 2 + r]));
  partial[(static_cast<size_t>(h) * nseq + s) * nb_max + r] = acc;
}

__global__ void profile_reduce_kernel(const double* __restrict__ partial, const int32_t* __restrict__ blk_off,
                                      int nseq, int nb_max, int hs, double* __restrict__ profile) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  const int s = blockIdx.y;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nb_max) return;
  const int nb = blk_off[s + 1] - blk_off[s];
  double acc = 0.0;
  if (r < nb) {
    for (int h = 0; h < hs; ++h) acc = __dadd_rn(acc, partial[(static_cast<size_t>(h) * nseq + s) * nb_max + r]);
    acc = acc / (static_cast<double>(hs) * static_cast<double>(nb));
  }
  profile[static_cast<size_t>(s) * nb_max + r] = acc;
}

__global__ void coverage_at_grid_kernel(const double* __restrict__ profile, const int32_t* __restrict__ blk_off,
                                        int nseq, int nb_max, const int32_t* __restrict__ grid, int ngrid,
                                        double* __restrict__ cov) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nseq * ngrid) return;
  const int s = t / ngrid, g = t % ngrid;
  const int nb = blk_off[s + 1] - blk_off[s];
  const int k = grid[g];
  double c = 0.0;
  if (k >= nb) {
    c = 1.0;  // dense (reference dst.cpp:58-59)
  } else if (k > 0) {
    const double* p = profile + static_cast<size_t>(s) * nb_max;
    for (int r = 0; r < k; ++r) c = __dadd_rn(c, p[r]);  // sequential, like dst.cpp:57
  }
  cov[t] = c;
}

}  // namespace
}  // namespace sbk

SB_API int sb_topk_select(const float* scores, const int32_t* blk_off, const int64_t* tri_off, int nseq,
                          int nb_total, int nb_max, int hs, int group, const int32_t* k_seq, int k_max,
                          int force_diag, int32_t* idx, int32_t* cnt, void* stream) {
  return sbk::abi_call([&] {
    sbk::require(group >= 1 && hs >= 1 && hs % group == 0, "hs must be a positive multiple of group");
    sbk::require(k_max >= 1, "k_max must be >= 1");
    sbk::require(nb_max <= sbk::kMaxRow, "rows longer than 4096 blocks are not supported");
    sbk::require(hs / group <= 65535, "too many selection heads");
    if (nseq == 0 || nb_total == 0) return;
    sbk::require(scores && blk_off && tri_off && k_seq && idx && cnt, "null pointer");
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    dim3 wgrid((nb_total + 7) / 8, hs / group);
    sbk::launch(sbk::topk_select_warp_kernel, wgrid, 256, 0, st, scores, blk_off, tri_off, nseq, nb_total, group, k_seq, k_max,
                                                         force_diag ? 1 : 0, idx, cnt);
    sbk::launched("sb_topk_select");
    if (nb_max > sbk::kWarpRow) {  // rows longer than 256 candidates
      dim3 grid(nb_total, hs / group);
      sbk::launch(sbk::topk_select_kernel, grid, sbk::kSelThreads, 0, st, scores, blk_off, tri_off, nseq, group, k_seq, k_max,
                                                                 force_diag ? 1 : 0, idx, cnt);
      sbk::launched("sb_topk_select");
    }
  });
}

SB_API size_t sb_coverage_profile_workspace_size(int64_t tri_total, int hs, int nseq, int nb_max) {
  const size_t sorted = (static_cast<size_t>(tri_total) * static_cast<size_t>(hs) * sizeof(float) + 255) & ~size_t(255);
  return sorted + static_cast<size_t>(hs) * static_cast<size_t>(nseq) * static_cast<size_t>(nb_max) * sizeof(double);
}

SB_API int sb_coverage_profile(const float* scores, const int32_t* blk_off, const int64_t* tri_off, int nseq,
                               int nb_total, int64_t tri_total_host, int nb_max, int hs, void* workspace,
                               double* profile, void* stream) {
  return sbk::abi_call([&] {
    sbk::require(hs >= 1 && hs <= 65535, "hs must be in [1, 65535]");
    sbk::require(tri_total_host >= 0, "tri_total must be >= 0");
    sbk::require(nb_max <= sbk::kMaxRow, "rows longer than 4096 blocks are not supported");
    if (nseq == 0 || nb_max == 0) return;
    sbk::require(scores && blk_off && tri_off && workspace && profile, "null pointer");
    int p2 = 1;
    while (p2 < nb_max) p2 <<= 1;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    float* sorted = static_cast<float*>(workspace);
    if (nb_total > 0) {
      // Rows of <= 256 blocks: one warp each; longer rows: one CTA each (shared-memory sort).
      const dim3 wgrid((nb_total + 7) / 8, hs);
      if (p2 <= 32) {
        sbk::launch(sbk::row_sorted_mass_warp_kernel<1>, wgrid, 256, 0, st, scores, blk_off, tri_off, nseq, nb_total, sorted);
      } else if (p2 <= 64) {
        sbk::launch(sbk::row_sorted_mass_warp_kernel<2>, wgrid, 256, 0, st, scores, blk_off, tri_off, nseq, nb_total, sorted);
      } else if (p2 <= 128) {
        sbk::launch(sbk::row_sorted_mass_warp_kernel<4>, wgrid, 256, 0, st, scores, blk_off, tri_off, nseq, nb_total, sorted);
      } else {
        sbk::launch(sbk::row_sorted_mass_warp_kernel<8>, wgrid, 256, 0, st, scores, blk_off, tri_off, nseq, nb_total, sorted);
      }
      sbk::launched("sb_coverage_profile/sort");
      if (nb_max > 256) {
        dim3 grid(nb_total, hs);
        sbk::launch(sbk::row_sorted_mass_kernel, grid, 256, p2 * sizeof(float), st, scores, blk_off, tri_off, nseq, p2, 256,
                                                                          sorted);
        sbk::launched("sb_coverage_profile/sort_long");
      }
    }
    const size_t sorted_bytes = (static_cast<size_t>(tri_total_host) * hs * sizeof(float) + 255) & ~size_t(255);
    double* partial = reinterpret_cast<double*>(static_cast<uint8_t*>(workspace) + sorted_bytes);
    dim3 g1((nb_max + 127) / 128, nseq, hs);
    sbk::launch(sbk::profile_partial_kernel, g1, 128, 0, st, sorted, blk_off, tri_off, nseq, nb_max, partial);
    sbk::launched("sb_coverage_profile/partial");
    dim3 g2((nb_max + 127) / 128, nseq);
    sbk::launch(sbk::profile_reduce_kernel, g2, 128, 0, st, partial, blk_off, nseq, nb_max, hs, profile);
    sbk::launched("sb_coverage_profile/reduce");
  });
}

SB_API int sb_coverage_at_grid(const double* profile, const int32_t* blk_off, int nseq, int nb_max,
                               const int32_t* grid, int ngrid, double* coverage, void* stream) {
  return sbk::abi_call([&] {
    sbk::require(ngrid >= 1, "ngrid must be >= 1");
    if (nseq == 0) return;
    sbk::require(profile && blk_off && grid && coverage, "null pointer");
    const int n = nseq * ngrid;
    sbk::launch(sbk::coverage_at_grid_kernel, (n + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream), 
        profile, blk_off, nseq, nb_max, grid, ngrid, coverage);
    sbk::launched("sb_coverage_at_grid");
  });
}
