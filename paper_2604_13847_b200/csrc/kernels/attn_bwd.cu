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
#include "fastmath.cuh"
#include "sb_kernels.h"
#include "sched.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

namespace sbk {
namespace {

using namespace sm100;

constexpr int kM = 128;
constexpr int kStages = 2;
constexpr int kBwdPoly = 2;  // exp2 pairs of every 8 on the FMA pipe (fastmath.cuh ex2_pair_n)
constexpr int kThreads = 352;  // warp 0 TMA, warp 1 UMMA, warps 2..9 two column-split math warpgroups, warp 10 TMA (V)
constexpr float kLog2e = 1.4426950408889634f;

__host__ __device__ constexpr uint32_t pow2_cols(int c) { return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512; }

// prep launch shape: rows per thread group and step (R), resident CTAs per SM, grid in CTAs per
// SM. Measured on C3 (ncu, per layer): R 4 / 4 CTAs 181 us, R 2 / 8 CTAs 167 us, R 1 / 8 CTAs
// (2048 threads per SM, one wave) 158 us.
#ifndef SB_PREP_R
#define SB_PREP_R 1
#endif
#ifndef SB_PREP_MINB
#define SB_PREP_MINB 8
#endif
#ifndef SB_PREP_GRID
#define SB_PREP_GRID 8
#endif
// ------------------------------------------------------------------------------------ prep
// lse2 = LSE * log2(e) and D = rowsum(dO * O) per (token, q head). With ores (the forward's bf16
// rounding residual of O), D = rowsum(dO * (O + O_res)): O to ~2^-16 instead of bf16, which keeps
// dS accurate on rows that attend few keys (there dP - D cancels).
// HBM-bound: O, dO (and O_res) are streamed once in memory order -- the d/8 threads of a
// (token, head) row take one 16-byte chunk each, consecutive rows are consecutive heads of a
// token, so a warp reads 512 contiguous bytes and the grid walks the tensors front to back (the
// earlier head-major walk touched every 8 KB token row once per head). Two rows per thread per
// step keep 4-6 loads in flight; the row's threads finish with xor-shuffles.
// One grid-stride pass over the rows: R rows per thread group and step, all 3R 16-byte loads
// issued before any arithmetic (kRes: the O residual is read and added).
template <bool kRes>
__device__ __forceinline__ void prep_rows(const uint16_t* __restrict__ o, const uint16_t* __restrict__ d_o,
                                          const uint16_t* __restrict__ ores, const float* __restrict__ lse,
                                          int total, int hq, int d, int tp, float* __restrict__ lse2,
                                          float* __restrict__ dvec) {
  constexpr int R = SB_PREP_R;
  const int tpr_log = d == 128 ? 4 : 3;  // log2(threads per row)
  const int sub = threadIdx.x & ((1 << tpr_log) - 1);
  const long long rows = static_cast<long long>(total) * hq;  // row = t * hq + h
  const long long stride = static_cast<long long>(gridDim.x) * (blockDim.x >> tpr_log);
  for (long long r0 = static_cast<long long>(blockIdx.x) * (blockDim.x >> tpr_log) + (threadIdx.x >> tpr_log);
       r0 < rows; r0 += R * stride) {
    uint4 a[R], b[R], c[R];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const long long r = r0 + u * stride;
      const size_t e = static_cast<size_t>(r < rows ? r : r0) * (d >> 3) + sub;
      a[u] = __ldg(reinterpret_cast<const uint4*>(o) + e);
      b[u] = __ldg(reinterpret_cast<const uint4*>(d_o) + e);
      if (kRes) c[u] = __ldg(reinterpret_cast<const uint4*>(ores) + e);
    }
    asm volatile("" ::: "memory");  // keeps every load above the arithmetic (ptxas interleaves otherwise)
    float acc[R];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const uint32_t wa[4] = {a[u].x, a[u].y, a[u].z, a[u].w}, wb[4] = {b[u].x, b[u].y, b[u].z, b[u].w};
      float x = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        x = fmaf(__uint_as_float(wa[e] << 16), __uint_as_float(wb[e] << 16), x);
        x = fmaf(__uint_as_float(wa[e] & 0xffff0000u), __uint_as_float(wb[e] & 0xffff0000u), x);
      }
      if (kRes) {
        const uint32_t wc[4] = {c[u].x, c[u].y, c[u].z, c[u].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          x = fmaf(__uint_as_float(wc[e] << 16), __uint_as_float(wb[e] << 16), x);
          x = fmaf(__uint_as_float(wc[e] & 0xffff0000u), __uint_as_float(wb[e] & 0xffff0000u), x);
        }
      }
      acc[u] = x;
    }
#pragma unroll
    for (int u = 0; u < R; ++u)
      for (int off = (1 << tpr_log) >> 1; off; off >>= 1) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], off);
    if (sub == 0) {
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const long long r = r0 + u * stride;
        if (r >= rows) break;
        const int t = static_cast<int>(r / hq), h = static_cast<int>(r - static_cast<long long>(t) * hq);
        dvec[static_cast<size_t>(h) * tp + t] = acc[u];
        lse2[static_cast<size_t>(h) * tp + t] = lse[static_cast<size_t>(h) * total + t] * kLog2e;
      }
    }
  }
}

__global__ void __launch_bounds__(256, SB_PREP_MINB) bwd_prep_kernel(const uint16_t* __restrict__ o, const uint16_t* __restrict__ d_o,
                                                       const uint16_t* __restrict__ ores,
                                                       const float* __restrict__ lse, int total, int hq, int d, int tp,
                                                       float* __restrict__ lse2, float* __restrict__ dvec) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  if (ores != nullptr)
    prep_rows<true>(o, d_o, ores, lse, total, hq, d, tp, lse2, dvec);
  else
    prep_rows<false>(o, d_o, ores, lse, total, hq, d, tp, lse2, dvec);
  // Padding columns [total, tp): never read for valid rows, but keep them finite.
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e < hq * (tp - total); e += blockDim.x) {
      const int h = e / (tp - total), t = total + e % (tp - total);
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
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
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
    SB_DCHECK(!pass || !hit || found + __popc(m & ((1u << lane) - 1u)) < tr_off[w + 1] - tr_off[w]);
    if (pass && hit) dst[found + __popc(m & ((1u << lane) - 1u))] = key;
    found += __popc(m);
  }
  if (!pass && lane == 0) tr_cnt[w] = found;
}

// Exclusive scan of n ints, out[n] = total (single CTA of 1024 threads). Thread t owns the
// contiguous segment [t * per, (t + 1) * per): it sums its segment with independent loads, one
// block-wide scan of the 1024 sums follows, then it writes its segment's prefixes. One pass
// instead of n / 1024 dependent tile rounds (10 rounds at C3: 11 -> ~4 us).
__global__ void __launch_bounds__(1024) scan_kernel(const int32_t* __restrict__ in, int n, int32_t* __restrict__ out) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  __shared__ int warp_sum[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int per = (n + 1023) / 1024;
  const int i0 = min(n, threadIdx.x * per), i1 = min(n, i0 + per);
  int v = 0;
  for (int i = i0; i < i1; ++i) v += __ldg(in + i);
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_sum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int w0 = warp_sum[lane];
    int wi = w0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    warp_sum[lane] = wi - w0;
  }
  __syncthreads();
  int run = warp_sum[warp] + incl - v;
  for (int i = i0; i < i1; ++i) {
    out[i] = run;
    run += __ldg(in + i);
  }
  if (threadIdx.x == 1023) out[n] = run;
}

// P^T for one key row (this thread) over this warpgroup's NC query columns col0 .. col0+NC:
// p[r] = 2^(S'^T * scale_log2). The UMMA already subtracted lse2[col] / scale_log2 from S^T
// through the augmented K step (see DkvCfg), so no per-column operand is read here; kMasked
// zeroes columns outside [r_lo, nq) (causal diagonal / sequence end).
template <int NC, bool kMasked>
__device__ __forceinline__ void dkv_p(const uint32_t (&sv)[NC / 32][32], float scale_log2, int col0, int r_lo, int nq,
                                      float (&p)[NC]) {
  const f2 sc = mk2(scale_log2, scale_log2);
#pragma unroll
  for (int pe = 0; pe < NC / 2; ++pe) {
    const int r = 2 * pe;
    f2 e = ex2_pair_n<kBwdPoly>(fmul2(mk2(__uint_as_float(sv[r / 32][r % 32]), __uint_as_float(sv[r / 32][r % 32 + 1])), sc), pe);
    if (kMasked) {
      e.x = (col0 + r < nq && col0 + r >= r_lo) ? e.x : 0.f;
      e.y = (col0 + r + 1 < nq && col0 + r + 1 >= r_lo) ? e.y : 0.f;
    }
    p[r] = e.x;
    p[r + 1] = e.y;
  }
}

// P for one query row over NC key columns col0 .. col0+NC: p[c] = 2^(S * scale_log2 - lse2)
// (row constant); kMasked zeroes columns >= lim.
template <int NC, bool kMasked>
__device__ __forceinline__ void dq_p(const uint32_t (&sv)[NC / 32][32], float neg_l2, float scale_log2, int col0,
                                     int lim, float (&p)[NC]) {
  const f2 sc = mk2(scale_log2, scale_log2), nl = mk2(neg_l2, neg_l2);
#pragma unroll
  for (int pe = 0; pe < NC / 2; ++pe) {
    const int c = 2 * pe;
    f2 e = ex2_pair_n<kBwdPoly>(ffma2(mk2(__uint_as_float(sv[c / 32][c % 32]), __uint_as_float(sv[c / 32][c % 32 + 1])), sc, nl),
                    pe);
    if (kMasked) {
      e.x = col0 + c < lim ? e.x : 0.f;
      e.y = col0 + c + 1 < lim ? e.y : 0.f;
    }
    p[c] = e.x;
    p[c + 1] = e.y;
  }
}

// TMEM column of the packed-bf16 A operand for UMMA K-step kk when each column half h of the
// B-wide score tile stores its packed values at the start of its own half (h * B / 2).
template <int B>
__device__ __forceinline__ uint32_t packed_col(int kk) {
  return static_cast<uint32_t>((kk / (B / 32)) * (B / 2) + (kk % (B / 32)) * 8);
}

// ------------------------------------------------------------------------------------ dkv
// Persistent: one CTA per SM walks key-block items (hk, gj) longest-first. Per item the CTA
// holds K / V (128 key rows) and streams every (q head, q block) that selected the block
// through a 2-stage Q / dO ring. TMEM: S^T | dP^T | dV | dK (512 columns for D = B = 128).
template <int D, int B>
struct DkvCfg {
  static constexpr int kChunks = D / 64;
  static constexpr int kTileBytes = kChunks * kM * 128;  // K or V (128 key rows)
  static constexpr int kQBytes = kChunks * B * 128;      // Q_i or dO_i (B query rows)
  // Augmented K step (one extra UMMA K = 16 slice, SWIZZLE_NONE K-major: core matrix (8 rows x
  // 16 B) (rg, kc) at rg * 256 + kc * 128). The key side holds (1, 1, 1, 0 ...) per key row, the
  // query side the three-term bf16 split of -lse2 / scale_log2 (for S^T) or -D (for dP^T) per
  // query row, so the UMMA produces S^T - lse2 / scale_log2 and dP^T - D directly and the
  // math warps read no per-column vectors from shared memory (whose crossbar the SS UMMA
  // operand reads saturate).
  static constexpr int kAugOnesBytes = kM * 32;
  static constexpr int kAugBytes = B * 32;
  static constexpr int kSmemTiles = 2 * kTileBytes + kStages * (2 * kQBytes) + kAugOnesBytes + kStages * 2 * kAugBytes;
  static constexpr int kSt = 0, kDPt = B, kDV = 2 * B, kDK = 2 * B + D;
  static constexpr uint32_t kCols = pow2_cols(2 * B + 2 * D);
  static constexpr int kSmemBytes = kSmemTiles + 1024 + 512;  // + alignment slack + DkvBars
};

__device__ __forceinline__ uint64_t desc_aug(uint32_t saddr) {  // SWIZZLE_NONE, LBO 128, SBO 256
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(128u >> 4) << 16;
  d |= static_cast<uint64_t>(256u >> 4) << 32;
  d |= 1ull << 46;
  return d;
}

// Byte offset of (row, k = 0) in an augmented slice; k = 0..3 are the 8 bytes from there.
__device__ __forceinline__ int aug_off(int row) { return (row >> 3) * 256 + (row & 7) * 16; }

// x -> three bf16 terms whose fp32 sum reproduces x to ~2^-24 relative, packed with a zero.
__device__ __forceinline__ uint2 split3_bf16(float x) {
  const __nv_bfloat16 h = __float2bfloat16_rn(x);
  const float r1 = x - __bfloat162float(h);
  const __nv_bfloat16 m = __float2bfloat16_rn(r1);
  const __nv_bfloat16 l = __float2bfloat16_rn(r1 - __bfloat162float(m));
  uint2 u;
  u.x = static_cast<uint32_t>(__bfloat16_as_ushort(h)) | (static_cast<uint32_t>(__bfloat16_as_ushort(m)) << 16);
  u.y = static_cast<uint32_t>(__bfloat16_as_ushort(l));
  return u;
}

// dK/dV work is claimed dynamically: round 0 of CTA c is entry c, every later round takes the next
// entry of the (head-major, longest-first) split order from a global cursor. The producer warp
// claims a round when it needs it and publishes the position through a small ring; the issuer,
// math and store roles read it in the same round order. A static snake assignment left the CTAs'
// loads 1.27x apart under C3's mix of single-pair and split heavy items (measured busy max / mean
// 1.25, per-CTA busy tracking a pair + item cost model with r = 0.995). Results do not depend on
// which CTA runs an entry.
constexpr int kSchedRing = 8;
constexpr int kSchedReaders = 10;  // warp leaders that read a slot: issuer, 8 math warps, store warp

struct DkvBars {
  uint64_t kv_full, kv_empty;
  uint64_t q_full[kStages], q_empty[kStages];    // Q_i (+ its augmented slice) ring
  uint64_t do_full[kStages], do_empty[kStages];  // dO_i (+ its augmented slice) ring
  uint64_t st_full, dpt_full;  // UMMA -> math: S^T / dP^T in TMEM
  uint64_t st_free;            // math -> UMMA: S^T read into registers (the next S^T may overwrite)
  uint64_t pds_part[2];        // math -> UMMA: P^T and dS^T (bf16) of 32-column chunk c2 packed over dP^T
  uint64_t acc_done;           // UMMA -> epilogue: the item's dV / dK are final
  uint64_t epi_free[kStages];  // epilogue -> producer: the item's dV / dK store read ring stage st
  uint64_t epi_staged[kStages];  // math -> store warp: the item's dV / dK are staged in ring stage st
  uint64_t sched_full[kSchedRing], sched_empty[kSchedRing];  // producer <-> roles: schedule ring
  int32_t sched_pos[kSchedRing];  // split-order position of round k in slot k % kSchedRing (-1: end)
  uint32_t tmem_base;
};
static_assert(sizeof(DkvBars) <= 512, "DkvBars fits the reserved tail of the dK/dV shared memory");

// TMEM column (relative to dP^T) of the packed-bf16 P^T (dS^T: + 16) for UMMA K step kk.
// Warpgroup hf owns query columns [hf * B/2, (hf + 1) * B/2) of dP^T; it writes chunk c2 (32
// query columns) as P^T packed into columns c2 * 32 + [0, 16) and dS^T into c2 * 32 + [16, 32)
// of its own range, i.e. over dP^T values it has already read.
template <int B>
__device__ __forceinline__ uint32_t pds_col(int kk) {
  constexpr int kPerWg = B / 32;  // K steps (16 query columns) per warpgroup
  const int hf = kk / kPerWg, r = kk % kPerWg;
  return static_cast<uint32_t>(hf * (B / 2) + (r >> 1) * 32 + (r & 1) * 8);
}

struct KvItem {
  int hk, gj, jl, seq0, seq_len, e0, ne;
};

// Split of long dK/dV items (dkv_split_kernel): an order entry is item | chunk << 22 | nchunks << 27.
// A key block listed by (almost) every later q block -- column-concentrated routing, e.g. a
// sink block, times the GQA group -- is one item up to ~4x a CTA's fair share of pairs; the
// LPT snake cannot balance that (C4 planted: makespan 1.52x the mean). Such items are cut into
// nchunks pair ranges whose fp32 dK / dV partials a second kernel sums in chunk order.
constexpr int kSplitItemBits = 22;  // item | chunk << 22 | nchunks << 26 (4 bits each: entries stay >= 0)
constexpr int kSplitMaxChunks = 15;
#ifndef SB_DKV_SPLIT_PER_CTA
#define SB_DKV_SPLIT_PER_CTA 4
#endif
constexpr int kSplitPerCta = SB_DKV_SPLIT_PER_CTA;  // cap = total pairs / (kSplitPerCta * grid)
constexpr int kSplitMinPairs = 16;
__host__ __device__ constexpr int split_slots(int grid) { return 2 * kSplitPerCta * grid; }

// One 32-byte record per split-order entry (dkv_records_kernel): the dK/dV roles read a chunk
// with two independent 16-byte loads instead of decoding it through a chain of dependent loads
// (order -> blk_off binary search -> cu / tr_off), which put ~2.5k cycles on every item
// boundary of every role.
struct alignas(16) KvRec {
  int e, hk, gj, jl, seq0, seq_len, e0, ne;
};

struct KvChunk {
  KvItem w;
  int it, c, nc, m0, items;  // item, chunk c of nc, its pair range [m0, m0 + items)
};

// dkv decodes items in place (order -> blk_off -> cu / tr_off): measured 5% faster than the
// prefetched ItemRec path the fwd / dq kernels use (2.01 vs 1.91 ms on C2).
__device__ __forceinline__ KvItem decode_kv(int it, const int32_t* cu, const int32_t* blk_off, int nseq, int nbt,
                                            const int32_t* tr_off) {
  KvItem w;
  w.hk = it / nbt;
  w.gj = it - w.hk * nbt;
  const int s = seq_of_block(blk_off, nseq, w.gj);
  w.jl = w.gj - blk_off[s];
  w.seq0 = cu[s];
  w.seq_len = cu[s + 1] - w.seq0;
  w.e0 = tr_off[it];
  w.ne = tr_off[it + 1] - w.e0;
  return w;
}

template <int D, int B>
__global__ void __launch_bounds__(kThreads, 1) attn_bwd_dkv_kernel(
    const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
    const __grid_constant__ CUtensorMap tm_dk, const __grid_constant__ CUtensorMap tm_dv,
    const int32_t* __restrict__ cu, const int32_t* __restrict__ blk_off, int nseq, int hq, int hkv, int hsel,
    const int32_t* __restrict__ tr_off, const int32_t* __restrict__ tr_ent, const float* __restrict__ lse2,
    const float* __restrict__ dvec, int tp, float scale, float scale_log2, uint16_t* __restrict__ dk,
    uint16_t* __restrict__ dv, const KvRec* __restrict__ recs, int32_t* __restrict__ sched_counts,
    const int32_t* __restrict__ slot_base, float* __restrict__ partials, unsigned long long* trace) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  using C = DkvCfg<D, B>;
  const int n_items = sched_counts[0];  // entries of the split order (dkv_split_kernel); [2] is the cursor
  // Debug: per-CTA start / end (globaltimer ns) at trace[8192 + 2 * cta + {0, 1}].
  if (trace != nullptr && threadIdx.x == 0) trace[8192 + 2 * blockIdx.x] = globaltimer_ns();
  // D = B = 128: an item's dV / dK (32 KB each) are stored by TMA through the Q / dO slots of
  // the ring stage its last pair used, free once acc_done fires (see the epilogue).
  constexpr bool kStagedEpi = D == 128 && B == 128;
  auto tr = [&](int slot, int g) {
    if (trace != nullptr && blockIdx.x == 0 && g < 256 && (threadIdx.x & 31) == 0) trace[g * 16 + slot] = clock64();
  };
  // Per-item boundary stamps (items t < 64): 0 K/V TMA issued, 1 issuer starts waiting for
  // kv_full, 2 kv_full seen, 3 math sees acc_done, 4 math epilogue done.
  auto tri = [&](int slot, int t) {
    if (trace != nullptr && blockIdx.x == 0 && t < 64 && (threadIdx.x & 31) == 0) trace[4096 + t * 8 + slot] = clock64();
  };
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* k_smem = smem;
  uint8_t* v_smem = smem + C::kTileBytes;
  uint8_t* q_smem = smem + 2 * C::kTileBytes;            // [stage]
  uint8_t* do_smem = q_smem + kStages * C::kQBytes;      // [stage]
  uint8_t* ones_smem = do_smem + kStages * C::kQBytes;                  // augmented key side
  uint8_t* qaug_smem = ones_smem + C::kAugOnesBytes;                    // [stage] -lse2 / scale_log2
  uint8_t* daug_smem = qaug_smem + kStages * C::kAugBytes;              // [stage] -D
  DkvBars* bars = reinterpret_cast<DkvBars*>(smem + C::kSmemTiles);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nbt = blk_off[nseq];
  const int grid = gridDim.x, cta = blockIdx.x;
  const int sg = hq / hsel;  // q heads per selection row
  const float inv_scale_log2 = 1.0f / scale_log2;

  if (threadIdx.x == 0) {
    mbar_init(&bars->kv_full, 1);
    mbar_init(&bars->kv_empty, 1);
    for (int st = 0; st < kStages; ++st) {
      mbar_init(&bars->q_full[st], 2);  // TMA expect_tx arrive + augmented-slice arrive
      mbar_init(&bars->q_empty[st], 1);
      mbar_init(&bars->do_full[st], 2);
      mbar_init(&bars->do_empty[st], 1);
    }
    mbar_init(&bars->st_full, 1);
    mbar_init(&bars->dpt_full, 1);
    mbar_init(&bars->st_free, 256);
    mbar_init(&bars->pds_part[0], 256);
    mbar_init(&bars->pds_part[1], 256);
    mbar_init(&bars->acc_done, 1);
    for (int st = 0; st < kStages; ++st) {
      mbar_init(&bars->epi_free[st], 1);
      mbar_init(&bars->epi_staged[st], 256);
    }
    for (int r = 0; r < kSchedRing; ++r) {
      mbar_init(&bars->sched_full[r], 1);
      mbar_init(&bars->sched_empty[r], kStagedEpi ? kSchedReaders : kSchedReaders - 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kCols>(&bars->tmem_base);
  {
    // Augmented slices: zero everything, then (1, 1, 1) in k = 0..2 of every key row.
    uint4* z = reinterpret_cast<uint4*>(ones_smem);
    for (int i = threadIdx.x; i < (C::kAugOnesBytes + kStages * 2 * C::kAugBytes) / 16; i += blockDim.x)
      z[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    for (int r = threadIdx.x; r < kM; r += blockDim.x)
      *reinterpret_cast<uint2*>(ones_smem + aug_off(r)) = make_uint2(0x3F803F80u, 0x00003F80u);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  // Split-order position of round k. The producer warp (whole warp, in round order) claims it
  // and publishes it in ring slot k % kSchedRing; every other role (whole warp, in round order)
  // reads it there and releases the slot.
  auto round_pos = [&](int k) {
    const int slot = k % kSchedRing;
    const uint32_t ph = (k / kSchedRing) & 1;
    int pos;
    if (warp == 0) {
      if (lane == 0) {
        if (k >= kSchedRing) mbar_wait(&bars->sched_empty[slot], ph ^ 1);
        pos = k == 0 ? cta : grid + atomicAdd(sched_counts + 2, 1);
        if (pos >= n_items) pos = -1;
        bars->sched_pos[slot] = pos;
        mbar_arrive(&bars->sched_full[slot]);  // release: the position is visible to the waiters
      }
      pos = __shfl_sync(0xffffffffu, pos, 0);
    } else {
      mbar_wait(&bars->sched_full[slot], ph);
      pos = *reinterpret_cast<volatile int32_t*>(&bars->sched_pos[slot]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->sched_empty[slot]);
    }
    return pos;
  };
  // Chunk of schedule round k of this CTA (false past the end). Each role calls it once per
  // round, in round order, until it returns false.
  auto next_chunk = [&](int k, KvChunk& ch) {
    const int pos = round_pos(k);
    if (pos < 0) return false;
    const int4 r0 = __ldg(reinterpret_cast<const int4*>(recs + pos));
    const int4 r1 = __ldg(reinterpret_cast<const int4*>(recs + pos) + 1);
    const int e = r0.x;
    ch.it = e & ((1 << kSplitItemBits) - 1);
    ch.c = (e >> kSplitItemBits) & 15;
    ch.nc = e >> (kSplitItemBits + 4);
    ch.w.hk = r0.y;
    ch.w.gj = r0.z;
    ch.w.jl = r0.w;
    ch.w.seq0 = r1.x;
    ch.w.seq_len = r1.y;
    ch.w.e0 = r1.z;
    ch.w.ne = r1.w;
    const int P = ch.w.ne * sg;
    ch.m0 = ch.c * P / ch.nc;
    ch.items = (ch.c + 1) * P / ch.nc - ch.m0;
    return true;
  };

  // (q head, q block) of the m-th pair of an item. Pairs are q-head major (GQA: the sg q heads of
  // the selected entries are walked one head at a time): 0.3-1 % faster than entry-major at C5
  // GQA, DRAM reads unchanged (profiles/r2/gqa_ab.md).
  auto pair_of = [&](const KvItem& w, int m, int& h, int& gi) {
    const int hh = m / w.ne;
    const int ent = __ldg(tr_ent + w.e0 + (m - hh * w.ne));
    const int hs = ent / nbt;
    gi = ent - hs * nbt;
    h = hs * sg + hh;
  };

  if (warp == 0) {
    // ------------------------------------------------------------ producer (whole warp)
    if (lane == 0) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
      tma_prefetch(&tm_do);
    }
    int g = 0, t = 0;  // global pair counter, item counter
    uint32_t epi_need = 0;            // bit st: an item epilogue is staging through ring stage st
    int epi_uses0 = 0, epi_uses1 = 0;  // epilogues assigned to stage 0 / 1 so far
    // Q / dO (+ augmented slices) of pair m of chunk ch into ring stage g % kStages.
    auto load_pair = [&](const KvChunk& ch, int m, int g) {
      const KvItem& w = ch.w;
      const int st = g % kStages;
      const uint32_t ph = (g / kStages) & 1;
      int h, gi;
      pair_of(w, ch.m0 + m, h, gi);
      const int q0 = w.seq0 + (gi - (w.gj - w.jl)) * B;  // gj - jl: the sequence's first block
      const int nq = min(B, w.seq_len - (gi - (w.gj - w.jl)) * B);
      // lse2 / D of the pair's query rows: all loads in flight before the ring-slot wait.
      float nl[B / 32], nd[B / 32];
#pragma unroll
      for (int e = 0; e < B / 32; ++e) {
        const int r = e * 32 + lane;
        const bool ok = r < nq;
        nl[e] = ok ? __ldg(lse2 + static_cast<size_t>(h) * tp + q0 + r) : 0.f;
        nd[e] = ok ? __ldg(dvec + static_cast<size_t>(h) * tp + q0 + r) : 0.f;
      }
      // Q and dO are separate rings: the UMMA releases Q_i after dK_i and dO_i after dV_i.
      if (lane == 0) tr(11, g);
      if (kStagedEpi && ((epi_need >> st) & 1u)) {  // an item's dV / dK store reads this stage
        mbar_wait(&bars->epi_free[st], ((st ? epi_uses1 : epi_uses0) - 1) & 1);
        epi_need &= ~(1u << st);
      }
      mbar_wait(&bars->q_empty[st], ph ^ 1);
      if (lane == 0) tr(12, g);
      if (lane == 0) {
        mbar_expect_tx(&bars->q_full[st], C::kQBytes);
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d(q_smem + st * C::kQBytes + c * B * 128, &tm_q, &bars->q_full[st], c * 64, h, q0);
      }
      uint8_t* qa = qaug_smem + st * C::kAugBytes;
#pragma unroll
      for (int e = 0; e < B / 32; ++e)
        *reinterpret_cast<uint2*>(qa + aug_off(e * 32 + lane)) = split3_bf16(-nl[e] * inv_scale_log2);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> UMMA operand reads
      __syncwarp();
      if (lane == 0) tr(13, g);
      if (lane == 0) mbar_arrive(&bars->q_full[st]);
      mbar_wait(&bars->do_empty[st], ph ^ 1);
      if (lane == 0) {
        mbar_expect_tx(&bars->do_full[st], C::kQBytes);
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d(do_smem + st * C::kQBytes + c * B * 128, &tm_do, &bars->do_full[st], c * 64, h, q0);
      }
      uint8_t* da = daug_smem + st * C::kAugBytes;
#pragma unroll
      for (int e = 0; e < B / 32; ++e)
        *reinterpret_cast<uint2*>(da + aug_off(e * 32 + lane)) = split3_bf16(-nd[e]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->do_full[st]);
    };
    // Non-empty chunks in schedule order from round k on (false past the end).
    auto next_nonempty = [&](int& k, KvChunk& out) {
      for (;; ++k)
        if (!next_chunk(k, out)) return false;
        else if (out.items > 0) return true;
    };
    // Per item: the first pair's Q / dO go first (they need a ring stage, not the K / V buffer),
    // then K / V once the previous item's last S^T / dP^T are done (kv_empty), then the next
    // item is decoded (its chain of dependent loads overlaps the tiles in flight) and its K / V
    // prefetched to L2, then the remaining pairs. Each chunk is decoded once. Single-pair items
    // (most of C3's under column-concentrated routing) were paced by this warp: decode, an
    // extra look-ahead decode and K / V before Q put ~8-9k cycles on every item.
    int kc = 0;
    KvChunk cur;
    bool have = next_nonempty(kc, cur);
    while (have) {
      const KvItem& w = cur.w;
      const int items = cur.items;
      const int kv0 = w.seq0 + w.jl * B;
      load_pair(cur, 0, g);
      if (lane == 0) {
        mbar_wait(&bars->kv_empty, (t & 1) ^ 1);
        mbar_expect_tx(&bars->kv_full, 2 * C::kTileBytes);
        for (int c = 0; c < C::kChunks; ++c) {
          tma_load_3d(k_smem + c * kM * 128, &tm_k, &bars->kv_full, c * 64, w.hk, kv0);
          tma_load_3d(v_smem + c * kM * 128, &tm_v, &bars->kv_full, c * 64, w.hk, kv0);
        }
        tri(0, t);
        if (trace != nullptr && blockIdx.x == 0 && t < 64) trace[4096 + t * 8 + 5] = static_cast<unsigned long long>(items);
      }
      __syncwarp();
      int kn = kc + 1;
      KvChunk nxt;
      const bool have_n = next_nonempty(kn, nxt);
      if (lane == 0 && have_n) {
        const int kv2 = nxt.w.seq0 + nxt.w.jl * B;
        for (int c = 0; c < C::kChunks; ++c) {
          tma_prefetch_l2_3d(&tm_k, c * 64, nxt.w.hk, kv2);
          tma_prefetch_l2_3d(&tm_v, c * 64, nxt.w.hk, kv2);
        }
      }
      for (int m = 1; m < items; ++m) load_pair(cur, m, g + m);
      g += items;
      if (kStagedEpi) {  // the item's epilogue stages through its last pair's ring stage
        const int sl = (g - 1) % kStages;
        if (sl) {
          ++epi_uses1;
        } else {
          ++epi_uses0;
        }
        epi_need |= 1u << sl;
      }
      ++t;
      cur = nxt;
      kc = kn;
      have = have_n;
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ UMMA issuer
    // Flat pair stream g over all items. S^T_{g+1} is issued as soon as the math warps have
    // read S^T_g (st_free), so it runs while they compute P_g / dS_g; P^T_g and dS^T_g come back
    // packed over dP^T_g's columns:
    //   St_g, dPt_g | [st_free_g] St_{g+1} | [pds_g] dV_g, dK_g, dPt_{g+1} | [st_free_{g+1}] ...
    // The pipe then only waits on the short dS tail of the math, never on P.
    {  // whole warp, converged; `leader` issues
      const uint32_t leader = elect_one();
      constexpr uint32_t idesc_t = idesc_bf16_f32(kM, B, false, false);
      constexpr uint32_t idesc_acc = idesc_bf16_f32(kM, D, false, true);
      const uint32_t k_addr = smem_u32(k_smem), v_addr = smem_u32(v_smem);
      auto qa = [&](int gg) { return smem_u32(q_smem + (gg % kStages) * C::kQBytes); };
      auto da = [&](int gg) { return smem_u32(do_smem + (gg % kStages) * C::kQBytes); };
      const uint32_t ones_addr = smem_u32(ones_smem);
      auto qaug = [&](int gg) { return smem_u32(qaug_smem + (gg % kStages) * C::kAugBytes); };
      auto daug = [&](int gg) { return smem_u32(daug_smem + (gg % kStages) * C::kAugBytes); };
      auto issue_st = [&](int gg) {
        if (gg > 0) mbar_wait(&bars->st_free, (gg - 1) & 1);  // S^T_{gg-1} read out of TMEM
        tr(8, gg);
        mbar_wait(&bars->q_full[gg % kStages], (gg / kStages) & 1);
        tr(9, gg);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off_m = (kk >> 2) * (kM * 128) + (kk & 3) * 32;
          const uint32_t off_n = (kk >> 2) * (B * 128) + (kk & 3) * 32;
          mma_ss(tmem + C::kSt, desc_sw128(k_addr + off_m, 16, 1024), desc_sw128(qa(gg) + off_n, 16, 1024), idesc_t,
                 kk > 0, leader);
        }
        mma_ss(tmem + C::kSt, desc_aug(ones_addr), desc_aug(qaug(gg)), idesc_t, 1u, leader);  // - lse2 / scale_log2
        tc_commit(&bars->st_full, leader);
      };
      auto issue_dpt = [&](int gg) {
        mbar_wait(&bars->do_full[gg % kStages], (gg / kStages) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off_m = (kk >> 2) * (kM * 128) + (kk & 3) * 32;
          const uint32_t off_n = (kk >> 2) * (B * 128) + (kk & 3) * 32;
          mma_ss(tmem + C::kDPt, desc_sw128(v_addr + off_m, 16, 1024), desc_sw128(da(gg) + off_n, 16, 1024), idesc_t,
                 kk > 0, leader);
        }
        mma_ss(tmem + C::kDPt, desc_aug(ones_addr), desc_aug(daug(gg)), idesc_t, 1u, leader);  // - D
        tc_commit(&bars->dpt_full, leader);
      };
      int g = 0, t = 0;
      for (int k = 0;; ++k) {
        KvChunk ch;
        if (!next_chunk(k, ch)) break;
        const int items = ch.items;
        if (items == 0) continue;
        tri(1, t);
        mbar_wait(&bars->kv_full, t & 1);
        tri(2, t);
        issue_st(g);
        issue_dpt(g);
        if (items == 1) tc_commit(&bars->kv_empty, leader);  // last S^T / dP^T of the item issued
        for (int m = 0; m < items; ++m, ++g) {
          if (m + 1 < items) issue_st(g + 1);
          tr(0, g);
          // dK first (Q_i is the ring the next S^T waits on), in two K halves: the K steps of
          // chunk c2 go as soon as both warpgroups packed that chunk's P^T / dS^T.
#pragma unroll
          for (int c2 = 0; c2 < B / 64; ++c2) {
            mbar_wait(&bars->pds_part[c2], g & 1);
            if (c2 == 0) tr(1, g);
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < B / 16; ++kk) {
              if (((kk % (B / 32)) >> 1) != c2) continue;
              mma_ts(tmem + C::kDK, tmem + C::kDPt + pds_col<B>(kk) + 16,
                     desc_sw128(qa(g) + kk * 2048, B * 128, 1024), idesc_acc, (m > 0 || c2 > 0 || kk > 0) ? 1u : 0u,
                     leader);
            }
          }
          tc_commit(&bars->q_empty[g % kStages], leader);
#pragma unroll
          for (int kk = 0; kk < B / 16; ++kk)
            mma_ts(tmem + C::kDV, tmem + C::kDPt + pds_col<B>(kk), desc_sw128(da(g) + kk * 2048, B * 128, 1024),
                   idesc_acc, (m > 0 || kk > 0) ? 1u : 0u, leader);
          tc_commit(&bars->do_empty[g % kStages], leader);
          tr(10, g);
          if (m + 1 < items) {
            issue_dpt(g + 1);
            if (m + 2 == items) tc_commit(&bars->kv_empty, leader);  // K (last S^T) and V (last dP^T) no longer read
          }
        }
        tc_commit(&bars->acc_done, leader);
        ++t;
      }
    }
  } else if (warp < 10) {
    // ------------------------------------------------------------ softmax-gradient + epilogue
    // Two warpgroups split every key row's B query columns (and the D output columns of the
    // epilogue) in halves; the math is column-independent, so they never synchronise.
    constexpr int HB = B / 2;
    const int quarter = warp & 3;
    const int hf = (warp - 2) >> 2;
    const int c = quarter * 32 + lane;  // key row
    const uint32_t lf = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t st_col = C::kSt + hf * HB, dpt_col = C::kDPt + hf * HB;
    int g = 0, t = 0;
    for (int k = 0;; ++k) {
      KvChunk ch;
      if (!next_chunk(k, ch)) break;
      const KvItem& w = ch.w;
      const int items = ch.items;
      const int kv0 = w.seq0 + w.jl * B;
      const int nkv = min(B, w.seq_len - w.jl * B);
      // Pair entries are loaded one pair ahead so their global-load latency is not exposed
      // after the st_full wait when S^T is already there.
      int ent_nx = __ldg(tr_ent + w.e0 + (w.ne > 0 ? ch.m0 % w.ne : 0));
      const int blk0 = w.gj - w.jl;
      for (int m = 0; m < items; ++m, ++g) {
        const int st = g % kStages;
        const int ent = ent_nx;
        if (m + 1 < items) ent_nx = __ldg(tr_ent + w.e0 + (ch.m0 + m + 1) % w.ne);
        const int gi = ent - (ent / nbt) * nbt;
        const int il = gi - blk0;
        const int nq = min(B, w.seq_len - il * B);
        // Valid query columns r: inside the sequence, and causal (key row c <= r) on the diagonal.
        const int r_lo = il == w.jl ? c : 0;
        mbar_wait(&bars->st_full, g & 1);
        if (threadIdx.x == 64) tr(4, g);
        tc_fence_after();
        float p[HB];
        {
          uint32_t sv[HB / 32][32];
#pragma unroll
          for (int c2 = 0; c2 < HB / 32; ++c2) tmem_ld32(tmem + lf + st_col + c2 * 32, sv[c2]);
          tmem_wait_ld();
          tc_fence_before();
          mbar_arrive(&bars->st_free);  // S^T_g is in registers: S^T_{g+1} may overwrite it
          if (r_lo <= hf * HB && nq == B) {
            dkv_p<HB, false>(sv, scale_log2, hf * HB, 0, B, p);
          } else {
            dkv_p<HB, true>(sv, scale_log2, hf * HB, r_lo, nq, p);
          }
        }
        if (threadIdx.x == 64) tr(5, g);
        mbar_wait(&bars->dpt_full, g & 1);
        if (threadIdx.x == 64) tr(6, g);
        tc_fence_after();
        {
          // dP^T chunks software-pipelined: chunk c2+1 is in flight while c2 is processed; P^T and
          // dS^T of chunk c2 are packed over chunk c2's own (already read) columns.
          uint32_t pv[2][32];
          tmem_ld32(tmem + lf + dpt_col, pv[0]);
          tmem_wait_ld();
#pragma unroll
          for (int c2 = 0; c2 < HB / 32; ++c2) {
            if (c2 + 1 < HB / 32) tmem_ld32(tmem + lf + dpt_col + (c2 + 1) * 32, pv[(c2 + 1) & 1]);
            uint32_t pw[16], dd[16];
#pragma unroll
            for (int e = 0; e < 32; e += 2) {  // dS^T = P^T (dP^T - D): the UMMA already subtracted D
              const int r = c2 * 32 + e;
              pw[e / 2] = pack_bf16x2(p[r], p[r + 1]);
              const f2 ds = fmul2(mk2(p[r], p[r + 1]),
                                  mk2(__uint_as_float(pv[c2 & 1][e]), __uint_as_float(pv[c2 & 1][e + 1])));
              dd[e / 2] = pack_bf16x2(ds.x, ds.y);
            }
            tmem_st16(tmem + lf + dpt_col + c2 * 32, pw);
            tmem_st16(tmem + lf + dpt_col + c2 * 32 + 16, dd);
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&bars->pds_part[c2]);
            if (c2 + 1 < HB / 32) tmem_wait_ld();
          }
        }
        if (threadIdx.x == 64) tr(7, g);
      }
      if (items > 0) {
        mbar_wait(&bars->acc_done, t & 1);
        if (threadIdx.x == 64) tri(3, t);
        tc_fence_after();
        ++t;
      }
      // Epilogue: dV and dK * scale for the valid key rows (zeros if nobody selected the block);
      // warpgroup hf writes output columns [hf * D/2, (hf + 1) * D/2).
      const bool store = c < nkv;
      if (ch.nc > 1) {
        // Split item: this chunk's fp32 dV / dK partials -> slot; dkv_split_reduce_kernel sums
        // the chunks in order (scale applied there) and writes the valid rows.
        if (kStagedEpi && threadIdx.x == 64) mbar_arrive(&bars->epi_free[(g - 1) % kStages]);
        const int slot = __ldg(slot_base + ch.it) + ch.c;
#pragma unroll
        for (int part = 0; part < 2; ++part) {
          const uint32_t col = (part == 0 ? C::kDV : C::kDK) + hf * (D / 2);
          float4* prow = reinterpret_cast<float4*>(partials + ((static_cast<size_t>(slot) * 2 + part) * kM + c) * D +
                                                   hf * (D / 2));
#pragma unroll
          for (int cc = 0; cc < D / 64; ++cc) {
            uint32_t v[32];
            tmem_ld32(tmem + lf + col + cc * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 8; ++e)
              prow[cc * 8 + e] = make_float4(__uint_as_float(v[4 * e]), __uint_as_float(v[4 * e + 1]),
                                             __uint_as_float(v[4 * e + 2]), __uint_as_float(v[4 * e + 3]));
          }
        }
      } else if (kStagedEpi && items > 0 && nkv == kM) {
        // Full key tile: dV -> the Q slot, dK -> the dO slot of the ring stage the item's last
        // pair used (all its UMMAs are complete), SW128 [chunk hf][key row], then TMA stores.
        // Row-per-thread stores held the math warps ~3000 cycles per item (skip-store bound
        // 6 % of the pass). The producer reloads that stage only after epi_free[sl].
        const int sl = (g - 1) % kStages;
#pragma unroll
        for (int part = 0; part < 2; ++part) {
          const uint32_t col = (part == 0 ? C::kDV : C::kDK) + hf * (D / 2);
          const float mul = part == 0 ? 1.0f : scale;
          uint8_t* sp = (part == 0 ? q_smem : do_smem) + sl * C::kQBytes + hf * (kM * 128) + c * 128;
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            uint32_t v[32];
            tmem_ld32(tmem + lf + col + cc * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int u = cc * 4 + k;
              uint4 q4;
              q4.x = pack_bf16x2(__uint_as_float(v[8 * k]) * mul, __uint_as_float(v[8 * k + 1]) * mul);
              q4.y = pack_bf16x2(__uint_as_float(v[8 * k + 2]) * mul, __uint_as_float(v[8 * k + 3]) * mul);
              q4.z = pack_bf16x2(__uint_as_float(v[8 * k + 4]) * mul, __uint_as_float(v[8 * k + 5]) * mul);
              q4.w = pack_bf16x2(__uint_as_float(v[8 * k + 6]) * mul, __uint_as_float(v[8 * k + 7]) * mul);
              *reinterpret_cast<uint4*>(sp + ((u ^ (c & 7)) << 4)) = q4;
            }
          }
        }
        // Warp 10 issues the TMA stores and waits for them to read the stage, so the math
        // warps go straight on to the next item's S^T.
        fence_proxy_async_smem();
        mbar_arrive(&bars->epi_staged[sl]);
      } else {
        if (kStagedEpi && items > 0 && threadIdx.x == 64) mbar_arrive(&bars->epi_free[(g - 1) % kStages]);
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        const uint32_t col = (part == 0 ? C::kDV : C::kDK) + hf * (D / 2);
        const float mul = part == 0 ? 1.0f : scale;
        uint16_t* row = (part == 0 ? dv : dk) + (static_cast<size_t>(kv0 + c) * hkv + w.hk) * D + hf * (D / 2);
#pragma unroll
        for (int cc = 0; cc < D / 64; ++cc) {
          uint32_t v[32];
          if (items > 0) {
            tmem_ld32(tmem + lf + col + cc * 32, v);
            tmem_wait_ld();
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = 0u;
          }
          if (store) {
            SB_DCHECK(kv0 + c < cu[nseq]);
            uint32_t w16[16];
#pragma unroll
            for (int e = 0; e < 16; ++e)
              w16[e] = pack_bf16x2(__uint_as_float(v[2 * e]) * mul, __uint_as_float(v[2 * e + 1]) * mul);
            store_64B(row + cc * 32, w16);
          }
        }
      }
      }
      if (threadIdx.x == 64 && items > 0) tri(4, t - 1);
      tc_fence_before();  // epilogue TMEM reads precede the next item's dV / dK (ordered via pt/dst_full)
    }
  } else if (kStagedEpi) {
    // ------------------------------------------------------------ dV / dK store warp (warp 10)
    // Mirrors the math warps' item walk: for every full key tile it waits for the staged dV / dK
    // (epi_staged), stores them by TMA, and hands the ring stage back to the producer once the
    // stores have read it (epi_free).
    int g = 0;
    uint32_t phase = 0;  // bit st: parity of the next epi_staged[st] phase
    for (int k = 0;; ++k) {
      KvChunk ch;
      if (!next_chunk(k, ch)) break;
      const KvItem& w = ch.w;
      const int items = ch.items;
      g += items;
      if (items == 0 || ch.nc > 1 || min(B, w.seq_len - w.jl * B) != kM) continue;
      const int sl = (g - 1) % kStages;
      const int kv0 = w.seq0 + w.jl * B;
      mbar_wait(&bars->epi_staged[sl], (phase >> sl) & 1u);
      phase ^= 1u << sl;
      if (lane == 0) {
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          tma_store_3d(&tm_dv, q_smem + sl * C::kQBytes + ch * (kM * 128), ch * 64, w.hk, kv0);
          tma_store_3d(&tm_dk, do_smem + sl * C::kQBytes + ch * (kM * 128), ch * 64, w.hk, kv0);
        }
        bulk_commit();
        bulk_wait_read();
        mbar_arrive(&bars->epi_free[sl]);
      }
      __syncwarp();
    }
    if (lane == 0) bulk_wait_all();  // outstanding dV / dK stores reach global before exit
  }
  tc_fence_before();
  __syncthreads();
  if (trace != nullptr && threadIdx.x == 0) trace[8192 + 2 * blockIdx.x + 1] = globaltimer_ns();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kCols>(tmem);
  }
}

// ------------------------------------------------------------------------------------ dq
// Persistent over (q head, q block) items longest-first. Q_i / dO_i of the item live in TMEM
// as the A operands of S = Q K^T and dP = dO V^T: the producer stages them in shared memory
// with TMA and the UMMA warp moves them in with tcgen05.cp, in order behind the previous item's
// last S / dP, so the staging buffer is free to prefetch the next item at once. Shared memory
// is then K / V rings only.
//   TMEM: S | dP | dQ | Q (packed) | dO (packed).
//   Flat block stream g: S_g, dP_g | [s_free_g] S_{g+1} | [ds_g] dQ_g, dP_{g+1} | ...
template <int D, int B>
struct DqCfg {
  static constexpr int kChunks = D / 64;
  static constexpr int kQBytes = kChunks * kM * 128;  // Q or dO tile (128 rows) in the staging buffer
  static constexpr int kKVBytes = kChunks * B * 128;  // K_j or V_j
  static constexpr int kBudget = 232448 - 1024 - 512 - 2 * kQBytes;
  static constexpr int kKStages = (kBudget / kKVBytes - 2) > 4 ? 4 : (kBudget / kKVBytes - 2);
  static constexpr int kVStages = (kBudget / kKVBytes - kKStages) > 4 ? 4 : (kBudget / kKVBytes - kKStages);
  static_assert(kKStages >= 2 && kVStages >= 2, "dq smem rings");
  static constexpr int kSmemTiles = 2 * kQBytes + (kKStages + kVStages) * kKVBytes;
  static constexpr int kS = 0, kDP = B, kDQ = 2 * B, kQa = 2 * B + D, kDOa = 2 * B + D + D / 2;
  static constexpr uint32_t kCols = pow2_cols(2 * B + 2 * D);
  static constexpr int kSmemBytes = kSmemTiles + 1024 + 512;
};

struct DqBars {
  uint64_t stage_full, stage_empty;  // Q / dO staging buffer (TMA -> tcgen05.cp)
  uint64_t dq_staged[2];             // math -> producer: item q's dQ is staged (full tile) / stored (partial), [q & 1]
  uint64_t k_full[4], k_empty[4], v_full[4], v_empty[4];
  uint64_t s_full, s_free, dp_full, dq_done, dq_free;
  uint64_t ds_part[2];  // math -> UMMA: dS of 32-column chunk c2 (of both halves) packed in TMEM
  uint32_t tmem_base;
};

__device__ __forceinline__ void tc_cp_128x256b(uint32_t taddr, uint64_t desc, uint32_t leader) {
  asm volatile(
      "{\n\t.reg .pred l;\n\tsetp.ne.b32 l, %2, 0;\n\t@l tcgen05.cp.cta_group::1.128x256b [%0], %1;\n\t}" ::"r"(taddr),
      "l"(desc), "r"(leader)
      : "memory");
}

template <int D, int B>
__global__ void __launch_bounds__(kThreads, 1) attn_bwd_dq_kernel(
    const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
    const __grid_constant__ CUtensorMap tm_dq, const int32_t* __restrict__ cu, const int32_t* __restrict__ blk_off,
    int nseq, int hq, int hkv, const int32_t* __restrict__ idx, const int32_t* __restrict__ cnt, int hsel, int k_max,
    const float* __restrict__ lse2, const float* __restrict__ dvec, int tp, float scale, float scale_log2,
    uint16_t* __restrict__ dq, const sched::ItemRec* __restrict__ recs, int n_items, unsigned long long* trace) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  using C = DqCfg<D, B>;
  constexpr int kKS = C::kKStages, kVS = C::kVStages;
  if (trace != nullptr && threadIdx.x == 0) trace[8192 + 2 * blockIdx.x] = globaltimer_ns();  // per-CTA span
  auto tr = [&](int slot, int g) {
    if (trace != nullptr && blockIdx.x == 0 && g < 256 && (threadIdx.x & 31) == 0) trace[g * 16 + slot] = clock64();
  };
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* q_stage = smem;                        // staging: Q_i
  uint8_t* do_stage = smem + C::kQBytes;          // staging: dO_i
  uint8_t* k_smem = smem + 2 * C::kQBytes;        // [kKS]
  uint8_t* v_smem = k_smem + kKS * C::kKVBytes;   // [kVS]
  DqBars* bars = reinterpret_cast<DqBars*>(smem + C::kSmemTiles);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nbt = blk_off[nseq];
  const int grid = gridDim.x, cta = blockIdx.x;

  if (threadIdx.x == 0) {
    mbar_init(&bars->stage_full, 1);
    mbar_init(&bars->stage_empty, 1);
    mbar_init(&bars->dq_staged[0], 256);
    mbar_init(&bars->dq_staged[1], 256);
    for (int st = 0; st < 4; ++st) {
      mbar_init(&bars->k_full[st], 1);
      mbar_init(&bars->k_empty[st], 1);
      mbar_init(&bars->v_full[st], 1);
      mbar_init(&bars->v_empty[st], 1);
    }
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->s_free, 256);
    mbar_init(&bars->dp_full, 1);
    mbar_init(&bars->ds_part[0], 256);
    mbar_init(&bars->ds_part[1], 256);
    mbar_init(&bars->dq_done, 1);
    mbar_init(&bars->dq_free, 256);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kCols>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  struct QItem {
    int h, i, seq0, seq_len, n, first;
    const int32_t* list;
  };
  // Item of a prefetched schedule record (sched::q_records_kernel): register arithmetic only.
  auto decode_q = [&](const sched::ItemRec& r) {
    QItem w;
    w.h = r.it / nbt;
    w.i = r.loc;
    w.seq0 = r.seq0;
    w.seq_len = r.seq_len;
    w.n = r.n;
    w.first = r.first;
    w.list = idx + static_cast<size_t>(r.base) * k_max;
    return w;
  };

  if (warp == 0 || warp == 10) {
    // Warp 0 stages Q/dO and streams K, warp 10 streams V (independent rings, separate warps).
    const int role = (warp == 10) ? 1 : 0;
    if (lane == 0) {
      if (role == 0) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_do);
      } else {
        tma_prefetch(&tm_v);
      }
      int g = 0, q = 0;
      // The producer also stores dQ: full tiles are staged by the math warps in the Q half of the
      // staging buffer, and item q + 2's Q / dO may overwrite it only once the store has read it.
      // Pending items q - 2 (p2) and q - 1 (p1): head, first row, full tile.
      int p1h = 0, p1r = 0, p2h = 0, p2r = 0;
      bool p1f = false, p2f = false;
      auto store_dq = [&](int qq, int h, int row0, bool full) {
        mbar_wait(&bars->dq_staged[qq & 1], (qq >> 1) & 1);
        if (full) {
          fence_proxy_async_smem();
#pragma unroll
          for (int c = 0; c < C::kChunks; ++c) tma_store_3d(&tm_dq, q_stage + c * (B * 128), c * 64, h, row0);
          bulk_commit();
          bulk_wait_read();
        }
      };
      for (sched::RecCursor cur(recs, n_items, grid, cta);;) {
        const sched::ItemRec rec = cur.next();
        if (rec.it < 0) break;
        const QItem w = decode_q(rec);
        if (w.n <= 0) continue;
        const int hk = w.h / (hq / hkv);
        if (role == 0) {
          const int row0 = w.seq0 + w.i * B;
          if (q >= 2) store_dq(q - 2, p2h, p2r, p2f);  // item q-2's dQ store has read the buffer
          p2h = p1h, p2r = p1r, p2f = p1f;
          p1h = w.h, p1r = row0, p1f = min(B, w.seq_len - w.i * B) == B;
          mbar_wait(&bars->stage_empty, (q & 1) ^ 1);
          mbar_expect_tx(&bars->stage_full, 2 * C::kQBytes);
          for (int c = 0; c < C::kChunks; ++c) {
            tma_load_3d(q_stage + c * kM * 128, &tm_q, &bars->stage_full, c * 64, w.h, row0);
            tma_load_3d(do_stage + c * kM * 128, &tm_do, &bars->stage_full, c * 64, w.h, row0);
          }
        }
        for (int j = 0; j < w.n; ++j, ++g) {
          const int kv_row = w.seq0 + __ldg(w.list + j) * B;
          if (role == 0) {
            const int st = g % kKS;
            tr(12, g);
            mbar_wait(&bars->k_empty[st], ((g / kKS) & 1) ^ 1);
            tr(13, g);
            mbar_expect_tx(&bars->k_full[st], C::kKVBytes);
            for (int c = 0; c < C::kChunks; ++c)
              tma_load_3d(k_smem + st * C::kKVBytes + c * B * 128, &tm_k, &bars->k_full[st], c * 64, hk, kv_row);
          } else {
            const int vst = g % kVS;
            tr(14, g);
            mbar_wait(&bars->v_empty[vst], ((g / kVS) & 1) ^ 1);
            tr(15, g);
            mbar_expect_tx(&bars->v_full[vst], C::kKVBytes);
            for (int c = 0; c < C::kChunks; ++c)
              tma_load_3d(v_smem + vst * C::kKVBytes + c * B * 128, &tm_v, &bars->v_full[vst], c * 64, hk, kv_row);
          }
        }
        ++q;
      }
      if (role == 0) {
        if (q >= 2) store_dq(q - 2, p2h, p2r, p2f);
        if (q >= 1) store_dq(q - 1, p1h, p1r, p1f);
        bulk_wait_all();  // outstanding dQ stores reach global before exit
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ UMMA issuer (whole warp)
    const uint32_t leader = elect_one();
    constexpr uint32_t idesc_s = idesc_bf16_f32(kM, B, false, false);
    constexpr uint32_t idesc_dq = idesc_bf16_f32(kM, D, false, true);
    const uint32_t k_addr = smem_u32(k_smem), v_addr = smem_u32(v_smem);
    const uint32_t qs_addr = smem_u32(q_stage), ds_addr = smem_u32(do_stage);
    auto load_qdo = [&](int qq) {  // staging -> TMEM, behind the previous item's last S / dP
      if (trace != nullptr && blockIdx.x == 0 && qq < 64 && lane == 0) trace[4096 + qq * 4 + 2] = clock64();
      mbar_wait(&bars->stage_full, qq & 1);
      if (trace != nullptr && blockIdx.x == 0 && qq < 64 && lane == 0) trace[4096 + qq * 4 + 3] = clock64();
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t off = (kk >> 2) * (kM * 128) + (kk & 3) * 32;
        tc_cp_128x256b(tmem + C::kQa + kk * 8, desc_sw128(qs_addr + off, 16, 1024), leader);
        tc_cp_128x256b(tmem + C::kDOa + kk * 8, desc_sw128(ds_addr + off, 16, 1024), leader);
      }
      tc_commit(&bars->stage_empty, leader);
    };
    auto issue_s = [&](int gg) {
      if (gg > 0) mbar_wait(&bars->s_free, (gg - 1) & 1);  // S_{gg-1} read out of TMEM
      const int st = gg % kKS;
      tr(2, gg);
      mbar_wait(&bars->k_full[st], (gg / kKS) & 1);
      tr(3, gg);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t off_n = (kk >> 2) * (B * 128) + (kk & 3) * 32;
        mma_ts(tmem + C::kS, tmem + C::kQa + kk * 8, desc_sw128(k_addr + st * C::kKVBytes + off_n, 16, 1024), idesc_s,
               kk > 0, leader);
      }
      tc_commit(&bars->s_full, leader);
    };
    auto issue_dp = [&](int gg) {
      const int vst = gg % kVS;
      tr(4, gg);
      mbar_wait(&bars->v_full[vst], (gg / kVS) & 1);
      tr(5, gg);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t off_n = (kk >> 2) * (B * 128) + (kk & 3) * 32;
        mma_ts(tmem + C::kDP, tmem + C::kDOa + kk * 8, desc_sw128(v_addr + vst * C::kKVBytes + off_n, 16, 1024),
               idesc_s, kk > 0, leader);
      }
      tc_commit(&bars->dp_full, leader);
      tc_commit(&bars->v_empty[vst], leader);
    };
    sched::RecCursor rc(recs, n_items, grid, cta);
    auto next_item = [&](QItem& w) -> bool {
      for (;;) {
        const sched::ItemRec rec = rc.next();
        if (rec.it < 0) return false;
        w = decode_q(rec);
        if (w.n > 0) return true;
      }
    };
    int g = 0, q = 0;
    QItem cur;
    bool have = next_item(cur);
    if (have) {
      load_qdo(0);
      issue_s(0);
      issue_dp(0);
    }
    while (have) {
      const int n = cur.n;
      QItem nxt;
      bool have_next = false;
      for (int j = 0; j < n; ++j, ++g) {
        const bool last = j + 1 == n;
        if (last) have_next = next_item(nxt);
        const bool more = !last || have_next;
        // Inside an item S_{g+1} goes ahead of dQ_g (it overlaps the math of g). At an item
        // boundary dQ_g goes first, so the dQ epilogue overlaps the next item's Q / dO copy and S_0.
        if (more && !last) issue_s(g + 1);
        tr(0, g);
        const int st = g % kKS;
        // dQ_g in two K halves: the K steps of dS chunk c2 go as soon as both warpgroups packed
        // that chunk, so half of the dS tail overlaps the UMMA.
#pragma unroll
        for (int c2 = 0; c2 < B / 64; ++c2) {
          mbar_wait(&bars->ds_part[c2], g & 1);
          if (c2 == 0) tr(1, g);
          tc_fence_after();
          if (j == 0 && c2 == 0) mbar_wait(&bars->dq_free, (q & 1) ^ 1);  // previous item's dQ read out
#pragma unroll
          for (int kk = 0; kk < B / 16; ++kk) {
            if (((kk % (B / 32)) >> 1) != c2) continue;
            mma_ts(tmem + C::kDQ, tmem + C::kDP + packed_col<B>(kk),
                   desc_sw128(k_addr + st * C::kKVBytes + kk * 2048, B * 128, 1024), idesc_dq,
                   (j > 0 || c2 > 0 || kk > 0) ? 1u : 0u, leader);
          }
        }
        tc_commit(&bars->k_empty[st], leader);
        if (last) tc_commit(&bars->dq_done, leader);
        tr(6, g);
        if (more && last) {
          load_qdo(q + 1);  // in order behind S_g / dP_g, the item's last readers of Q / dO
          issue_s(g + 1);
        }
        if (more) issue_dp(g + 1);
      }
      cur = nxt;
      have = have_next;
      ++q;
    }
  } else if (warp < 10) {
    // ------------------------------------------------------------ math + epilogue
    // Two warpgroups split every query row's B key columns and the D output columns in halves.
    constexpr int HB = B / 2;
    const int quarter = warp & 3;
    const int hf = (warp - 2) >> 2;
    const int r = quarter * 32 + lane;
    const uint32_t lf = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t s_col = C::kS + hf * HB, dp_col = C::kDP + hf * HB;
    int g = 0, q = 0;
    for (sched::RecCursor cur(recs, n_items, grid, cta);;) {
      const sched::ItemRec rec = cur.next();
      if (rec.it < 0) break;
      const QItem w = decode_q(rec);
      const int row0 = w.seq0 + w.i * B;
      const int nrows = min(B, w.seq_len - w.i * B);
      const bool valid = r < nrows;
      uint16_t* dq_row = dq + (static_cast<size_t>(row0 + r) * hq + w.h) * D + hf * (D / 2);
      if (w.n <= 0) {
        if (valid)
          for (int e = 0; e < D / 16; ++e) reinterpret_cast<uint4*>(dq_row)[e] = make_uint4(0, 0, 0, 0);
        continue;
      }
      const float l2 = valid ? __ldg(lse2 + static_cast<size_t>(w.h) * tp + row0 + r) : 0.f;
      const float dd = valid ? __ldg(dvec + static_cast<size_t>(w.h) * tp + row0 + r) : 0.f;
      int jb_nx = w.first;  // loaded one block ahead (see the dkv math loop)
      for (int j = 0; j < w.n; ++j, ++g) {
        const int jb = jb_nx;
        if (j + 1 < w.n) jb_nx = __ldg(w.list + j + 1);
        const int key_lim = min(B, w.seq_len - jb * B);
        const int lim = valid ? min(key_lim, jb == w.i ? r + 1 : B) : 0;
        mbar_wait(&bars->s_full, g & 1);
        if (threadIdx.x == 64) tr(8, g);
        tc_fence_after();
        float p[HB];
        {
          uint32_t sv[HB / 32][32];
#pragma unroll
          for (int c2 = 0; c2 < HB / 32; ++c2) tmem_ld32(tmem + lf + s_col + c2 * 32, sv[c2]);
          tmem_wait_ld();
          tc_fence_before();
          mbar_arrive(&bars->s_free);  // S_g is in registers: S_{g+1} may overwrite it
          if (__all_sync(0xffffffffu, lim >= (hf + 1) * HB)) {
            dq_p<HB, false>(sv, -l2, scale_log2, hf * HB, B, p);
          } else {
            dq_p<HB, true>(sv, -l2, scale_log2, hf * HB, lim, p);
          }
        }
        if (threadIdx.x == 64) tr(9, g);
        mbar_wait(&bars->dp_full, g & 1);
        if (threadIdx.x == 64) tr(10, g);
        tc_fence_after();
        {
          // dP chunks software-pipelined; dS of chunk c2 is packed into columns [c2 * 16, c2 * 16 + 16)
          // of this half, which belong to chunks already read.
          uint32_t pv[2][32];
          tmem_ld32(tmem + lf + dp_col, pv[0]);
          tmem_wait_ld();
#pragma unroll
          for (int c2 = 0; c2 < HB / 32; ++c2) {
            if (c2 + 1 < HB / 32) tmem_ld32(tmem + lf + dp_col + (c2 + 1) * 32, pv[(c2 + 1) & 1]);
            uint32_t dsp[16];
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
              const int c = c2 * 32 + e;
              const f2 ds = fmul2(mk2(p[c], p[c + 1]), fadd2(mk2(__uint_as_float(pv[c2 & 1][e]),
                                                                  __uint_as_float(pv[c2 & 1][e + 1])),
                                                              mk2(-dd, -dd)));
              dsp[e / 2] = pack_bf16x2(ds.x, ds.y);
            }
            tmem_st16(tmem + lf + dp_col + c2 * 16, dsp);
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&bars->ds_part[c2]);
            if (c2 + 1 < HB / 32) tmem_wait_ld();
          }
        }
        if (threadIdx.x == 64) tr(11, g);
      }
      mbar_wait(&bars->dq_done, q & 1);
      if (trace != nullptr && blockIdx.x == 0 && q < 64 && threadIdx.x == 64) trace[4096 + q * 4] = clock64();
      tc_fence_after();
      uint32_t v[D / 64][32];
#pragma unroll
      for (int cc = 0; cc < D / 64; ++cc) tmem_ld32(tmem + lf + C::kDQ + hf * (D / 2) + cc * 32, v[cc]);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&bars->dq_free);
      if (nrows == B) {
        // Full tile: dQ goes out by TMA through the Q half of the staging buffer, once the next
        // item's tcgen05.cp has read its Q / dO from it (no next item: the buffer is idle).
        // The producer issues the store (dq_staged) and loads item q + 2's Q / dO once it has
        // read the buffer. Row-per-thread stores cost ~4.6 % of the pass (skip-store bound).
        bool more = false;
        for (sched::RecCursor peek = cur;;) {
          const sched::ItemRec nr = peek.next();
          if (nr.it < 0) break;
          if (nr.n > 0) {
            more = true;
            break;
          }
        }
        if (more) mbar_wait(&bars->stage_empty, (q & 1) ^ 1);
        if (r < B) {
#pragma unroll
          for (int u = 0; u < D / 16; ++u) {  // 16-byte units of this thread's D/2 columns
            const int ug = hf * (D / 16) + u, d0 = u * 8;
            uint4 q4;
            q4.x = pack_bf16x2(__uint_as_float(v[d0 / 32][d0 % 32]) * scale, __uint_as_float(v[d0 / 32][d0 % 32 + 1]) * scale);
            q4.y = pack_bf16x2(__uint_as_float(v[d0 / 32][d0 % 32 + 2]) * scale, __uint_as_float(v[d0 / 32][d0 % 32 + 3]) * scale);
            q4.z = pack_bf16x2(__uint_as_float(v[d0 / 32][d0 % 32 + 4]) * scale, __uint_as_float(v[d0 / 32][d0 % 32 + 5]) * scale);
            q4.w = pack_bf16x2(__uint_as_float(v[d0 / 32][d0 % 32 + 6]) * scale, __uint_as_float(v[d0 / 32][d0 % 32 + 7]) * scale);
            *reinterpret_cast<uint4*>(q_stage + (ug >> 3) * (B * 128) + r * 128 + (((ug & 7) ^ (r & 7)) << 4)) = q4;
          }
        }
        fence_proxy_async_smem();
      } else {
        if (valid) {  // the last (partial) tile of a sequence: a box would cross into the next
          SB_DCHECK(row0 + r < cu[nseq]);
#pragma unroll
          for (int cc = 0; cc < D / 64; ++cc) {
            uint32_t w16[16];
#pragma unroll
            for (int e = 0; e < 16; ++e)
              w16[e] = pack_bf16x2(__uint_as_float(v[cc][2 * e]) * scale, __uint_as_float(v[cc][2 * e + 1]) * scale);
            store_64B(dq_row + cc * 32, w16);
          }
        }
      }
      mbar_arrive(&bars->dq_staged[q & 1]);
      if (trace != nullptr && blockIdx.x == 0 && q < 64 && threadIdx.x == 64) trace[4096 + q * 4 + 1] = clock64();
      ++q;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (trace != nullptr && threadIdx.x == 0) trace[8192 + 2 * blockIdx.x + 1] = globaltimer_ns();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kCols>(tmem);
  }
}

// ------------------------------------------------------------------------------------ fused
// Single-pass backward for D = B = 128: 5 UMMAs per (key block, q tile) pair instead of the
// two-pass 7. Persistent over key-block items (hk, gj) like the dK/dV pass; per pair it also
// forms the pair's dQ partial dS K in TMEM, which a dedicated warpgroup streams out through a
// small shared-memory ring and TMA-reduce-adds (cp.reduce.async.bulk.tensor, fp32 add in L2) into
// an fp32 dQ accumulator, converted to bf16 by a final elementwise pass. The accumulation order
// of dQ across key blocks is not fixed, so dQ is reproducible to fp32 rounding only; the two-pass
// path stays as the bit-deterministic mode (dK / dV here accumulate in a fixed order).
//
// TMEM (512 columns): SP | dQ | dV | dK. SP holds the pair's two score tiles in turn (S^T and
// dP^T; the math warps read the first before the second is issued) and then P^T | dS^T packed as
// bf16, the A operands of dV += P^T dO and dK += dS^T Q. dQ = dS K reads dS from a dedicated
// shared-memory tile (MN-major A); dP^T_{g+1} is issued after dQ_g, so its completion frees that
// tile for dS_{g+1} with no extra barrier. dO is single-buffered (released after dV_g).
// An item's first pair computes dP^T before S^T, so the next key block's K load (single K
// buffer: K is read by S^T and by dQ up to the item's last pair) overlaps that first dP^T.
//   Issue order: A_g, [sp_free] B_g, [p_ready] dV_g, [ds_ready] dK_g, A_{g+1}, [dsm_ready, dq_free]
//   dQ_g, [sp_free] B_{g+1}, ...   (A / B = S^T / dP^T, swapped on an item's first pair)
// Warps: 0 TMA producer, 1 UMMA issuer, 2-3 idle (WG0, 72 registers); 4-11 two math warpgroups
// splitting every key row's query columns in halves (184 registers); 12-15 the dQ reducer
// (72 registers).
constexpr int kFusedThreads = 512;
constexpr int kRedCols = 16;    // fp32 dQ columns per TMA reduce box (64-byte rows, 64B swizzle)
constexpr int kRedStages = 2;   // staging ring depth

struct FusedCfg {
  static constexpr int kTile = 2 * kM * 128;  // 128 rows x 128 bf16 columns (two SW128 chunks)
  static constexpr int kAug = kM * 32;
  static constexpr int kStage = kM * kRedCols * 4;
  // K | V | Q[2] | dO | dS | ones | qaug[2] | daug | dQ staging[kRedStages]
  static constexpr int kSmemTiles = 6 * kTile + 4 * kAug + kRedStages * kStage;
  static constexpr int kSP = 0, kDQ = 128, kDV = 256, kDK = 384;
  static constexpr uint32_t kCols = 512;
  static constexpr int kSmemBytes = kSmemTiles + 1024 + 256;
};
static_assert(FusedCfg::kSmemBytes <= 232448, "fused backward shared memory");

struct FusedBars {
  uint64_t k_full, k_empty, v_full, v_empty;
  uint64_t q_full[2], q_empty[2], do_full, do_empty;
  uint64_t sp_full, sp_free;               // UMMA <-> math: a score tile in SP / the first one read
  uint64_t p_ready, ds_ready, dsm_ready;   // math -> UMMA: P^T, dS^T packed in SP; dS in smem
  uint64_t dq_full, dq_free;               // UMMA <-> reducer: the pair's dQ partial in TMEM / read
  uint64_t acc_done;                       // UMMA -> math: the item's dV / dK are final
  uint32_t tmem_base;
};

// Pair decode shared by the roles: the m-th (q head, q block) pair of a key-block item.
struct PairCursor {
  const int32_t* tr_ent;
  int nbt, sg;
  __device__ __forceinline__ void get(const KvItem& w, int m, int& h, int& gi) const {
    const int ent = __ldg(tr_ent + w.e0 + m / sg);
    const int hs = ent / nbt;
    gi = ent - hs * nbt;
    h = hs * sg + m % sg;
  }
};

__global__ void __launch_bounds__(kFusedThreads, 1) attn_bwd_fused_kernel(
    const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
    const __grid_constant__ CUtensorMap tm_dqacc, const int32_t* __restrict__ cu, const int32_t* __restrict__ blk_off,
    int nseq, int hq, int hkv, int hsel, const int32_t* __restrict__ tr_off, const int32_t* __restrict__ tr_ent,
    const float* __restrict__ lse2, const float* __restrict__ dvec, int tp, float scale, float scale_log2,
    uint16_t* __restrict__ dk, uint16_t* __restrict__ dv, const int32_t* __restrict__ order, int n_items) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  constexpr int D = 128, B = 128;
  using C = FusedCfg;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* k_smem = smem;
  uint8_t* v_smem = smem + C::kTile;
  uint8_t* q_smem = smem + 2 * C::kTile;   // [2]
  uint8_t* do_smem = smem + 4 * C::kTile;
  uint8_t* ds_smem = smem + 5 * C::kTile;  // dS_g, MN-major A operand of dQ_g
  uint8_t* ones_smem = smem + 6 * C::kTile;
  uint8_t* qaug_smem = ones_smem + C::kAug;      // [2] -lse2 / scale_log2
  uint8_t* daug_smem = qaug_smem + 2 * C::kAug;  // -D
  uint8_t* red_smem = daug_smem + C::kAug;       // [kRedStages] dQ staging
  FusedBars* bars = reinterpret_cast<FusedBars*>(smem + C::kSmemTiles);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nbt = blk_off[nseq];
  const int grid = gridDim.x, cta = blockIdx.x;
  const int sg = hq / hsel;
  const float inv_scale_log2 = 1.0f / scale_log2;
  const PairCursor pc{tr_ent, nbt, sg};

  if (threadIdx.x == 0) {
    mbar_init(&bars->k_full, 1);
    mbar_init(&bars->k_empty, 1);
    mbar_init(&bars->v_full, 1);
    mbar_init(&bars->v_empty, 1);
    for (int st = 0; st < 2; ++st) {
      mbar_init(&bars->q_full[st], 2);  // TMA expect_tx arrive + augmented-slice arrive
      mbar_init(&bars->q_empty[st], 1);
    }
    mbar_init(&bars->do_full, 2);
    mbar_init(&bars->do_empty, 1);
    mbar_init(&bars->sp_full, 1);
    mbar_init(&bars->sp_free, 256);
    mbar_init(&bars->p_ready, 256);
    mbar_init(&bars->ds_ready, 256);
    mbar_init(&bars->dsm_ready, 256);
    mbar_init(&bars->dq_full, 1);
    mbar_init(&bars->dq_free, 128);
    mbar_init(&bars->acc_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kCols>(&bars->tmem_base);
  {
    uint4* z = reinterpret_cast<uint4*>(ones_smem);
    for (int i = threadIdx.x; i < 4 * C::kAug / 16; i += blockDim.x) z[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    for (int r = threadIdx.x; r < kM; r += blockDim.x)
      *reinterpret_cast<uint2*>(ones_smem + aug_off(r)) = make_uint2(0x3F803F80u, 0x00003F80u);
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp < 4) {
    setmaxnreg_dec<72>();
    if (warp == 0) {
      // ---------------------------------------------------------- producer (whole warp)
      if (lane == 0) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        tma_prefetch(&tm_do);
      }
      int g = 0, t = 0;
      auto load_q = [&](int gg, int h, int q0, int nq) {
        const int st = gg & 1;
        float nl[B / 32];
#pragma unroll
        for (int e = 0; e < B / 32; ++e) {
          const int r = e * 32 + lane;
          nl[e] = r < nq ? __ldg(lse2 + static_cast<size_t>(h) * tp + q0 + r) : 0.f;
        }
        mbar_wait(&bars->q_empty[st], ((gg >> 1) & 1) ^ 1);
        if (lane == 0) {
          mbar_expect_tx(&bars->q_full[st], C::kTile);
          for (int c = 0; c < 2; ++c)
            tma_load_3d(q_smem + st * C::kTile + c * kM * 128, &tm_q, &bars->q_full[st], c * 64, h, q0);
        }
        uint8_t* qa = qaug_smem + st * C::kAug;
#pragma unroll
        for (int e = 0; e < B / 32; ++e)
          *reinterpret_cast<uint2*>(qa + aug_off(e * 32 + lane)) = split3_bf16(-nl[e] * inv_scale_log2);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->q_full[st]);
      };
      auto load_do = [&](int gg, int h, int q0, int nq) {
        float nd[B / 32];
#pragma unroll
        for (int e = 0; e < B / 32; ++e) {
          const int r = e * 32 + lane;
          nd[e] = r < nq ? __ldg(dvec + static_cast<size_t>(h) * tp + q0 + r) : 0.f;
        }
        mbar_wait(&bars->do_empty, (gg & 1) ^ 1);
        if (lane == 0) {
          mbar_expect_tx(&bars->do_full, C::kTile);
          for (int c = 0; c < 2; ++c) tma_load_3d(do_smem + c * kM * 128, &tm_do, &bars->do_full, c * 64, h, q0);
        }
#pragma unroll
        for (int e = 0; e < B / 32; ++e)
          *reinterpret_cast<uint2*>(daug_smem + aug_off(e * 32 + lane)) = split3_bf16(-nd[e]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->do_full);
      };
      for (int k = 0;; ++k) {
        const int it = sched::snake_item(order, n_items, grid, cta, k);
        if (it < 0) break;
        const KvItem w = decode_kv(it, cu, blk_off, nseq, nbt, tr_off);
        const int items = w.ne * sg;
        if (items == 0) continue;
        const int kv0 = w.seq0 + w.jl * B;
        const int blk0 = w.gj - w.jl;
        if (lane == 0) {  // V first: the item's first UMMA is dP^T
          tma_prefetch_l2_3d(&tm_k, 0, w.hk, kv0);
          tma_prefetch_l2_3d(&tm_k, 64, w.hk, kv0);
          mbar_wait(&bars->v_empty, (t & 1) ^ 1);
          mbar_expect_tx(&bars->v_full, C::kTile);
          for (int c = 0; c < 2; ++c) tma_load_3d(v_smem + c * kM * 128, &tm_v, &bars->v_full, c * 64, w.hk, kv0);
        }
        for (int m = 0; m < items; ++m, ++g) {
          int h, gi;
          pc.get(w, m, h, gi);
          const int q0 = w.seq0 + (gi - blk0) * B;
          const int nq = min(B, w.seq_len - (gi - blk0) * B);
          if (m == 0) {
            load_do(g, h, q0, nq);
            load_q(g, h, q0, nq);
            if (lane == 0) {  // K after the first pair's dO / Q: the previous item's last dQ reads K
              mbar_wait(&bars->k_empty, (t & 1) ^ 1);
              mbar_expect_tx(&bars->k_full, C::kTile);
              for (int c = 0; c < 2; ++c) tma_load_3d(k_smem + c * kM * 128, &tm_k, &bars->k_full, c * 64, w.hk, kv0);
            }
          } else {
            load_q(g, h, q0, nq);
            load_do(g, h, q0, nq);
          }
        }
        ++t;
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------- UMMA issuer (whole warp)
      const uint32_t leader = elect_one();
      constexpr uint32_t idesc_t = idesc_bf16_f32(kM, B, false, false);
      constexpr uint32_t idesc_acc = idesc_bf16_f32(kM, D, false, true);
      constexpr uint32_t idesc_dq = idesc_bf16_f32(kM, D, true, true);
      const uint32_t k_addr = smem_u32(k_smem), v_addr = smem_u32(v_smem), ones_addr = smem_u32(ones_smem);
      const uint32_t do_addr = smem_u32(do_smem), ds_addr = smem_u32(ds_smem);
      auto qa = [&](int gg) { return smem_u32(q_smem + (gg & 1) * C::kTile); };
      auto issue_st = [&](int gg) {
        mbar_wait_spin(&bars->q_full[gg & 1], (gg >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * (kM * 128) + (kk & 3) * 32;
          mma_ss(tmem + C::kSP, desc_sw128(k_addr + off, 16, 1024), desc_sw128(qa(gg) + off, 16, 1024), idesc_t,
                 kk > 0, leader);
        }
        mma_ss(tmem + C::kSP, desc_aug(ones_addr), desc_aug(smem_u32(qaug_smem + (gg & 1) * C::kAug)), idesc_t, 1u,
               leader);
        tc_commit(&bars->sp_full, leader);
      };
      auto issue_dpt = [&](int gg) {
        mbar_wait_spin(&bars->do_full, gg & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * (kM * 128) + (kk & 3) * 32;
          mma_ss(tmem + C::kSP, desc_sw128(v_addr + off, 16, 1024), desc_sw128(do_addr + off, 16, 1024), idesc_t,
                 kk > 0, leader);
        }
        mma_ss(tmem + C::kSP, desc_aug(ones_addr), desc_aug(smem_u32(daug_smem)), idesc_t, 1u, leader);
        tc_commit(&bars->sp_full, leader);
      };
      int g = 0, t = 0, k = 0;
      bool a_issued = false;  // tile A of pair g already issued (at the end of pair g - 1)
      auto next_item = [&](KvItem& out) -> bool {
        for (;; ++k) {
          const int it = sched::snake_item(order, n_items, grid, cta, k);
          if (it < 0) return false;
          out = decode_kv(it, cu, blk_off, nseq, nbt, tr_off);
          if (out.ne * sg > 0) {
            ++k;
            return true;
          }
        }
      };
      KvItem w;
      bool have = next_item(w);
      while (have) {
        const int items = w.ne * sg;
        KvItem nx;
        bool have_nx = false;
        for (int m = 0; m < items; ++m, ++g) {
          const bool last = m + 1 == items;
          if (!a_issued) {  // only the CTA's very first pair: dP^T first
            mbar_wait_spin(&bars->v_full, t & 1);
            issue_dpt(g);
          }
          a_issued = false;
          mbar_wait_spin(&bars->sp_free, g & 1);  // tile B
          if (m == 0) {
            mbar_wait_spin(&bars->k_full, t & 1);
            issue_st(g);
          } else {
            issue_dpt(g);
          }
          if (last) tc_commit(&bars->v_empty, leader);  // the item's last dP^T is issued
          mbar_wait_spin(&bars->p_ready, g & 1);  // dV_g += P^T dO_g (TS: P^T packed at SP + hf*64 + [0, 32))
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < B / 16; ++kk)
            mma_ts(tmem + C::kDV, tmem + C::kSP + (kk >> 2) * 64 + (kk & 3) * 8,
                   desc_sw128(do_addr + kk * 2048, kM * 128, 1024), idesc_acc, (m > 0 || kk > 0) ? 1u : 0u, leader);
          tc_commit(&bars->do_empty, leader);
          mbar_wait_spin(&bars->ds_ready, g & 1);  // dK_g += dS^T Q_g (TS: dS^T packed at SP + hf*64 + [32, 64))
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < B / 16; ++kk)
            mma_ts(tmem + C::kDK, tmem + C::kSP + (kk >> 2) * 64 + 32 + (kk & 3) * 8,
                   desc_sw128(qa(g) + kk * 2048, kM * 128, 1024), idesc_acc, (m > 0 || kk > 0) ? 1u : 0u, leader);
          tc_commit(&bars->q_empty[g & 1], leader);
          // tile A of the next pair (overwrites SP after dV_g / dK_g read it: in-order pipe)
          if (!last) {
            issue_st(g + 1);
            a_issued = true;
          } else {
            have_nx = next_item(nx);
            if (have_nx) {
              mbar_wait_spin(&bars->v_full, (t + 1) & 1);
              issue_dpt(g + 1);
              a_issued = true;
            }
          }
          // dQ_g = dS_g K  (SS: A = dS MN-major; B = K MN-major)
          mbar_wait_spin(&bars->dsm_ready, g & 1);
          if (g > 0) mbar_wait_spin(&bars->dq_free, (g - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < B / 16; ++kk)
            mma_ss(tmem + C::kDQ, desc_sw128(ds_addr + kk * 2048, kM * 128, 1024),
                   desc_sw128(k_addr + kk * 2048, kM * 128, 1024), idesc_dq, kk > 0 ? 1u : 0u, leader);
          tc_commit(&bars->dq_full, leader);
          if (last) {
            tc_commit(&bars->acc_done, leader);
            tc_commit(&bars->k_empty, leader);
          }
        }
        ++t;
        w = nx;
        have = have_nx;
      }
    }
  } else if (warp < 12) {
    // ------------------------------------------------------------ math + dK/dV epilogue
    setmaxnreg_inc<184>();
    constexpr int HB = B / 2;
    const int quarter = warp & 3;
    const int hf = (warp - 4) >> 2;
    const int c = quarter * 32 + lane;  // TMEM lane: key row
    const uint32_t lf = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t sp = tmem + lf + C::kSP + hf * HB;
    int g = 0, t = 0;
    for (int k = 0;; ++k) {
      const int it = sched::snake_item(order, n_items, grid, cta, k);
      if (it < 0) break;
      const KvItem w = decode_kv(it, cu, blk_off, nseq, nbt, tr_off);
      const int items = w.ne * sg;
      const int kv0 = w.seq0 + w.jl * B;
      const int nkv = min(B, w.seq_len - w.jl * B);
      const int blk0 = w.gj - w.jl;
      for (int m = 0; m < items; ++m, ++g) {
        int h, gi;
        pc.get(w, m, h, gi);
        const int il = gi - blk0;
        const int nq = min(B, w.seq_len - il * B);
        // Valid query columns r >= r_lo: r >= key row on the diagonal; none for key rows past the
        // sequence end (their dS must be 0: dQ sums over every key row of the tile).
        const int r_lo = c >= nkv ? B : (il == w.jl ? c : 0);
        // ta <- S^T, tb <- dP^T. Tiles arrive as A then B (sp_full completions 2g, 2g + 1); A is
        // S^T except on an item's first pair (dP^T first). When S^T comes first its exponentials
        // run while the UMMA computes dP^T.
        uint32_t ta[HB / 32][32], tb[HB / 32][32];
        float p[HB];
        auto exp_p = [&]() {
          if (r_lo <= hf * HB && nq == B) {
            dkv_p<HB, false>(ta, scale_log2, hf * HB, 0, B, p);
          } else {
            dkv_p<HB, true>(ta, scale_log2, hf * HB, r_lo, nq, p);
          }
        };
        if (m > 0) {
          mbar_wait_spin(&bars->sp_full, 0);
          tc_fence_after();
#pragma unroll
          for (int c2 = 0; c2 < HB / 32; ++c2) tmem_ld32(sp + c2 * 32, ta[c2]);
          tmem_wait_ld();
          tc_fence_before();
          mbar_arrive(&bars->sp_free);
          exp_p();
          mbar_wait_spin(&bars->sp_full, 1);
          tc_fence_after();
#pragma unroll
          for (int c2 = 0; c2 < HB / 32; ++c2) tmem_ld32(sp + c2 * 32, tb[c2]);
          tmem_wait_ld();
        } else {
          mbar_wait_spin(&bars->sp_full, 0);
          tc_fence_after();
#pragma unroll
          for (int c2 = 0; c2 < HB / 32; ++c2) tmem_ld32(sp + c2 * 32, tb[c2]);
          tmem_wait_ld();
          tc_fence_before();
          mbar_arrive(&bars->sp_free);
          mbar_wait_spin(&bars->sp_full, 1);
          tc_fence_after();
#pragma unroll
          for (int c2 = 0; c2 < HB / 32; ++c2) tmem_ld32(sp + c2 * 32, ta[c2]);
          tmem_wait_ld();
          exp_p();
        }
        {
          uint32_t pw[2][16];
#pragma unroll
          for (int e = 0; e < HB; e += 2) pw[e / 32][(e % 32) / 2] = pack_bf16x2(p[e], p[e + 1]);
          tmem_st16(sp, pw[0]);
          tmem_st16(sp + 16, pw[1]);
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&bars->p_ready);
        }
        uint32_t dsw[HB / 2];
#pragma unroll
        for (int e = 0; e < HB; e += 2) {  // dS^T = P^T (dP^T - D): the UMMA already subtracted D
          const f2 ds = fmul2(mk2(p[e], p[e + 1]),
                              mk2(__uint_as_float(tb[e / 32][e % 32]), __uint_as_float(tb[e / 32][e % 32 + 1])));
          dsw[e / 2] = pack_bf16x2(ds.x, ds.y);
        }
        {
          uint32_t d0[16], d1[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            d0[e] = dsw[e];
            d1[e] = dsw[16 + e];
          }
          tmem_st16(sp + 32, d0);
          tmem_st16(sp + 48, d1);
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&bars->ds_ready);
        }
        // dS (bf16) as the MN-major A operand of dQ_g: chunk hf holds query columns
        // [hf*64, hf*64 + 64) of every key row c (128-byte rows, SW128). dQ_{g-1} has read the
        // tile: it was issued before dP^T_g, whose completion (tile B / A above) we waited for.
        uint8_t* dsm = ds_smem + hf * (kM * 128) + c * 128;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          *reinterpret_cast<uint4*>(dsm + ((u ^ (c & 7)) << 4)) =
              make_uint4(dsw[4 * u], dsw[4 * u + 1], dsw[4 * u + 2], dsw[4 * u + 3]);
        fence_proxy_async_smem();
        mbar_arrive(&bars->dsm_ready);
      }
      // Epilogue: dV and dK * scale for the valid key rows (zeros if nobody selected the block).
      if (items > 0) {
        mbar_wait(&bars->acc_done, t & 1);
        tc_fence_after();
        ++t;
      }
      const bool store = c < nkv;
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        const uint32_t col = (part == 0 ? C::kDV : C::kDK) + hf * (D / 2);
        const float mul = part == 0 ? 1.0f : scale;
        uint16_t* row = (part == 0 ? dv : dk) + (static_cast<size_t>(kv0 + c) * hkv + w.hk) * D + hf * (D / 2);
#pragma unroll
        for (int cc = 0; cc < D / 64; ++cc) {
          uint32_t vv[32];
          if (items > 0) {
            tmem_ld32(tmem + lf + col + cc * 32, vv);
            tmem_wait_ld();
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) vv[e] = 0u;
          }
          if (store) {
            uint32_t w16[16];
#pragma unroll
            for (int e = 0; e < 16; ++e)
              w16[e] = pack_bf16x2(__uint_as_float(vv[2 * e]) * mul, __uint_as_float(vv[2 * e + 1]) * mul);
            store_64B(row + cc * 32, w16);
          }
        }
      }
      tc_fence_before();  // epilogue TMEM reads precede the next item's first dV / dK (ordered via p_ready)
    }
  } else {
    // ------------------------------------------------------------ dQ reducer (warps 12..15)
    // Per pair: the 128 x 128 fp32 dQ partial (TMEM lanes = query rows) in 32-column slices ->
    // 16-column boxes through a kRedStages ring (64-byte rows, 64B swizzle) -> TMA reduce-add.
    setmaxnreg_dec<72>();
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t lf = static_cast<uint32_t>(quarter * 32) << 16;
    const bool elected = r == 0;
    int g = 0, n = 0;  // pair counter, staged box counter
    for (int k = 0;; ++k) {
      const int it = sched::snake_item(order, n_items, grid, cta, k);
      if (it < 0) break;
      const KvItem w = decode_kv(it, cu, blk_off, nseq, nbt, tr_off);
      const int items = w.ne * sg;
      const int blk0 = w.gj - w.jl;
      for (int m = 0; m < items; ++m, ++g) {
        int h, gi;
        pc.get(w, m, h, gi);
        const int q0 = w.seq0 + (gi - blk0) * B;
        mbar_wait(&bars->dq_full, g & 1);
        tc_fence_after();
#pragma unroll 1
        for (int sl = 0; sl < D / 32; ++sl) {
          uint32_t v[32];
          tmem_ld32(tmem + lf + C::kDQ + sl * 32, v);
          tmem_wait_ld();
          if (sl == D / 32 - 1) {
            tc_fence_before();
            mbar_arrive(&bars->dq_free);  // the whole partial is in registers / staged
          }
#pragma unroll
          for (int half = 0; half < 32 / kRedCols; ++half, ++n) {
            uint8_t* stg = red_smem + (n % kRedStages) * C::kStage;
            if (elected) bulk_wait_read<kRedStages - 1>();  // this slot's previous box has been read
            named_bar_sync(3, 128);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int e = half * kRedCols + 4 * u;
              *reinterpret_cast<uint4*>(stg + r * 64 + ((u ^ ((r >> 1) & 3)) << 4)) =
                  make_uint4(v[e], v[e + 1], v[e + 2], v[e + 3]);
            }
            fence_proxy_async_smem();
            named_bar_sync(3, 128);
            if (elected) {
              tma_reduce_add_3d(&tm_dqacc, stg, sl * 32 + half * kRedCols, h, q0);
              bulk_commit();
            }
          }
        }
      }
    }
    if (elected) bulk_wait_all();  // every dQ reduce has landed before the kernel ends
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kCols>(tmem);
  }
}

// Split order for the dK/dV pass (one CTA of 1024 threads). cap = max(kSplitMinPairs,
// ceil(total pairs / (kSplitPerCta * grid))); an item of P > cap pairs becomes nc = ceil(P / cap)
// consecutive entries (chunks) at its place in the longest-first order, and gets slot_base[it]
// (its first fp32 partial slot) and a split_list entry {it, nc, slot0}. counts = {entries,
// split items}. Thread t owns positions [t * per, (t + 1) * per): count, block scan, write.
__global__ void __launch_bounds__(1024) dkv_split_kernel(const int32_t* __restrict__ order, int n,
                                                         const int32_t* __restrict__ tr_off, int kv_items, int sg,
                                                         int grid, int32_t* __restrict__ out,
                                                         int32_t* __restrict__ counts, int32_t* __restrict__ slot_base,
                                                         int4* __restrict__ split_list) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  __shared__ int wsum[3][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int total = __ldg(tr_off + kv_items) * sg;
  const int cap = max(kSplitMinPairs, (total + kSplitPerCta * grid - 1) / (kSplitPerCta * grid));
  const int per = (n + 1023) / 1024;
  const int i0 = min(n, threadIdx.x * per), i1 = min(n, i0 + per);
  auto nchunks = [&](int it) {
    const int P = (__ldg(tr_off + it + 1) - __ldg(tr_off + it)) * sg;
    return P > cap ? min(kSplitMaxChunks, (P + cap - 1) / cap) : 1;
  };
  int v[3] = {0, 0, 0};  // entries, split items, partial slots
  for (int i = i0; i < i1; ++i) {
    const int nc = nchunks(__ldg(order + i));
    v[0] += nc;
    if (nc > 1) {
      v[1] += 1;
      v[2] += nc;
    }
  }
  int x[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {  // block-wide exclusive scan
    int incl = v[j];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[j][warp] = incl;
    x[j] = incl - v[j];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int w0 = wsum[j][lane];
      int incl = w0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      wsum[j][lane] = incl - w0;
    }
  }
  __syncthreads();
  int oa = x[0] + wsum[0][warp], ob = x[1] + wsum[1][warp], oc = x[2] + wsum[2][warp];
  for (int i = i0; i < i1; ++i) {
    const int it = __ldg(order + i);
    const int nc = nchunks(it);
    for (int q = 0; q < nc; ++q) out[oa + q] = it | (q << kSplitItemBits) | (nc << (kSplitItemBits + 4));
    oa += nc;
    if (nc > 1) {
      SB_DCHECK(oc + nc <= split_slots(grid));
      slot_base[it] = oc;
      split_list[ob] = make_int4(it, nc, oc, 0);
      ++ob;
      oc += nc;
    }
  }
  if (threadIdx.x == 1023) {
    counts[0] = oa;
    counts[1] = ob;
    counts[2] = 0;  // the dK/dV pass's dynamic schedule cursor
  }
}

// KvRec of every split-order entry (positions < counts[0]), grid-stride.
__global__ void __launch_bounds__(256) dkv_records_kernel(const int32_t* __restrict__ order,
                                                          const int32_t* __restrict__ counts,
                                                          const int32_t* __restrict__ cu,
                                                          const int32_t* __restrict__ blk_off, int nseq, int nbt,
                                                          const int32_t* __restrict__ tr_off, KvRec* __restrict__ recs) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  const int n = __ldg(counts);
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const int e = order[p];
    const KvItem w = decode_kv(e & ((1 << kSplitItemBits) - 1), cu, blk_off, nseq, nbt, tr_off);
    reinterpret_cast<int4*>(recs + p)[0] = make_int4(e, w.hk, w.gj, w.jl);
    reinterpret_cast<int4*>(recs + p)[1] = make_int4(w.seq0, w.seq_len, w.e0, w.ne);
  }
}

// dK / dV of the split items: sum of the chunks' fp32 partials in chunk order (deterministic),
// dK * scale, bf16, valid key rows only. One thread per 4-column granule; a task is 256
// granules (256 / (D / 4) key rows) of one part of one split item, grid-strided. All of a
// granule's nc (<= 15) partial loads are issued before the adds.
template <int D, int B>
// Split reduce launch shape (ncu, C3 profile-only launches): all chunk loads in flight at 78
// registers, 8 CTAs per SM grid, 27-28 us; 4-chunk batches at 32 registers (8 CTAs of 256 per
// SM), 16 CTAs per SM grid, 16-19 us.
#ifndef SB_REDUCE_BATCHED
#define SB_REDUCE_BATCHED 1
#endif
#ifndef SB_REDUCE_MINB
#define SB_REDUCE_MINB 8
#endif
#ifndef SB_REDUCE_GRID
#define SB_REDUCE_GRID 16
#endif
__global__ void __launch_bounds__(256, SB_REDUCE_MINB) dkv_split_reduce_kernel(const int4* __restrict__ split_list,
                                                               const int32_t* __restrict__ counts,
                                                               const float* __restrict__ partials,
                                                               const int32_t* __restrict__ cu,
                                                               const int32_t* __restrict__ blk_off, int nseq, int nbt,
                                                               int hkv, float scale, uint16_t* __restrict__ dk,
                                                               uint16_t* __restrict__ dv) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  constexpr int kG = kM * D / 4;         // float4 granules per part (128 key rows)
  constexpr int kTasksPerPart = kG / 256;
  const int n_tasks = __ldg(counts + 1) * 2 * kTasksPerPart;
  for (int task = blockIdx.x; task < n_tasks; task += gridDim.x) {
    const int si = task / (2 * kTasksPerPart);
    const int rem_t = task - si * 2 * kTasksPerPart;
    const int part = rem_t / kTasksPerPart;
    const int gidx = (rem_t - part * kTasksPerPart) * 256 + threadIdx.x;  // granule in the part
    const int row = gidx / (D / 4), c4 = gidx - row * (D / 4);
    const int4 e = __ldg(split_list + si);
    const int it = e.x, nc = e.y, slot0 = e.z;
    const int hk = it / nbt, gj = it - hk * nbt;
    const int s = seq_of_block(blk_off, nseq, gj);
    const int kv0 = cu[s] + (gj - blk_off[s]) * B;
    const int nkv = min(B, cu[s + 1] - kv0);
    if (row >= nkv) continue;
    const float4* p = reinterpret_cast<const float4*>(partials) + (static_cast<size_t>(slot0) * 2 + part) * kG + gidx;
#if SB_REDUCE_BATCHED
    // Chunks in batches of 4 loads, summed in chunk order from chunk 0's value (bit-identical).
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int q0 = 0; q0 < nc; q0 += 4) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (q0 + u < nc) v[u] = __ldg(p + static_cast<size_t>(q0 + u) * 2 * kG);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (q0 + u >= nc) break;
        if (q0 + u == 0) {
          a = v[u];
        } else {
          a.x += v[u].x, a.y += v[u].y, a.z += v[u].z, a.w += v[u].w;
        }
      }
    }
#else
    float4 v[kSplitMaxChunks];
#pragma unroll
    for (int q = 0; q < kSplitMaxChunks; ++q)
      if (q < nc) v[q] = __ldg(p + static_cast<size_t>(q) * 2 * kG);
    float4 a = v[0];
#pragma unroll
    for (int q = 1; q < kSplitMaxChunks; ++q)
      if (q < nc) a.x += v[q].x, a.y += v[q].y, a.z += v[q].z, a.w += v[q].w;
#endif
    const float mul = part ? scale : 1.0f;
    uint2 o;
    o.x = pack_bf16x2(a.x * mul, a.y * mul);
    o.y = pack_bf16x2(a.z * mul, a.w * mul);
    *reinterpret_cast<uint2*>((part ? dk : dv) + (static_cast<size_t>(kv0 + row) * hkv + hk) * D + c4 * 4) = o;
  }
}

// dQ = bf16(acc * scale): 8 fp32 -> 8 bf16 (one 16-byte store) per thread and step.
__global__ void __launch_bounds__(256) dq_convert_kernel(const float4* __restrict__ acc, size_t n8, float scale,
                                                         uint4* __restrict__ dq) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const float4 a = __ldg(acc + 2 * i), b = __ldg(acc + 2 * i + 1);
    dq[i] = make_uint4(pack_bf16x2(a.x * scale, a.y * scale), pack_bf16x2(a.z * scale, a.w * scale),
                       pack_bf16x2(b.x * scale, b.y * scale), pack_bf16x2(b.z * scale, b.w * scale));
  }
}

// ------------------------------------------------------------------------------------ host
constexpr int kMaxKvCost = 1023;  // longest-first order resolution (costs above share the top bin)
unsigned long long* g_trace_bwd = nullptr;  // debug timeline buffer (sb_debug_set_trace_bwd)
unsigned long long* g_trace_dq = nullptr;   // debug timeline buffer (sb_debug_set_trace_dq)

struct BwdWorkspace {
  size_t lse2, dvec, tr_cnt, tr_off, tr_ent, order_q, order_kv, order_kv_matched, rec_q, dqacc;
  size_t order_split, split_counts, slot_base, split_list, partials, recs_split, total;
  int tp;
};

inline size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

BwdWorkspace bwd_layout(int total, int nb_total, int hq, int hkv, int hsel, int k_max, bool fused = true) {
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
  w.order_q = off;
  off = align256(off + sched::order_workspace_bytes(hq * nb_total, hq * (k_max + 1)));
  w.order_kv = off;
  off = align256(off + sched::order_workspace_bytes(hkv * nb_total, hkv * (kMaxKvCost + 1)));
  w.order_kv_matched = off;
  off = align256(off + static_cast<size_t>(hkv) * nb_total * 4);
  w.rec_q = off;
  off = align256(off + sched::rec_workspace_bytes(hq * nb_total));
  // dK/dV item split (dkv_split_kernel): entries, {entries, split items}, per-item first slot,
  // split list, fp32 partials [slot][dV, dK][128 key rows][D <= 128].
  const int sms = sched::num_sms();
  const size_t kv_items = static_cast<size_t>(hkv) * nb_total;
  w.order_split = off;
  off = align256(off + (kv_items + split_slots(sms)) * 4);
  w.split_counts = off;
  off = align256(off + 16);
  w.slot_base = off;
  off = align256(off + kv_items * 4);
  w.split_list = off;
  off = align256(off + static_cast<size_t>(split_slots(sms)) * 16);
  w.partials = off;
  off = align256(off + static_cast<size_t>(split_slots(sms)) * 2 * kM * 128 * 4);
  w.recs_split = off;
  off = align256(off + (kv_items + split_slots(sms)) * sizeof(KvRec));
  w.dqacc = off;  // fused path (D = 128): fp32 dQ accumulator [T][Hq][128]
  if (fused) off = align256(off + static_cast<size_t>(total) * hq * 128 * 4);
  w.total = off;
  return w;
}

template <int D, int B>
void launch_bwd(const uint16_t* q, const uint16_t* k, const uint16_t* v, const uint16_t* o, const uint16_t* d_o,
                const uint16_t* ores, const float* lse, const int32_t* cu, const int32_t* blk_off, int nseq, int total, int nb_total, int hq,
                int hkv, const int32_t* idx, const int32_t* cnt, int hsel, int k_max, float scale, uint16_t* dq,
                uint16_t* dk, uint16_t* dv, uint8_t* ws, cudaStream_t st, bool fused_requested) {
  constexpr bool kFusable = D == 128 && B == 128;
  const bool fused = kFusable && fused_requested;
  const BwdWorkspace w = bwd_layout(total, nb_total, hq, hkv, hsel, k_max, fused);
  float* lse2 = reinterpret_cast<float*>(ws + w.lse2);
  float* dvec = reinterpret_cast<float*>(ws + w.dvec);
  int32_t* tr_cnt = reinterpret_cast<int32_t*>(ws + w.tr_cnt);
  int32_t* tr_off = reinterpret_cast<int32_t*>(ws + w.tr_off);
  int32_t* tr_ent = reinterpret_cast<int32_t*>(ws + w.tr_ent);
  const float scale_log2 = scale * kLog2e;
  const int sms = sched::num_sms();

  launch(bwd_prep_kernel, sms * SB_PREP_GRID, 256, 0, st, o, d_o, ores, lse, total, hq, D, w.tp, lse2,
                                                                         dvec);
  launched("sb_sparse_attn_bwd/prep");
  const int kv_items = hkv * nb_total;
  const int rows_per_kv = hsel / hkv;
  launch(transpose_sel_kernel, (kv_items + 3) / 4, 128, 0, st, idx, cnt, blk_off, nseq, hkv, rows_per_kv, k_max, 0,
                                                            tr_cnt, nullptr, nullptr);
  launched("sb_sparse_attn_bwd/transpose_count");
  launch(scan_kernel, 1, 1024, 0, st, tr_cnt, kv_items, tr_off);
  launched("sb_sparse_attn_bwd/scan");
  launch(transpose_sel_kernel, (kv_items + 3) / 4, 128, 0, st, idx, cnt, blk_off, nseq, hkv, rows_per_kv, k_max, 1,
                                                            tr_cnt, tr_off, tr_ent);
  launched("sb_sparse_attn_bwd/transpose_fill");
  // Two-pass dK/dV (dynamic claiming): long items lead their head (CostFromLists::lead). Fused
  // (static snake + round matching): plain head-major longest-first.
  const int grid_kv = std::min(kv_items, sms);
  sched::CostFromLists kv_cost{tr_off, hq / hsel, kMaxKvCost, nb_total, hkv};
#ifndef SB_DKV_LEAD
#define SB_DKV_LEAD 1
#endif
  if (!fused && SB_DKV_LEAD) {
    // Long = over a quarter of the split cap; a cap-sized entry lasts ~hkv / 4 heads' stretch of
    // the list (cap = total / (kSplitPerCta * grid) pairs, one head = total / (hkv * grid) per CTA).
#ifndef SB_DKV_LONG_FRAC
#define SB_DKV_LONG_FRAC 4
#endif
#ifndef SB_DKV_LONG_MIN
#define SB_DKV_LONG_MIN kSplitMinPairs
#endif
    kv_cost.long_div = SB_DKV_LONG_FRAC * kSplitPerCta * grid_kv;
    kv_cost.long_min = SB_DKV_LONG_MIN;
    kv_cost.lead = (hkv + kSplitPerCta - 1) / kSplitPerCta;
  }
  const int32_t* order_kv_lpt = sched::build_order(kv_cost, kv_items, ws + w.order_kv, st, "sb_sparse_attn_bwd/order_kv");
  // Round matching (sched.cuh) runs its rounds in sequence on one CTA, ~5.3 us per round of 148
  // (both cost constants below were calibrated on B200)
  // items on B200; it wins ~6 % of the dK/dV pass where items are long (C5: -4 to -10 % bwd) and
  // loses where they are short (C2: 295 us of matching for ~110 us won). Use it only when 6 % of
  // the dK/dV upper-bound estimate (hq * NB * k_max q tiles at ~2.3 us, causal half) exceeds it.
  const double match_us = 5.3 * ((kv_items + grid_kv - 1) / grid_kv);
  const double dkv_est_us = static_cast<double>(hq) * nb_total * k_max * 2.3 / 2.0 / grid_kv;
  const int32_t* order_kv = order_kv_lpt;
  // match_rounds_kernel keeps per-CTA state in 256-entry shared arrays: grid_kv <= 256 (B200: 148).
  // Only the fused kernel walks a static snake; the two-pass dK/dV kernel claims entries dynamically.
  if (fused && grid_kv <= sched::kMatchMaxGrid && match_us < 0.06 * dkv_est_us) {
    int32_t* matched = reinterpret_cast<int32_t*>(ws + w.order_kv_matched);
    launch(sched::match_rounds_kernel<sched::ListCost>, 1, sched::kMatchThreads, 0, st, sched::ListCost{tr_off, hq / hsel}, order_kv_lpt,
                                                                   kv_items, grid_kv, matched);
    launched("sb_sparse_attn_bwd/order_kv_match");
    order_kv = matched;
  }
  if constexpr (kFusable) {
    if (fused) {
      float* dqacc = reinterpret_cast<float*>(ws + w.dqacc);
      cuda_check(cudaMemsetAsync(dqacc, 0, static_cast<size_t>(total) * hq * D * 4, st), "sb_sparse_attn_bwd: dQ acc");
      const CUtensorMap tq = make_thd_map(q, total, hq, D, kM);
      const CUtensorMap tdo = make_thd_map(d_o, total, hq, D, kM);
      const CUtensorMap tk = make_thd_map(k, total, hkv, D, kM);
      const CUtensorMap tv = make_thd_map(v, total, hkv, D, kM);
      const CUtensorMap tacc = make_thd_map_f32(dqacc, total, hq, D, kM, kRedCols);
      set_smem_once(attn_bwd_fused_kernel, FusedCfg::kSmemBytes, "sb_sparse_attn_bwd: smem attribute (fused)");
      launch(attn_bwd_fused_kernel, std::min(kv_items, sms), kFusedThreads, FusedCfg::kSmemBytes, st, 
          tq, tk, tv, tdo, tacc, cu, blk_off, nseq, hq, hkv, hsel, tr_off, tr_ent, lse2, dvec, w.tp, scale, scale_log2,
          dk, dv, order_kv, kv_items);
      launched("sb_sparse_attn_bwd/fused");
      const size_t n8 = static_cast<size_t>(total) * hq * D / 8;
      launch(dq_convert_kernel, std::max(1, std::min<int>(sms * 8, static_cast<int>((n8 + 255) / 256))), 256, 0, st, 
          reinterpret_cast<const float4*>(dqacc), n8, scale, reinterpret_cast<uint4*>(dq));
      launched("sb_sparse_attn_bwd/dq_convert");
      return;
    }
  }
  // Long items -> chunks (see kSplitItemBits); the dK/dV pass walks the split order.
  require(kv_items < (1 << kSplitItemBits), "sb_sparse_attn_bwd: too many (kv head, key block) items");
  int32_t* order_split = reinterpret_cast<int32_t*>(ws + w.order_split);
  int32_t* split_counts = reinterpret_cast<int32_t*>(ws + w.split_counts);
  int32_t* slot_base = reinterpret_cast<int32_t*>(ws + w.slot_base);
  int4* split_list = reinterpret_cast<int4*>(ws + w.split_list);
  float* partials = reinterpret_cast<float*>(ws + w.partials);
  launch(dkv_split_kernel, 1, 1024, 0, st, order_kv, kv_items, tr_off, kv_items, hq / hsel, grid_kv, order_split,
                                       split_counts, slot_base, split_list);
  launched("sb_sparse_attn_bwd/split");
  KvRec* recs_split = reinterpret_cast<KvRec*>(ws + w.recs_split);
  {
    const int n_max = kv_items + split_slots(sms);
    launch(dkv_records_kernel, std::max(1, std::min(4 * sms, (n_max + 255) / 256)), 256, 0, st, order_split,
           split_counts, cu, blk_off, nseq, nb_total, tr_off, recs_split);
    launched("sb_sparse_attn_bwd/records_kv");
  }
  const int q_items = hq * nb_total;
  auto* rec_q = reinterpret_cast<sched::ItemRec*>(ws + w.rec_q);
  sched::build_q_schedule(sched::CostFromCnt{cnt, k_max, hq, hsel, nb_total}, q_items, ws + w.order_q, rec_q, cu,
                          blk_off, nseq, idx, k_max, st, "sb_sparse_attn_bwd/order_q");

  // dK / dV: key tiles are 128 rows (UMMA M); query tiles are B rows (UMMA N).
  {
    using C = DkvCfg<D, B>;
    const CUtensorMap tq = make_thd_map(q, total, hq, D, B);
    const CUtensorMap tdo = make_thd_map(d_o, total, hq, D, B);
    const CUtensorMap tk = make_thd_map(k, total, hkv, D, kM);
    const CUtensorMap tv = make_thd_map(v, total, hkv, D, kM);
    const CUtensorMap tdk = make_thd_map(dk, total, hkv, D, kM);
    const CUtensorMap tdv = make_thd_map(dv, total, hkv, D, kM);
    auto kern = attn_bwd_dkv_kernel<D, B>;
    set_smem_once(kern, C::kSmemBytes, "sb_sparse_attn_bwd: smem attribute (dkv)");
    launch(kern, std::min(kv_items, sms), kThreads, C::kSmemBytes, st, tq, tk, tv, tdo, tdk, tdv, cu, blk_off, nseq, hq, hkv, hsel,
                                                                   tr_off, tr_ent, lse2, dvec, w.tp, scale,
                                                                   scale_log2, dk, dv, recs_split, split_counts,
                                                                   slot_base, partials, g_trace_bwd);
    launched("sb_sparse_attn_bwd/dkv");
    launch(dkv_split_reduce_kernel<D, B>, SB_REDUCE_GRID * sms, 256, 0, st, split_list, split_counts, partials, cu, blk_off, nseq,
                                                            nb_total, hkv, scale, dk, dv);
    launched("sb_sparse_attn_bwd/split_reduce");
  }
  {
    using C = DqCfg<D, B>;
    const CUtensorMap tq = make_thd_map(q, total, hq, D, kM);
    const CUtensorMap tdo = make_thd_map(d_o, total, hq, D, kM);
    const CUtensorMap tk = make_thd_map(k, total, hkv, D, B);
    const CUtensorMap tv = make_thd_map(v, total, hkv, D, B);
    const CUtensorMap tdq = make_thd_map(dq, total, hq, D, B);
    auto kern = attn_bwd_dq_kernel<D, B>;
    set_smem_once(kern, C::kSmemBytes, "sb_sparse_attn_bwd: smem attribute (dq)");
    launch(kern, std::min(q_items, sms), kThreads, C::kSmemBytes, st, tq, tk, tv, tdo, tdq, cu, blk_off, nseq, hq, hkv, idx,
                                                                  cnt, hsel, k_max, lse2, dvec, w.tp, scale,
                                                                  scale_log2, dq, rec_q, q_items, g_trace_dq);
    launched("sb_sparse_attn_bwd/dq");
  }
}

}  // namespace
}  // namespace sbk

// Debug only: device buffer of 256 x 16 uint64 for CTA 0 of the dK/dV pass (NULL disables).
SB_API void sb_debug_set_trace_bwd(unsigned long long* buf) { sbk::g_trace_bwd = buf; }
// Debug only: the same for CTA 0 of the dQ pass.
SB_API void sb_debug_set_trace_dq(unsigned long long* buf) { sbk::g_trace_dq = buf; }

SB_API size_t sb_sparse_attn_bwd_workspace_size(int total_tokens, int nb_total, int hq, int hkv, int head_dim, int hsel,
                                                int k_max) {
  (void)head_dim;
  return sbk::bwd_layout(total_tokens, nb_total, hq, hkv, hsel, k_max).total;
}

SB_API size_t sb_sparse_attn_bwd_workspace_size_ex(int nseq, int total_tokens, int nb_total, int hq, int hkv,
                                                   int head_dim, int hsel, int k_max, int block_size, int flags) {
  (void)head_dim;
  const bool fused = (flags & SB_BWD_FUSED) != 0;  // only the fused pass needs the fp32 dQ accumulator
  if (block_size != 256) return sbk::bwd_layout(total_tokens, nb_total, hq, hkv, hsel, k_max, fused).total;
  return sbk::expand256_workspace_bytes(nseq, nb_total, hsel, k_max) +
         sbk::bwd_layout(total_tokens, 2 * nb_total, hq, hkv, hsel, 2 * k_max, fused).total;
}

SB_API int sb_sparse_attn_bwd_ex(const uint16_t* q, const uint16_t* k, const uint16_t* v, const uint16_t* o,
                                 const uint16_t* o_res, const uint16_t* d_o, const float* lse, const int32_t* cu_seqlens, const int32_t* blk_off,
                                 int nseq, int total_tokens, int nb_total, int hq, int hkv, int head_dim, int block_size,
                                 const int32_t* idx, const int32_t* cnt, int hsel, int k_max, float scale, uint16_t* dq,
                                 uint16_t* dk, uint16_t* dv, void* workspace, void* stream, int flags) {
  return sbk::abi_call([&] {
    sbk::require(head_dim == 64 || head_dim == 128, "head_dim must be 64 or 128");
    sbk::require(block_size == 64 || block_size == 128 || block_size == 256, "block_size must be 64, 128 or 256");
    sbk::require(hq >= 1 && hkv >= 1 && hq % hkv == 0, "hq must be a positive multiple of hkv");
    sbk::require(hsel >= hkv && hq % hsel == 0 && hsel % hkv == 0,
                 "hsel must divide hq and be a multiple of hkv (each selection row maps to one kv head)");
    sbk::require(k_max >= 1, "k_max must be >= 1");
    sbk::require((flags & ~(SB_BWD_DETERMINISTIC | SB_BWD_FUSED)) == 0, "unknown flags");
    sbk::require((flags & SB_BWD_DETERMINISTIC) == 0 || (flags & SB_BWD_FUSED) == 0,
                 "SB_BWD_FUSED is not deterministic (dQ is reduce-added in fp32)");
    if (nseq == 0 || nb_total == 0 || total_tokens == 0) return;
    sbk::require(q && k && v && o && d_o && lse && cu_seqlens && blk_off && idx && cnt && dq && dk && dv && workspace,
                 "null pointer");
    sbk::require((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v) |
                  reinterpret_cast<uintptr_t>(o) | reinterpret_cast<uintptr_t>(d_o) | reinterpret_cast<uintptr_t>(dq) |
                  reinterpret_cast<uintptr_t>(dk) | reinterpret_cast<uintptr_t>(dv) |
                  reinterpret_cast<uintptr_t>(workspace) | reinterpret_cast<uintptr_t>(o_res)) % 16 == 0,
                 "q/k/v/o/o_res/dO/dQ/dK/dV/workspace must be 16-byte aligned");
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    const bool det = (flags & SB_BWD_FUSED) != 0;  // fused requested (the default two-pass is deterministic)
    if (block_size == 256) {  // workspace: sb_sparse_attn_bwd_workspace_size_ex
      const sbk::Expanded256 e =
          sbk::expand_selection_256(cu_seqlens, blk_off, nseq, nb_total, hsel, idx, cnt, k_max, ws, st);
      if (head_dim == 128)
        return sbk::launch_bwd<128, 128>(q, k, v, o, d_o, o_res, lse, cu_seqlens, e.blk_off, nseq, total_tokens,
                                         e.nb_total, hq, hkv, e.idx, e.cnt, hsel, e.k_max, scale, dq, dk, dv,
                                         ws + e.used, st, det);
      return sbk::launch_bwd<64, 128>(q, k, v, o, d_o, o_res, lse, cu_seqlens, e.blk_off, nseq, total_tokens,
                                      e.nb_total, hq, hkv, e.idx, e.cnt, hsel, e.k_max, scale, dq, dk, dv, ws + e.used,
                                      st, det);
    }
#define SB_BWD_CASE(DD, BB)                                                                                     \
  if (head_dim == DD && block_size == BB)                                                                       \
    return sbk::launch_bwd<DD, BB>(q, k, v, o, d_o, o_res, lse, cu_seqlens, blk_off, nseq, total_tokens, nb_total, hq, \
                                   hkv, idx, cnt, hsel, k_max, scale, dq, dk, dv, ws, st, det);
    SB_BWD_CASE(128, 128)
    SB_BWD_CASE(128, 64)
    SB_BWD_CASE(64, 128)
    SB_BWD_CASE(64, 64)
#undef SB_BWD_CASE
  });
}

SB_API int sb_sparse_attn_bwd(const uint16_t* q, const uint16_t* k, const uint16_t* v, const uint16_t* o,
                              const uint16_t* d_o, const float* lse, const int32_t* cu_seqlens, const int32_t* blk_off,
                              int nseq, int total_tokens, int nb_total, int hq, int hkv, int head_dim, int block_size,
                              const int32_t* idx, const int32_t* cnt, int hsel, int k_max, float scale, uint16_t* dq,
                              uint16_t* dk, uint16_t* dv, void* workspace, void* stream) {
  return sb_sparse_attn_bwd_ex(q, k, v, o, nullptr, d_o, lse, cu_seqlens, blk_off, nseq, total_tokens, nb_total, hq, hkv,
                               head_dim, block_size, idx, cnt, hsel, k_max, scale, dq, dk, dv, workspace, stream, 0);
}
