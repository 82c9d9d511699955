// Work order for the persistent attention kernels: head-major, longest-first within a head.
//
// Work items (one q block x head, or one key block x kv head) have very different costs in a
// varlen batch with per-sequence keep counts (1 .. k_max selected blocks). Items are sorted by
// the key (head, cost descending): keeping one head's items together makes the ~148 resident
// CTAs share that head's K/V (or Q/dO) slabs in L2 (16 MB per head at 32K tokens, d=128),
// while longest-first inside the head and across the whole list keeps the tail short. CTAs
// of the dQ pass walk the list in snake order (c, 2G-1-c, 2G+c, ...); the forward (per item
// stream) and the dK/dV pass take their first round there and claim every later entry from a
// global cursor (attn_fwd.cu kFwdRing, attn_bwd.cu kSchedRing). The sort is a counting sort on
// the device (histogram, scan, scatter).
#pragma once

#include "common.cuh"

namespace sbk {
namespace sched {
namespace {  // internal linkage: included by several translation units

// Sort keys in [0, bins): key = head * (max_cost + 1) + (max_cost - min(cost, max_cost)).
struct CostFromCnt {  // fwd / dq: item = h * NB + gi, cost = cnt[srow(h)][gi]
  const int32_t* cnt;
  int max_cost;
  int hq, hsel, nb_total;
  __device__ int operator()(int item) const {
    const int h = item / nb_total, gi = item - h * nb_total;
    const int c = cnt[static_cast<size_t>(h / (hq / hsel)) * nb_total + gi];
    return h * (max_cost + 1) + (max_cost - min(c, max_cost));
  }
  int bins() const { return hq * (max_cost + 1); }
};

struct CostFromLists {  // dkv: item = hk * NB + gj, cost = (#selection rows listing it) * heads per row
  const int32_t* tr_off;
  int per_entry;
  int max_cost;
  int nb_total, hkv;
  // lead > 0 (dK/dV, dynamic claiming): an item longer than thr = max(long_min, ceil(total /
  // long_div)) pairs is ordered with head hk - lead instead of its own head, so no long item is
  // claimed in the last `lead` heads' stretch of the list and the pass ends on short items. With
  // plain head-major order the last head's long items (split chunks and items just under the
  // split cap, ~100 us each at C3) ran alone after every other CTA had finished.
  int lead = 0, long_div = 1, long_min = 0;
  __device__ int operator()(int item) const {
    int hk = item / nb_total;
    const int c = (tr_off[item + 1] - tr_off[item]) * per_entry;
    if (lead > 0) {
      const int total = tr_off[nb_total * hkv] * per_entry;
      const int thr = max(long_min, (total + long_div - 1) / long_div);
      if (c > thr) hk = max(0, hk - lead);
    }
    return hk * (max_cost + 1) + (max_cost - min(c, max_cost));
  }
  int bins() const { return hkv * (max_cost + 1); }
};

template <typename Key>
__global__ void key_hist_kernel(Key key, int n_items, int32_t* __restrict__ hist) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_items; i += gridDim.x * blockDim.x)
    atomicAdd(hist + key(i), 1);
}

// start[b] = number of items with key < b (exclusive scan, one CTA of 1024); resets the
// histogram so it can serve as the scatter cursor. Warp w owns a contiguous segment of
// 32 * per bins and walks it with coalesced loads: pass 1 sums the segment, one block-wide
// scan of the 32 warp totals, pass 2 re-walks it with a warp inclusive scan per 32 bins (the
// bin count reaches ~3 * 10^4 for the key-block order).
__global__ void __launch_bounds__(1024) key_start_kernel(int32_t* __restrict__ hist, int bins,
                                                         int32_t* __restrict__ start) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  __shared__ int warp_sum[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int per = (bins + 1023) / 1024;  // 32-bin steps per warp
  const int seg0 = warp * 32 * per;
  int v = 0;
#pragma unroll 4
  for (int it = 0; it < per; ++it) {
    const int b = seg0 + it * 32 + lane;
    v += b < bins ? hist[b] : 0;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) warp_sum[warp] = v;
  __syncthreads();
  if (warp == 0) {
    const int x = warp_sum[lane];
    int incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    warp_sum[lane] = incl - x;  // exclusive
  }
  __syncthreads();
  int carry = warp_sum[warp];
  for (int it = 0; it < per; ++it) {
    const int b = seg0 + it * 32 + lane;
    const int h = b < bins ? hist[b] : 0;
    int incl = h;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (b < bins) {
      start[b] = carry + incl - h;
      hist[b] = 0;
    }
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
}

template <typename Key>
__global__ void scatter_kernel(Key key, int n_items, const int32_t* __restrict__ start,
                               int32_t* __restrict__ cursor, int32_t* __restrict__ order) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_items; i += gridDim.x * blockDim.x) {
    const int b = key(i);
    order[start[b] + atomicAdd(cursor + b, 1)] = i;
  }
}

// The whole counting sort in one CTA (shared-memory histogram, in-place exclusive scan, scatter
// with the scanned starts as cursors): one launch instead of memset + three kernels, ~10 us per
// order on the small per-layer item counts (the multi-kernel path is launch-latency bound).
// 32 KB of shared memory: zeroing and scanning more bins in one CTA costs more than the launches
// it saves (the dK/dV order's 32 x 1024 bins: 15.6 us one-CTA vs ~11 us multi-kernel).
constexpr int kSortOneCtaMaxBins = 8192;
constexpr int kSortOneCtaMaxItems = 1 << 17;
template <typename Key>
__device__ __forceinline__ void sort_one_cta_body(Key key, int n_items, int bins, int32_t* __restrict__ order,
                                                  int32_t* sh, int* warp_sum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int b = threadIdx.x; b < bins; b += 1024) sh[b] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n_items; i += 1024) atomicAdd(&sh[key(i)], 1);
  __syncthreads();
  const int per = (bins + 1023) / 1024;  // 32-bin steps per warp
  const int seg0 = warp * 32 * per;
  int v = 0;
  for (int it = 0; it < per; ++it) {
    const int b = seg0 + it * 32 + lane;
    v += b < bins ? sh[b] : 0;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) warp_sum[warp] = v;
  __syncthreads();
  if (warp == 0) {
    const int x = warp_sum[lane];
    int incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    warp_sum[lane] = incl - x;
  }
  __syncthreads();
  int carry = warp_sum[warp];
  for (int it = 0; it < per; ++it) {
    const int b = seg0 + it * 32 + lane;
    const int h = b < bins ? sh[b] : 0;
    int incl = h;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (b < bins) sh[b] = carry + incl - h;
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n_items; i += 1024) order[atomicAdd(&sh[key(i)], 1)] = i;
}

template <typename Key>
__global__ void __launch_bounds__(1024) sort_one_cta_kernel(Key key, int n_items, int bins,
                                                            int32_t* __restrict__ order) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  extern __shared__ int32_t sh[];
  __shared__ int warp_sum[32];
  sort_one_cta_body(key, n_items, bins, order, sh, warp_sum);
}

inline size_t order_workspace_bytes(int n_items, int bins) {
  return (static_cast<size_t>(n_items) + 2 * static_cast<size_t>(bins) + 64) * sizeof(int32_t);
}

// Writes order[0..n_items) (ascending key) into ws. Returns the order pointer.
template <typename Key>
int32_t* build_order(Key key, int n_items, void* ws, cudaStream_t st, const char* who) {
  const int bins = key.bins();
  int32_t* order = static_cast<int32_t*>(ws);
  if (bins <= kSortOneCtaMaxBins && n_items <= kSortOneCtaMaxItems) {
    const int smem = bins * static_cast<int>(sizeof(int32_t));
    set_smem_once(sort_one_cta_kernel<Key>, smem, who);
    launch(sort_one_cta_kernel<Key>, 1, 1024, smem, st, key, n_items, bins, order);
    launched(who);
    return order;
  }
  int32_t* hist = order + n_items;
  int32_t* start = hist + bins;
  cuda_check(cudaMemsetAsync(hist, 0, sizeof(int32_t) * bins, st), who);
  const int blocks = min(1184, (n_items + 255) / 256);
  launch(key_hist_kernel<Key>, blocks, 256, 0, st, key, n_items, hist);
  launched(who);
  launch(key_start_kernel, 1, 1024, 0, st, hist, bins, start);
  launched(who);
  launch(scatter_kernel<Key>, blocks, 256, 0, st, key, n_items, start, hist, order);
  launched(who);
  return order;
}

// Round matching over a longest-first order. The snake layout hands every CTA exactly one item
// per round of `grid` consecutive positions; plain snake ignores what each CTA already holds, so
// when a round straddles two heads (head-major order) or costs fall steeply inside a round the
// per-CTA totals drift apart (modelled 1.03-1.11 max/mean at C2 / C5). Here, round by round, the
// largest item of the round goes to the least-loaded CTA so far (ties by index), written back at
// that CTA's snake slot, so the hot kernels walk `out` exactly as they walk `order`. Items stay in
// their round, so head-major L2 locality is kept. One CTA runs the rounds in sequence.
// Only the placement changes: every item is still computed whole by one CTA, so outputs are
// bit-identical.
// 1024 threads: thread (target = t & 255, chunk = t >> 8) counts its quarter of the pairwise
// compares and adds them into the target's rank, so a round costs ~40 compares and 4 barriers.
constexpr int kMatchThreads = 1024;
constexpr int kMatchMaxGrid = 256;  // shared arrays below are sized per CTA of the consuming grid
template <typename Cost>
__global__ void __launch_bounds__(kMatchThreads) match_rounds_kernel(Cost cost, const int32_t* __restrict__ order,
                                                                     int n_items, int grid, int32_t* __restrict__ out) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  __shared__ int load[kMatchMaxGrid], item_cost[kMatchMaxGrid], item_id[kMatchMaxGrid], cta_at[kMatchMaxGrid],
      rank_cta[kMatchMaxGrid], rank_item[kMatchMaxGrid];
  if (grid > kMatchMaxGrid) __trap();  // host gates on grid <= kMatchMaxGrid (B200 has 148 SMs)
  const int t = threadIdx.x, tgt = t & 255, chunk = t >> 8;
  const int per = (grid + 3) / 4, u0 = chunk * per, u1 = min(grid, u0 + per);
  if (t < 256) load[t] = 0;
  const int rounds = (n_items + grid - 1) / grid;
  for (int r = 0; r < rounds; ++r) {
    const int base = r * grid;
    const int m = min(grid, n_items - base);
    const bool odd = r & 1;
    if (t < 256) {
      rank_cta[t] = 0;
      rank_item[t] = 0;
      if (t < m) {
        item_id[t] = order[base + t];
        item_cost[t] = cost(item_id[t]);
      }
    }
    __syncthreads();
    // CTAs whose snake slot in this round exists (all of them except in the last round).
    if (tgt < grid && (odd ? grid - 1 - tgt : tgt) < m) {
      const int L = load[tgt];
      int rk = 0;
      for (int u = u0; u < u1; ++u) {
        if ((odd ? grid - 1 - u : u) >= m) continue;
        const int Lu = load[u];
        rk += (Lu < L) || (Lu == L && u < tgt);
      }
      if (rk) atomicAdd(&rank_cta[tgt], rk);
    }
    if (tgt < m) {
      const int c = item_cost[tgt];
      int rk = 0;
      for (int u = u0; u < min(u1, m); ++u) {
        const int cu = item_cost[u];
        rk += (cu > c) || (cu == c && u < tgt);
      }
      if (rk) atomicAdd(&rank_item[tgt], rk);
    }
    __syncthreads();
    if (t < grid && (odd ? grid - 1 - t : t) < m) cta_at[rank_cta[t]] = t;
    __syncthreads();
    if (t < m) {
      const int cta = cta_at[rank_item[t]];
      out[base + (odd ? grid - 1 - cta : cta)] = item_id[t];
      load[cta] += item_cost[t];
    }
    __syncthreads();
  }
}

struct ListCost {  // dkv item cost in q tiles: (#selection rows listing it) * heads per row, + 1 boundary
  const int32_t* tr_off;
  int per_entry;
  __device__ int operator()(int item) const { return (tr_off[item + 1] - tr_off[item]) * per_entry + 1; }
};

// Item handled by CTA `cta` of `grid` in round k of the snake order (or -1 when exhausted).
__device__ __forceinline__ int snake_item(const int32_t* __restrict__ order, int n_items, int grid, int cta, int k) {
  const int pos = k * grid + ((k & 1) ? (grid - 1 - cta) : cta);
  return pos < n_items ? __ldg(order + pos) : -1;
}

// One record per schedule position, so a persistent CTA's roles read an item with one 32-byte
// load (prefetched a whole item ahead by RecCursor) instead of decoding it at the item
// boundary through a chain of dependent global loads (order -> blk_off binary search -> cu ->
// cnt / tr_off -> list[0]); that chain put ~2-3k cycles on every boundary of every role.
struct ItemRec {
  int it;       // item id (h * nbt + gi for q items, hk * nbt + gj for kv items)
  int s;        // sequence
  int loc;      // block index inside the sequence
  int seq0;     // first token of the sequence
  int seq_len;  // tokens in the sequence
  int n;        // q items: selected key blocks (cnt); kv items: listing selection rows
  int base;     // q items: selection row srow * nbt + gi; kv items: tr_off[it]
  int first;    // q items: first selected key block; kv items: first listing entry
};
static_assert(sizeof(ItemRec) == 32, "ItemRec is two 16-byte loads");

inline size_t rec_workspace_bytes(int n_items) { return static_cast<size_t>(n_items) * sizeof(ItemRec) + 256; }

__device__ __forceinline__ ItemRec q_record(int it, const int32_t* __restrict__ cu, const int32_t* __restrict__ blk_off,
                                            int nseq, int nbt, int hq, int hsel, const int32_t* __restrict__ idx,
                                            const int32_t* __restrict__ cnt, int k_max) {
  ItemRec r;
  r.it = it;
  const int h = r.it / nbt, gi = r.it - h * nbt;
  r.s = seq_of_block(blk_off, nseq, gi);
  r.loc = gi - blk_off[r.s];
  r.seq0 = cu[r.s];
  r.seq_len = cu[r.s + 1] - r.seq0;
  r.base = (h / (hq / hsel)) * nbt + gi;
  r.n = cnt[r.base];
  r.first = r.n > 0 ? idx[static_cast<size_t>(r.base) * k_max] : 0;
  return r;
}

__global__ void q_records_kernel(const int32_t* __restrict__ order, int n_items, const int32_t* __restrict__ cu,
                                 const int32_t* __restrict__ blk_off, int nseq, int nbt, int hq, int hsel,
                                 const int32_t* __restrict__ idx, const int32_t* __restrict__ cnt, int k_max,
                                 ItemRec* __restrict__ rec) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos == 0) *reinterpret_cast<int*>(rec + n_items) = 0;  // the forward's dynamic-claim cursor
  if (pos >= n_items) return;
  rec[pos] = q_record(order[pos], cu, blk_off, nseq, nbt, hq, hsel, idx, cnt, k_max);
}

// Longest-first q-item order + its records (fwd and dQ passes). Returns the order pointer.
inline int32_t* build_q_schedule(const CostFromCnt& key, int n_items, void* order_ws, ItemRec* rec,
                                 const int32_t* cu, const int32_t* blk_off, int nseq, const int32_t* idx, int k_max,
                                 cudaStream_t st, const char* who) {
  // (Fusing the records into the one-CTA sort measured 50 us against 13 + 4: each record is a
  // chain of dependent loads, which one CTA cannot overlap the way 40 CTAs do.)
  int32_t* order = build_order(key, n_items, order_ws, st, who);
  launch(q_records_kernel, (n_items + 255) / 256, 256, 0, st, order, n_items, cu, blk_off, nseq, key.nb_total, key.hq,
                                                          key.hsel, idx, key.cnt, k_max, rec);
  launched(who);
  return order;
}

__global__ void kv_records_kernel(const int32_t* __restrict__ order, int n_items, const int32_t* __restrict__ cu,
                                  const int32_t* __restrict__ blk_off, int nseq, int nbt,
                                  const int32_t* __restrict__ tr_off, const int32_t* __restrict__ tr_ent,
                                  ItemRec* __restrict__ rec) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= n_items) return;
  ItemRec r;
  r.it = order[pos];
  const int hk = r.it / nbt, gj = r.it - hk * nbt;
  r.s = seq_of_block(blk_off, nseq, gj);
  r.loc = gj - blk_off[r.s];
  r.seq0 = cu[r.s];
  r.seq_len = cu[r.s + 1] - r.seq0;
  r.base = tr_off[r.it];
  r.n = tr_off[r.it + 1] - r.base;
  r.first = r.n > 0 ? tr_ent[r.base] : 0;
  rec[pos] = r;
}

// Walks a CTA's snake-order records; next() returns the current record (it = -1 past the end)
// while the load of the following one is already in flight.
struct RecCursor {
  const int4* rec;
  int n_items, grid, cta, k, kstep;
  int4 a, b;
  // Rounds k0, k0 + kstep, ... of the CTA's snake order (kstep 2: one of two item streams).
  __device__ RecCursor(const ItemRec* r, int n, int g, int c, int k0 = 0, int step = 1)
      : rec(reinterpret_cast<const int4*>(r)), n_items(n), grid(g), cta(c), k(k0), kstep(step) {
    load();
  }
  __device__ __forceinline__ void load() {
    const int pos = k * grid + ((k & 1) ? (grid - 1 - cta) : cta);
    if (pos < n_items) {
      a = __ldg(rec + 2 * pos);
      b = __ldg(rec + 2 * pos + 1);
    } else {
      a = make_int4(-1, 0, 0, 0);
      b = make_int4(0, 0, 0, 0);
    }
  }
  __device__ __forceinline__ ItemRec next() {
    const ItemRec r{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    k += kstep;
    if (r.it >= 0) load();
    return r;
  }
};

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    cuda_check(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev), "SM count");
  }
  return n;
}

}  // namespace
}  // namespace sched
}  // namespace sbk
