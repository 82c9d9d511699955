// K8: on-device DST decision for fixed-base mode.
//
// In fixed-base mode every input of the tuner except the routing profile is known on the host
// before the step: x_i (summed length), k_base, T_base = predict(x_i, k_base), the anchor
// (select_anchor over all micro-batches) and k_anchor = align(x_i, anchor), hence also the
// bottleneck flag T_base > anchor. Only the coverage test of tune_budget (reference
// dst.cpp:107-143) needs this layer's profile, which K4 produces on the device. This kernel
// merges the micro-batch's member profiles exactly as make_micro_batch (workload.cpp:64-99)
// and runs the coverage test and the smallest-safe-budget search (dst.cpp:87-103), so the
// keep counts go from K4 straight to the selector with no host round trip per layer.
//
// Bit-exactness with the host: every fp64 operation is an explicitly rounded intrinsic in the
// host's order (no FMA contraction), sums are sequential left to right, and the merged profile
// needs no re-sort (a non-negatively weighted sum of non-increasing vectors is non-increasing
// under monotone rounding, and so is its division by the norm).
#include "common.cuh"
#include "sb_kernels.h"

namespace sbk {
namespace {

constexpr int kDstThreads = 256;
constexpr int kDstMaxWidth = 4096;

// coverage(profile, k) of the normalised merged profile acc[0..m): 0 for k <= 0, 1 for k >= m,
// else the sequential sum of the first k entries (dst.cpp:53-61).
__device__ double coverage_seq(const double* acc, int m, int k) {
  if (k <= 0) return 0.0;
  if (k >= m) return 1.0;
  double c = 0.0;
  for (int j = 0; j < k; ++j) c = __dadd_rn(c, acc[j]);
  return c;
}

__global__ void __launch_bounds__(kDstThreads) dst_decide_kernel(
    const double* __restrict__ profile, const int32_t* __restrict__ blk_off, const int32_t* __restrict__ cu,
    int nb_max, const int32_t* __restrict__ mb_off, const int32_t* __restrict__ k_base,
    const int32_t* __restrict__ k_anchor, const int32_t* __restrict__ bottleneck, const int32_t* __restrict__ grid,
    int ngrid, double p, int32_t* __restrict__ k_final, double* __restrict__ cov_drop, int32_t* __restrict__ k_seq) {
  pdl_wait();  // see launch() (common.cuh)
  pdl_trigger();
  __shared__ double acc[kDstMaxWidth];
  __shared__ double sh_norm;
  __shared__ int sh_kf;
  const int mb = blockIdx.x;
  const int s0 = mb_off[mb], s1 = mb_off[mb + 1];
  int width = 0;
  long long total = 0;
  for (int s = s0; s < s1; ++s) {
    width = max(width, blk_off[s + 1] - blk_off[s]);
    total += cu[s + 1] - cu[s];
  }
  const double total_d = static_cast<double>(total);
  // Token-weighted sum, zero-padded to the widest member, members in order (workload.cpp:79-90).
  for (int j = threadIdx.x; j < width; j += blockDim.x) {
    double a = 0.0;
    for (int s = s0; s < s1; ++s) {
      if (j < blk_off[s + 1] - blk_off[s]) {
        const double w = __ddiv_rn(static_cast<double>(cu[s + 1] - cu[s]), total_d);
        a = __dadd_rn(a, __dmul_rn(w, profile[static_cast<size_t>(s) * nb_max + j]));
      }
    }
    acc[j] = a;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double norm = 0.0;
    for (int j = 0; j < width; ++j) norm = __dadd_rn(norm, acc[j]);
    sh_norm = norm;
  }
  __syncthreads();
  const double norm = sh_norm;
  if (norm > 0.0)
    for (int j = threadIdx.x; j < width; j += blockDim.x) acc[j] = __ddiv_rn(acc[j], norm);
  __syncthreads();
  if (threadIdx.x == 0) {
    const int kb = k_base[mb], ka = k_anchor[mb];
    const double cb = coverage_seq(acc, width, kb);
    int kf;
    if (!bottleneck[mb]) {
      kf = ka;  // expand into the slack (or keep)
    } else if (__dadd_rn(cb, -coverage_seq(acc, width, ka)) <= p) {
      kf = ka;  // anchor-aligned budget is coverage-safe
    } else {  // smallest grid budget within p of the base coverage; densest if none
      auto safe = [&](int gi) { return __dadd_rn(cb, -coverage_seq(acc, width, grid[gi])) <= p; };
      int unsafe = 0, ok = ngrid - 1;
      if (!safe(ok)) {
        kf = grid[ok];
      } else if (safe(unsafe)) {
        kf = grid[unsafe];
      } else {
        while (ok - unsafe > 1) {
          const int mid = unsafe + (ok - unsafe) / 2;
          if (safe(mid)) {
            ok = mid;
          } else {
            unsafe = mid;
          }
        }
        kf = grid[ok];
      }
    }
    k_final[mb] = kf;
    cov_drop[mb] = __dadd_rn(cb, -coverage_seq(acc, width, kf));
    sh_kf = kf;
  }
  __syncthreads();
  const int kf = sh_kf;
  for (int s = s0 + threadIdx.x; s < s1; s += blockDim.x) k_seq[s] = min(kf, blk_off[s + 1] - blk_off[s]);
}

}  // namespace
}  // namespace sbk

SB_API int sb_dst_decide(const double* profile, const int32_t* blk_off, const int32_t* cu_seqlens, int nb_max,
                         const int32_t* mb_off, int n_mb, const int32_t* k_base, const int32_t* k_anchor,
                         const int32_t* bottleneck, const int32_t* grid, int ngrid, double threshold_p,
                         int32_t* k_final, double* coverage_drop, int32_t* k_seq, void* stream) {
  return sbk::abi_call([&] {
    sbk::require(ngrid >= 1, "ngrid must be >= 1");
    sbk::require(nb_max >= 1 && nb_max <= sbk::kDstMaxWidth, "nb_max must be in [1, 4096]");
    sbk::require(threshold_p >= 0.0 && threshold_p <= 1.0, "threshold_p must be in [0, 1]");
    if (n_mb == 0) return;
    sbk::require(profile && blk_off && cu_seqlens && mb_off && k_base && k_anchor && bottleneck && grid && k_final &&
                     coverage_drop && k_seq,
                 "null pointer");
    sbk::launch(sbk::dst_decide_kernel, n_mb, sbk::kDstThreads, 0, static_cast<cudaStream_t>(stream), 
        profile, blk_off, cu_seqlens, nb_max, mb_off, k_base, k_anchor, bottleneck, grid, ngrid, threshold_p, k_final,
        coverage_drop, k_seq);
    sbk::launched("sb_dst_decide");
  });
}
