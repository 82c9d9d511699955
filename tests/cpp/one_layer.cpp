// Compiled C++ caller of the drop-in boundary (test infrastructure): the role of the reference's
// step driver (simulate_iteration, proj/core/src/sim.cpp:277) with its simulated step replaced by
// the kernels. It plans one optimizer step through the C++ host API (include/sparsebalance/*.hpp:
// generate_samples -> plan_step with SAB + DST), then runs rank 0's first micro-batch through the
// kernel C ABI (include/sb_kernels.h: block pool -> block scores -> top-k at the planned keep
// count -> sparse attention fwd -> bwd) on device memory it owns, and checks every stage against
// the C oracle (oracle/sb_oracle.h). Exit 0 = all checks passed.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../oracle/sb_oracle.h"
#include "sb_kernels.h"
#include "sparsebalance/profile_table.hpp"
#include "sparsebalance/sab.hpp"
#include "sparsebalance/step.hpp"
#include "sparsebalance/workload.hpp"

namespace sb = sparsebalance;

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      return 2;                                                                      \
    }                                                                                \
  } while (0)
#define SB(x)                                                                                \
  do {                                                                                       \
    if ((x) != 0) {                                                                          \
      std::fprintf(stderr, "%s:%d %s failed: %s\n", __FILE__, __LINE__, #x, sb_last_error()); \
      return 2;                                                                              \
    }                                                                                        \
  } while (0)

static uint16_t to_bf16(float f) {  // round to nearest even
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}
static float from_bf16(uint16_t h) {
  uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

template <typename T>
static T* dev_copy(const std::vector<T>& h) {
  T* d = nullptr;
  if (cudaMalloc(&d, std::max<size_t>(1, h.size()) * sizeof(T)) != cudaSuccess) return nullptr;
  cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
  return d;
}
template <typename T>
static std::vector<T> host_copy(const T* d, size_t n) {
  std::vector<T> h(n);
  cudaMemcpy(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost);
  return h;
}

// The bf16 parity rule of tests/tolerance.py: max err <= 2e-2 max|ref|; per (token, head) row
// with norm above 5 % of the largest row norm, ||err_row|| <= 2e-2 ||ref_row||; relative Frobenius < 2e-2.
static bool close_bf16(const char* name, const std::vector<uint16_t>& got, const std::vector<double>& ref, int d) {
  double amax = 0, emax = 0, worst = 0, num = 0, den = 0, rms_max = 0;
  const size_t rows = ref.size() / d;
  std::vector<double> rms(rows, 0.0), rerr(rows, 0.0);
  for (size_t i = 0; i < ref.size(); ++i) {
    const double g = from_bf16(got[i]), e = std::fabs(g - ref[i]);
    if (!std::isfinite(g)) return std::printf("%s: non-finite\n", name), false;
    amax = std::max(amax, std::fabs(ref[i]));
    emax = std::max(emax, e);
    rms[i / d] += ref[i] * ref[i];
    rerr[i / d] += e * e;
    num += e * e;
    den += ref[i] * ref[i];
  }
  for (auto& r : rms) rms_max = std::max(rms_max, r = std::sqrt(r));
  for (size_t r = 0; r < rows; ++r)
    if (rms[r] > 0.05 * rms_max) worst = std::max(worst, std::sqrt(rerr[r]) / rms[r]);
  const double fro = std::sqrt(num / std::max(den, 1e-300));
  const bool ok = emax <= 2e-2 * amax && worst <= 2e-2 && fro < 2e-2;
  std::printf("%-3s max err %.3e (max|ref| %.3e)  worst row rel L2 %.3e  rel Fro %.3e  %s\n", name, emax, amax, worst,
              fro, ok ? "ok" : "FAIL");
  return ok;
}

int main() {
  // ---- host half: plan one step exactly as a reference caller would (C++ API, unchanged names)
  sb::LengthDistributionSpec spec;  // bimodal: short ~ 900, long ~ 5000 tokens
  spec.min_length = 64;
  spec.max_length = 8192;
  spec.short_log_mean = std::log(900.0);
  spec.long_log_mean = std::log(5000.0);
  sb::ConcentrationSpec conc;
  const int kBlock = 128, kLayers = 2, kGbs = 8, kMbs = 2, kDp = 2;
  const auto samples = sb::generate_samples(spec, kGbs, conc, kLayers, kBlock, 7);
  sb::CostModelSpec model;
  model.block_size = kBlock;
  const sb::ProfileTable table = sb::synthesize_table(model, sb::default_length_bins(), sb::default_budget_grid(), 42);
  sb::SparsityEstimator est = sb::make_estimator(sb::default_bin_edges(8192), table.budget_grid, 0.2, 32.0);
  sb::StepSetup setup;
  setup.shape.gbs = kGbs;
  setup.shape.mbs = kMbs;
  setup.shape.dp = kDp;
  setup.num_layers = kLayers;
  setup.dst.threshold_p = 0.1;
  setup.dst.anchor = sb::AnchorStrategy::kMean;
  const sb::StepPlan plan = sb::plan_step(samples, sb::Strategy::kSabDst, setup, table, est, 0);
  const auto& ids = plan.plan.micro_batch_bins.at(0).at(0);
  const int k_final = plan.budgets.at(0).at(0).at(0);
  std::vector<int32_t> cu{0};
  for (std::int64_t id : ids) cu.push_back(cu.back() + static_cast<int32_t>(samples.at(static_cast<size_t>(id)).length));
  const int nseq = static_cast<int>(cu.size()) - 1, T = cu.back();
  std::printf("plan_step: rank 0 micro-batch 0 = %d sequences, %d tokens, layer-0 k_final %d\n", nseq, T, k_final);

  // ---- device half through the kernel C ABI
  const int Hq = 2, Hkv = 2, D = 128;
  std::vector<int32_t> blk(nseq + 1);
  std::vector<int64_t> tri(nseq + 1);
  int nbt = 0, nbm = 0;
  int64_t trit = 0;
  SB(sb_block_layout_host(cu.data(), nseq, kBlock, blk.data(), tri.data(), &nbt, &trit, &nbm));
  std::vector<int32_t> k_seq(nseq);
  for (int s = 0; s < nseq; ++s) k_seq[s] = std::min(k_final, blk[s + 1] - blk[s]);
  const int k_max = *std::max_element(k_seq.begin(), k_seq.end());
  uint64_t lcg = 12345;
  auto rnd = [&] {  // ~N(0,1) from a sum of uniforms
    double a = 0;
    for (int i = 0; i < 4; ++i) {
      lcg = lcg * 6364136223846793005ull + 1442695040888963407ull;
      a += static_cast<double>(lcg >> 11) / 9007199254740992.0;
    }
    return static_cast<float>((a - 2.0) * 1.7320508);
  };
  std::vector<uint16_t> q(size_t(T) * Hq * D), k(size_t(T) * Hkv * D), v(k.size()), dO(q.size());
  for (auto* t : {&q, &k, &v, &dO})
    for (auto& x : *t) x = to_bf16(rnd());
  const float scale = 1.0f / std::sqrt(static_cast<float>(D));

  uint16_t *dq_in = dev_copy(q), *dk_in = dev_copy(k), *dv_in = dev_copy(v), *ddo = dev_copy(dO);
  int32_t *dcu = dev_copy(cu), *dblk = dev_copy(blk), *dks = dev_copy(k_seq);
  int64_t* dtri = dev_copy(tri);
  float *qbar, *kbar, *S, *lse;
  int32_t *idx, *cnt;
  uint16_t *o, *ores, *gq, *gk, *gv;
  CK(cudaMalloc(&qbar, size_t(nbt) * Hq * D * 4));
  CK(cudaMalloc(&kbar, size_t(nbt) * Hkv * D * 4));
  CK(cudaMalloc(&S, size_t(Hq) * std::max<int64_t>(1, trit) * 4));
  CK(cudaMalloc(&idx, size_t(Hq) * nbt * k_max * 4));
  CK(cudaMalloc(&cnt, size_t(Hq) * nbt * 4));
  CK(cudaMalloc(&o, q.size() * 2));
  CK(cudaMalloc(&ores, q.size() * 2));
  CK(cudaMalloc(&lse, size_t(Hq) * T * 4));
  CK(cudaMalloc(&gq, q.size() * 2));
  CK(cudaMalloc(&gk, k.size() * 2));
  CK(cudaMalloc(&gv, v.size() * 2));
  void *wf, *wb;
  CK(cudaMalloc(&wf, std::max<size_t>(16, sb_sparse_attn_fwd_workspace_size(nbt, Hq, k_max))));
  CK(cudaMalloc(&wb, std::max<size_t>(16, sb_sparse_attn_bwd_workspace_size(T, nbt, Hq, Hkv, D, Hq, k_max))));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  SB(sb_block_pool(dq_in, dcu, dblk, nseq, nbt, Hq, D, kBlock, qbar, st));
  SB(sb_block_pool(dk_in, dcu, dblk, nseq, nbt, Hkv, D, kBlock, kbar, st));
  SB(sb_block_scores(qbar, kbar, dblk, dtri, nseq, nbm, Hq, Hkv, D, scale, S, st));
  SB(sb_topk_select(S, dblk, dtri, nseq, nbt, nbm, Hq, 1, dks, k_max, 1, idx, cnt, st));
  SB(sb_sparse_attn_fwd_ex(dq_in, dk_in, dv_in, dcu, dblk, nseq, T, nbt, Hq, Hkv, D, kBlock, idx, cnt, Hq, k_max,
                           scale, o, ores, lse, wf, st));
  SB(sb_sparse_attn_bwd_ex(dq_in, dk_in, dv_in, o, ores, ddo, lse, dcu, dblk, nseq, T, nbt, Hq, Hkv, D, kBlock, idx, cnt,
                           Hq, k_max, scale, gq, gk, gv, wb, st, 0));
  CK(cudaStreamSynchronize(st));

  // ---- oracle checks
  bool ok = true;
  const auto hS = host_copy(S, size_t(Hq) * trit);
  std::vector<double> rqb(size_t(nbt) * Hq * D), rkb(size_t(nbt) * Hkv * D), rS(size_t(Hq) * trit);
  orc_block_pool(q.data(), cu.data(), blk.data(), nseq, Hq, D, kBlock, rqb.data());
  orc_block_pool(k.data(), cu.data(), blk.data(), nseq, Hkv, D, kBlock, rkb.data());
  orc_block_scores(rqb.data(), rkb.data(), blk.data(), tri.data(), nseq, Hq, Hkv, D, scale, rS.data());
  double smax = 0, serr = 0;
  for (size_t i = 0; i < rS.size(); ++i) {
    smax = std::max(smax, std::fabs(rS[i]));
    serr = std::max(serr, std::fabs(hS[i] - rS[i]) - 1e-4 * std::fabs(rS[i]));
  }
  const bool s_ok = serr <= 1e-5 * smax;
  std::printf("scores  %s (fp32 1e-4 rule)\n", s_ok ? "ok" : "FAIL");
  ok &= s_ok;
  const auto hidx = host_copy(idx, size_t(Hq) * nbt * k_max);
  const auto hcnt = host_copy(cnt, size_t(Hq) * nbt);
  std::vector<int32_t> ridx(hidx.size()), rcnt(hcnt.size());
  orc_topk_select(hS.data(), blk.data(), tri.data(), nseq, Hq, 1, k_seq.data(), k_max, 1, ridx.data(), rcnt.data());
  const bool sel_ok = ridx == hidx && rcnt == hcnt;
  std::printf("selection %s (bit-exact)\n", sel_ok ? "ok" : "FAIL");
  ok &= sel_ok;
  std::vector<double> ro(q.size()), rl(size_t(Hq) * T), rdq(q.size()), rdk(k.size()), rdv(v.size());
  orc_sparse_attn_fwd(q.data(), k.data(), v.data(), cu.data(), blk.data(), nseq, T, Hq, Hkv, D, kBlock, hidx.data(),
                      hcnt.data(), Hq, k_max, scale, ro.data(), rl.data());
  orc_sparse_attn_bwd(q.data(), k.data(), v.data(), ro.data(), dO.data(), rl.data(), cu.data(), blk.data(), nseq, T,
                      Hq, Hkv, D, kBlock, hidx.data(), hcnt.data(), Hq, k_max, scale, rdq.data(), rdk.data(),
                      rdv.data());
  ok &= close_bf16("O", host_copy(o, q.size()), ro, D);
  ok &= close_bf16("dQ", host_copy(gq, q.size()), rdq, D);
  ok &= close_bf16("dK", host_copy(gk, k.size()), rdk, D);
  ok &= close_bf16("dV", host_copy(gv, v.size()), rdv, D);
  std::printf("one_layer %s\n", ok ? "ok" : "FAILED");
  return ok ? 0 : 1;
}
