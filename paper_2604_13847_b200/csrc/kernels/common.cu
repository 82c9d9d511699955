// C ABI plumbing shared by every kernel entry point: last-error string, launch counter and
// the host-side block layout helper.
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "sb_kernels.h"

namespace sbk {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }

namespace {
std::mutex g_attr_mu;
std::unordered_map<const void*, int> g_attr;  // kernel -> dynamic shared memory opted into
}  // namespace

bool smem_attr_needed(const void* kernel, int bytes) {
  std::lock_guard<std::mutex> lk(g_attr_mu);
  const auto it = g_attr.find(kernel);
  return it == g_attr.end() || it->second < bytes;
}

void smem_attr_done(const void* kernel, int bytes) {
  std::lock_guard<std::mutex> lk(g_attr_mu);
  g_attr[kernel] = bytes;
}
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

}  // namespace sbk

SB_API const char* sb_last_error(void) { return sbk::g_last_error.c_str(); }

SB_API uint64_t sb_launch_count(void) { return sbk::g_launches.load(); }

SB_API int sb_block_layout_host(const int32_t* cu, int nseq, int block_size, int32_t* blk_off,
                                int64_t* tri_off, int* nb_total, int64_t* tri_total, int* nb_max) {
  return sbk::abi_call([&] {
    sbk::require(cu != nullptr && blk_off != nullptr && tri_off != nullptr, "null pointer");
    sbk::require(nseq >= 0, "nseq must be >= 0");
    sbk::require(block_size == 64 || block_size == 128 || block_size == 256, "block_size must be 64, 128 or 256");
    sbk::require(nseq == 0 || cu[0] == 0, "cu_seqlens[0] must be 0");
    blk_off[0] = 0;
    tri_off[0] = 0;
    int mx = 0;
    for (int s = 0; s < nseq; ++s) {
      const int len = cu[s + 1] - cu[s];
      sbk::require(len >= 0, "cu_seqlens must be non-decreasing");
      const int nb = (len + block_size - 1) / block_size;
      blk_off[s + 1] = blk_off[s] + nb;
      tri_off[s + 1] = tri_off[s] + static_cast<int64_t>(nb) * (nb + 1) / 2;
      mx = nb > mx ? nb : mx;
    }
    if (nb_total) *nb_total = blk_off[nseq];
    if (tri_total) *tri_total = tri_off[nseq];
    if (nb_max) *nb_max = mx;
  });
}
