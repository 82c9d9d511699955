// K6 placeholder (replaced by the tcgen05 backward).
#include "common.cuh"
#include "sb_kernels.h"

SB_API size_t sb_sparse_attn_bwd_workspace_size(int, int, int, int, int, int, int) { return 0; }

SB_API int sb_sparse_attn_bwd(const uint16_t*, const uint16_t*, const uint16_t*, const uint16_t*, const uint16_t*,
                              const float*, const int32_t*, const int32_t*, int, int, int, int, int, int, int,
                              const int32_t*, const int32_t*, int, int, float, uint16_t*, uint16_t*, uint16_t*, void*,
                              void*) {
  return sbk::abi_call([&] { throw std::runtime_error("sb_sparse_attn_bwd: not built yet"); });
}
