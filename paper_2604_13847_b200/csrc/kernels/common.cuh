// Shared helpers for the sm_100a kernels and their C ABI.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <stdexcept>
#include <string>

#define SB_API extern "C" __attribute__((visibility("default")))

namespace sbk {

// Error raised for invalid arguments (ABI code 1); anything else maps to code 2.
struct ArgError : std::runtime_error {
  explicit ArgError(const std::string& m) : std::runtime_error(m) {}
};

void set_last_error(const std::string& msg);
void count_launch();

template <typename F>
int abi_call(F&& f) {
  try {
    f();
    return 0;
  } catch (const ArgError& e) {
    set_last_error(e.what());
    return 1;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return 2;
  }
}

inline void require(bool ok, const char* what) {
  if (!ok) throw ArgError(what);
}

inline void cuda_check(cudaError_t e, const char* where) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(where) + ": " + cudaGetErrorString(e));
}

// Check the launch that was just issued and count it.
inline void launched(const char* name) {
  cuda_check(cudaGetLastError(), name);
  count_launch();
}

__device__ __forceinline__ float bf2f(uint16_t h) { return __uint_as_float(static_cast<uint32_t>(h) << 16); }

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

// Sequence owning global block gi (binary search in blk_off[0..nseq]).
__device__ __forceinline__ int seq_of_block(const int32_t* blk_off, int nseq, int gi) {
  int lo = 0, hi = nseq;  // blk_off[lo] <= gi < blk_off[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(blk_off + mid) <= gi) lo = mid; else hi = mid;
  }
  return lo;
}

}  // namespace sbk
