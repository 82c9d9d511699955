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

// Programmatic dependent launch. Every kernel is launched with programmatic stream
// serialization (launch() below): its grid may be scheduled while the previous kernel in the
// stream is still running, so launch latency and prologues (barrier init, TMEM allocation,
// descriptor prefetch) overlap the predecessor's tail. Each kernel therefore calls pdl_wait()
// before its first global-memory access that may depend on an earlier kernel (the wait returns
// once the predecessor grid has completed and its writes are visible), then pdl_trigger() so its
// own dependent may be scheduled. A successor can only occupy resources that are free, so a
// persistent kernel's successor starts on SMs as its CTAs exit.
__device__ __forceinline__ unsigned long long globaltimer_ns() {  // debug timelines (SM-independent clock)
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...), "cudaLaunchKernelEx");
}

// Opt a kernel into `bytes` of dynamic shared memory once per process (the attribute is sticky;
// calling cudaFuncSetAttribute on every launch puts a driver call on the per-layer host path).
bool smem_attr_needed(const void* kernel, int bytes);  // common.cu: per-kernel record of the set value
void smem_attr_done(const void* kernel, int bytes);
template <typename K>
inline void set_smem_once(K kernel, int bytes, const char* where) {
  const void* key = reinterpret_cast<const void*>(kernel);
  if (!smem_attr_needed(key, bytes)) return;
  cuda_check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), where);
  smem_attr_done(key, bytes);
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

// 64 contiguous output bytes (16 packed words) from one thread: two 256-bit stores
// (STG.256, sm_100) when 32-byte aligned, else four 128-bit stores. Halves the store count of
// the epilogues, whose issue rate bounds the item-boundary time.
__device__ __forceinline__ void store_64B(void* dst, const uint32_t (&w)[16]) {
  if ((reinterpret_cast<uintptr_t>(dst) & 31u) == 0) {
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst), "r"(w[0]), "r"(w[1]),
                 "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                 : "memory");
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(static_cast<char*>(dst) + 32),
                 "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15])
                 : "memory");
  } else {
    uint4* d4 = static_cast<uint4*>(dst);
#pragma unroll
    for (int e = 0; e < 4; ++e) d4[e] = make_uint4(w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
  }
}

// Block size 256 on the B = 128 kernels (expand256.cu): the selection re-expressed over a padded
// 128 layout (blk_off = 2 x the 256 one), nb_total and k_max doubled.
struct Expanded256 {
  int32_t* blk_off;
  int32_t* idx;
  int32_t* cnt;
  int nb_total, k_max;
  size_t used;  // workspace bytes taken from the front
};
size_t expand256_workspace_bytes(int nseq, int nb256, int hsel, int k_max);
Expanded256 expand_selection_256(const int32_t* cu, const int32_t* blk_off256, int nseq, int nb256, int hsel,
                                 const int32_t* idx, const int32_t* cnt, int k_max, uint8_t* ws, cudaStream_t st);

// Debug builds (`make debug`: -DSB_DEBUG_CHECKS) trap on a violated index invariant at the
// kernels' global store sites (compute-sanitizer is not available on the B200 pool).
#ifdef SB_DEBUG_CHECKS
#define SB_DCHECK(cond) \
  do {                  \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define SB_DCHECK(cond) \
  do {                  \
  } while (0)
#endif

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
