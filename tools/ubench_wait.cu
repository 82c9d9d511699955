// Microbenchmark (not product code): cost that a warp waiting on an mbarrier imposes on a
// compute warp sharing its SM sub-partition, for several wait implementations.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2604_13847_b200/csrc/kernels/sm100.cuh"
using namespace sbk::sm100;

__device__ __forceinline__ bool try_wait_plain(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}

__global__ void k(int mode, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, mbar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&mbar, 1); fence_barrier_init(); }
  if (warp == 7) tmem_alloc<512>(&tbase);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp == 0 && mode >= 9) {  // TMEM-load warp (SMSP 0): lanes 0..31 of TMEM, columns 256..
    const unsigned long long t0 = clock64();
    uint32_t acc = 0;
    for (int i = 0; i < iters / 4; ++i) {
      uint32_t v[32];
      tmem_ld32(tmem + 256 + (i & 3) * 32, v);
      tmem_wait_ld();
      acc += v[lane & 31] ^ v[0];
    }
    const unsigned long long t1 = clock64();
    if (lane == 0) { out[0] = t1 - t0; mbar_arrive(&bar); }
    if (acc == 1234u) out[1] = 1;
  } else if (warp == 0) {  // compute warp (SMSP 0)
    float x0 = lane, x1 = lane + 1, x2 = lane + 2, x3 = lane + 3, x4 = 1.f, x5 = 2.f, x6 = 3.f, x7 = 4.f;
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll 16
      for (int e = 0; e < 64; ++e) {
        x0 = fmaf(x0, 0.999f, 0.001f); x1 = fmaf(x1, 0.999f, 0.001f); x2 = fmaf(x2, 0.999f, 0.001f);
        x3 = fmaf(x3, 0.999f, 0.001f); x4 = fmaf(x4, 0.999f, 0.001f); x5 = fmaf(x5, 0.999f, 0.001f);
        x6 = fmaf(x6, 0.999f, 0.001f); x7 = fmaf(x7, 0.999f, 0.001f);
      }
    }
    const unsigned long long t1 = clock64();
    if (lane == 0) {
      out[0] = t1 - t0;
      mbar_arrive(&bar);
    }
    if (x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == 1234.f) out[1] = 1;
  } else if ((mode == 6 && warp == 4) || (mode == 7 && warp == 5) || (mode == 8 && warp == 4) ||
             (mode == 10 && warp == 4) || (mode == 11 && warp == 5)) {
    // UMMA issuer: a long stream of 128x128x16 SS MMAs (queue always full); mode 6 same SMSP
    // as the compute warp, 7 another SMSP, 8 same SMSP but single-lane issue.
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const uint32_t idesc = idesc_bf16_f32(128, 128, false, false);
    const uint32_t leader = elect_one();
    for (int i = 0; i < 6000; ++i) {
      if (mode == 8) {
        if (lane == 0) mma_ss(tmem, desc_sw128(a + (i & 3) * 32, 16, 1024), desc_sw128(b + (i & 3) * 32, 16, 1024), idesc, i > 0);
      } else {
        mma_ss(tmem, desc_sw128(a + (i & 3) * 32, 16, 1024), desc_sw128(b + (i & 3) * 32, 16, 1024), idesc, i > 0, leader);
      }
    }
    if (mode == 8) { if (lane == 0) tc_commit(&mbar); } else { tc_commit(&mbar, leader); }
    mbar_wait(&mbar, 0);
  } else if (warp == 4 && mode > 0 && mode < 6) {  // waiter on the same SMSP (warp 4 % 4 == 0)
    if (mode == 1) { while (!mbar_try_wait_sleep(&bar, 0)) {} }
    else if (mode == 2) { while (!try_wait_plain(&bar, 0)) {} }
    else if (mode == 3) { while (!test_wait(&bar, 0)) {} }
    else if (mode == 4) { while (!test_wait(&bar, 0)) { __nanosleep(256); } }
    else if (mode == 5) { if (lane == 0) { while (!mbar_try_wait_sleep(&bar, 0)) {} } __syncwarp(); }
  }
  tc_fence_before(); __syncthreads();
  if (warp == 7) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 16);
  const char* names[] = {"no waiter", "try_wait + suspend hint (all lanes)", "try_wait plain (all lanes)",
                         "test_wait spin", "test_wait + nanosleep(256)", "try_wait + hint (lane 0 only)",
                         "UMMA issuer, same SMSP (converged)", "UMMA issuer, other SMSP", "UMMA issuer, same SMSP (lane 0)",
                         "TMEM-ld warp alone", "TMEM-ld warp + UMMA issuer same SMSP", "TMEM-ld warp + UMMA issuer other SMSP"};
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int mode = 0; mode < 12; ++mode) {
    k<<<1, 256, 100 * 1024>>>(mode, 2000, d);
    cudaDeviceSynchronize();
    unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("%-40s compute warp cycles %llu\n", names[mode], c);
  }
  return 0;
}
