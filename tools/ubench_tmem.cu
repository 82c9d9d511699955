// Microbenchmark (not product code): tcgen05 SS-MMA throughput and tcgen05.ld bandwidth on one SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2604_13847_b200/csrc/kernels/sm100.cuh"
using namespace sbk::sm100;

__global__ void __launch_bounds__(320, 1) bench(int mode, int iters, int nwarps_ld, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 1) tmem_alloc<512>(&tmem_base);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tmem_base;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  unsigned long long t0 = clock64(), t1 = t0;
  if (mode == 0) {  // back-to-back SS MMAs M=128 N=128 K=16 (x iters), one thread
    if (threadIdx.x == 32) {
      const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
      const uint32_t idesc = idesc_bf16_f32(128, 128, false, false);
      for (int i = 0; i < iters; ++i) {
        mma_ss(tmem, desc_sw128(a + (i & 3) * 32, 16, 1024), desc_sw128(b + (i & 3) * 32, 16, 1024), idesc, i > 0);
      }
      tc_commit(&bar);
      mbar_wait(&bar, 0);
      t1 = clock64();
      out[2] = t1 - t0;
    }
  } else if (mode == 1) {  // TS MMAs: A from TMEM cols 128.., B from smem, N=128
    if (threadIdx.x == 32) {
      const uint32_t b = smem_u32(smem + 32768);
      const uint32_t idesc = idesc_bf16_f32(128, 128, false, true);
      for (int i = 0; i < iters; ++i)
        mma_ts(tmem, tmem + 256 + (i & 7) * 8, desc_sw128(b + (i & 7) * 2048, 128 * 128, 1024), idesc, i > 0);
      tc_commit(&bar);
      mbar_wait(&bar, 0);
      t1 = clock64();
      out[2] = t1 - t0;
    }
  } else if (mode == 4 || mode == 6) {  // N=64 MMAs: TS (mode 4) / SS (mode 6)
    if (threadIdx.x == 32) {
      const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
      const uint32_t idesc = idesc_bf16_f32(128, 64, false, false);
      for (int i = 0; i < iters; ++i) {
        if (mode == 4)
          mma_ts(tmem, tmem + 256 + (i & 7) * 8, desc_sw128(b + (i & 3) * 32, 16, 1024), idesc, i > 0);
        else
          mma_ss(tmem, desc_sw128(a + (i & 3) * 32, 16, 1024), desc_sw128(b + (i & 3) * 32, 16, 1024), idesc, i > 0);
      }
      tc_commit(&bar);
      mbar_wait(&bar, 0);
      t1 = clock64();
      out[2] = t1 - t0;
    }
  } else if (mode == 5) {  // TS MMA N=128 while nwarps_ld warps stream tcgen05.ld of other columns
    if (threadIdx.x == 32) {
      const uint32_t b = smem_u32(smem + 32768);
      const uint32_t idesc = idesc_bf16_f32(128, 128, false, true);
      for (int i = 0; i < iters; ++i)
        mma_ts(tmem, tmem + 256 + (i & 7) * 8, desc_sw128(b + (i & 7) * 2048, 128 * 128, 1024), idesc, i > 0);
      tc_commit(&bar);
      mbar_wait(&bar, 0);
      t1 = clock64();
      out[2] = t1 - t0;
    } else if (warp >= 2 && warp < 2 + nwarps_ld) {
      const uint32_t lf = static_cast<uint32_t>((warp & 3) * 32) << 16;
      uint32_t acc = 0;
      for (int i = 0; i < iters / 4; ++i) {
        uint32_t v[2][32];
#pragma unroll
        for (int c = 0; c < 2; ++c) tmem_ld32(tmem + lf + 128 + ((warp - 2) / 4) * 64 + c * 32, v[c]);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int e = 0; e < 32; e += 8) acc ^= v[c][e];
      }
      if (acc == 0xdeadbeef) out[1] = acc;
      unsigned long long t2 = clock64();
      if (lane == 0) atomicMax(out + 3, t2 - t0);
    }
  } else if (mode == 7 || mode == 8) {  // SS MMA N=64 rotating over 4 accumulators (7) / N=256 (8)
    if (threadIdx.x == 32) {
      const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
      const uint32_t idesc = idesc_bf16_f32(128, mode == 7 ? 64 : 256, false, false);
      for (int i = 0; i < iters; ++i) {
        const uint32_t d = mode == 7 ? (i & 3) * 64 : 0;
        mma_ss(tmem + d, desc_sw128(a + (i & 3) * 32, 16, 1024), desc_sw128(b + (i & 3) * 32, 16, 1024), idesc,
               i > 3);
      }
      tc_commit(&bar);
      mbar_wait(&bar, 0);
      t1 = clock64();
      out[2] = t1 - t0;
    }
  } else if (mode == 9 || mode == 10) {  // TS (A at cols 256..) then SS writing cols 256.. (9, WAR) / 384.. (10)
    if (threadIdx.x == 32) {
      const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
      const uint32_t idesc_ss = idesc_bf16_f32(128, 128, false, false);
      const uint32_t idesc_ts = idesc_bf16_f32(128, 128, false, true);
      const uint32_t dst = mode == 9 ? 256 : 384;
      for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(tmem, tmem + 256 + (kk & 3) * 8, desc_sw128(b + (kk & 7) * 2048, 128 * 128, 1024), idesc_ts, i > 0 || kk > 0);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ss(tmem + dst, desc_sw128(a + (kk & 3) * 32, 16, 1024), desc_sw128(b + (kk & 3) * 32, 16, 1024), idesc_ss,
                 kk > 0);
      }
      tc_commit(&bar);
      mbar_wait(&bar, 0);
      t1 = clock64();
      out[2] = t1 - t0;
    }
  } else if (mode == 2) {  // tcgen05.ld bandwidth: nwarps_ld warps read 128 columns each, iters times
    if (warp >= 2 && warp < 2 + nwarps_ld) {
      const uint32_t lf = static_cast<uint32_t>((warp & 3) * 32) << 16;
      uint32_t acc = 0;
      for (int i = 0; i < iters; ++i) {
        uint32_t v[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(tmem + lf + ((warp - 2) / 4) * 128 + c * 32, v[c]);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int e = 0; e < 32; e += 8) acc ^= v[c][e];
      }
      if (acc == 0xdeadbeef) out[1] = acc;
      t1 = clock64();
      if (lane == 0) atomicMax(out + 2, t1 - t0);
    }
  } else if (mode == 3) {  // tcgen05.st bandwidth
    if (warp >= 2 && warp < 2 + nwarps_ld) {
      const uint32_t lf = static_cast<uint32_t>((warp & 3) * 32) << 16;
      uint32_t v[32];
      for (int e = 0; e < 32; ++e) v[e] = e + lane;
      for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 2; ++c) tmem_st32(tmem + lf + ((warp - 2) / 4) * 64 + c * 32, v);
        tmem_wait_st();
      }
      t1 = clock64();
      if (lane == 0) atomicMax(out + 2, t1 - t0);
    }
  }
  __syncthreads();
  tc_fence_before(); __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 32);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  auto run = [&](int mode, int iters, int nw, const char* name, double bytes_or_flop, const char* unit) {
    cudaMemset(d, 0, 32);
    bench<<<1, 320, 100 * 1024>>>(mode, iters, nw, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c = 0; cudaMemcpy(&c, d + 2, 8, cudaMemcpyDeviceToHost);
    printf("%-40s iters=%6d warps=%d cycles=%10llu  %.1f %s/cycle  (%s)\n", name, iters, nw, c, bytes_or_flop / c, unit,
           cudaGetErrorString(e));
  };
  for (int it : {64, 512, 4096}) run(0, it, 0, "SS MMA 128x128x16", 2.0 * 128 * 128 * 16 * it, "FLOP");
  for (int it : {64, 512, 4096}) run(1, it, 0, "TS MMA 128x128x16", 2.0 * 128 * 128 * 16 * it, "FLOP");
  for (int it : {512, 4096}) run(4, it, 0, "TS MMA 128x64x16", 2.0 * 128 * 64 * 16 * it, "FLOP");
  for (int it : {512, 4096}) run(6, it, 0, "SS MMA 128x64x16", 2.0 * 128 * 64 * 16 * it, "FLOP");
  for (int it : {512, 4096}) run(7, it, 0, "SS MMA 128x64x16, 4 accumulators", 2.0 * 128 * 64 * 16 * it, "FLOP");
  for (int it : {512, 4096}) run(8, it, 0, "SS MMA 128x256x16", 2.0 * 128 * 256 * 16 * it, "FLOP");
  for (int it : {64, 512}) run(9, it, 0, "8 TS + 8 SS overwriting TS A (WAR)", 2.0 * 128 * 128 * 16 * 16 * it, "FLOP");
  for (int it : {64, 512}) run(10, it, 0, "8 TS + 8 SS, disjoint", 2.0 * 128 * 128 * 16 * 16 * it, "FLOP");
  for (int nw : {0, 4, 8}) run(5, 4096, nw, "TS MMA 128x128x16 + ld warps", 2.0 * 128 * 128 * 16 * 4096, "FLOP");
  for (int nw : {4, 8}) for (int it : {64, 1024}) run(2, it, nw, "tcgen05.ld 32x32b.x32 (128 cols)", 1.0 * nw * 32 * 128 * 4 * it, "B");
  for (int nw : {4, 8}) for (int it : {64, 1024}) run(3, it, nw, "tcgen05.st 32x32b.x32 (64 cols)", 1.0 * nw * 32 * 64 * 4 * it, "B");
  return 0;
}
