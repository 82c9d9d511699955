// Check (not product code): tcgen05.cp 128x256b from a SWIZZLE_128B K-major tile into TMEM as
// a packed-bf16 UMMA A operand, ordered before a TS UMMA issued by the same thread; and its cost.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../paper_2604_13847_b200/csrc/kernels/sm100.cuh"
using namespace sbk::sm100;

__device__ __forceinline__ void tc_cp_128x256b(uint32_t taddr, uint64_t desc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(desc) : "memory");
}

// SW128 K-major: chunk c (64 elements) at c*rows*128; row r at r*128; 16-byte unit u at ((u ^ (r&7)) * 16).
__device__ __forceinline__ int sw_off(int r, int k, int rows) {
  const int c = k / 64, kk = k % 64, u = kk / 8, e = kk % 8;
  return c * rows * 128 + r * 128 + ((u ^ (r & 7)) * 16) + e * 2;
}

__global__ void k(const __nv_bfloat16* A, const __nv_bfloat16* B, float* C, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sa = sm;           // 128 x 128 (A, SW128)
  uint8_t* sb = sm + 32768;   // 128 x 128 (B, N rows x K, SW128)
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 128 * 128; i += blockDim.x) {
    const int r = i / 128, kk = i % 128;
    *reinterpret_cast<__nv_bfloat16*>(sa + sw_off(r, kk, 128)) = A[i];
    *reinterpret_cast<__nv_bfloat16*>(sb + sw_off(r, kk, 128)) = B[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(sa), b = smem_u32(sb);
    unsigned long long t0 = clock64();
    for (int kk = 0; kk < 8; ++kk)
      tc_cp_128x256b(tmem + 256 + kk * 8, desc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024));
    for (int kk = 0; kk < 8; ++kk)
      mma_ts(tmem, tmem + 256 + kk * 8, desc_sw128(b + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
             idesc_bf16_f32(128, 128, false, false), kk > 0);
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    // cost of 64 copies (64 KB) alone
    for (int rep = 0; rep < 8; ++rep)
      for (int kk = 0; kk < 8; ++kk)
        tc_cp_128x256b(tmem + 320 + kk * 8, desc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024));
    tc_commit(&bar);
    mbar_wait(&bar, 1);
    unsigned long long t2 = clock64();
    // 64 MMAs alone vs 64 MMAs + 16 cps (64 KB) interleaved
    for (int i = 0; i < 64; ++i)
      mma_ts(tmem, tmem + 256 + (i & 7) * 8, desc_sw128(b + ((i & 7) >> 2) * 16384 + (i & 3) * 32, 16, 1024),
             idesc_bf16_f32(128, 128, false, false), 1u);
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t3 = clock64();
    for (int i = 0; i < 64; ++i) {
      mma_ts(tmem, tmem + 256 + (i & 7) * 8, desc_sw128(b + ((i & 7) >> 2) * 16384 + (i & 3) * 32, 16, 1024),
             idesc_bf16_f32(128, 128, false, false), 1u);
      if (i & 3) {} else tc_cp_128x256b(tmem + 384 + ((i >> 2) & 7) * 8, desc_sw128(a + (((i >> 2) & 7) >> 2) * 16384 + ((i >> 2) & 3) * 32, 16, 1024));
    }
    tc_commit(&bar);
    mbar_wait(&bar, 1);
    unsigned long long t4 = clock64();
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
    cyc[3] = t4 - t3;
  }
  __syncthreads();
  tc_fence_after();
  for (int c = 0; c < 4; ++c) {
    uint32_t v[32];
    tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c * 32, v);
    tmem_wait_ld();
    for (int e = 0; e < 32; ++e) C[(warp * 32 + lane) * 128 + c * 32 + e] = __uint_as_float(v[e]);
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

int main() {
  static __nv_bfloat16 ha[128 * 128], hb[128 * 128];
  static float fa[128 * 128], fb[128 * 128], hc[128 * 128];
  for (int i = 0; i < 128 * 128; ++i) {
    fa[i] = __bfloat162float(__float2bfloat16(((i * 37 + 11) % 17 - 8) / 8.0f));
    fb[i] = __bfloat162float(__float2bfloat16(((i * 53 + 5) % 13 - 6) / 4.0f));
    ha[i] = __float2bfloat16(fa[i]); hb[i] = __float2bfloat16(fb[i]);
  }
  __nv_bfloat16 *da, *db; float* dc; unsigned long long* dcy;
  cudaMalloc(&da, sizeof(ha)); cudaMalloc(&db, sizeof(hb)); cudaMalloc(&dc, sizeof(hc)); cudaMalloc(&dcy, 32);
  cudaMemcpy(da, ha, sizeof(ha), cudaMemcpyHostToDevice); cudaMemcpy(db, hb, sizeof(hb), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  k<<<1, 128, 65536 + 1024>>>(da, db, dc, dcy);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hc, dc, sizeof(hc), cudaMemcpyDeviceToHost);
  unsigned long long cy[4]; cudaMemcpy(cy, dcy, 32, cudaMemcpyDeviceToHost);
  printf("64 TS MMAs alone %llu cycles; with 16 interleaved cps %llu cycles\n", cy[2], cy[3]);
  double err = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 128; ++n) {
      double ref = 0;
      for (int kk = 0; kk < 128; ++kk) ref += fa[m * 128 + kk] * fb[n * 128 + kk];
      err = fmax(err, fabs(ref - hc[m * 128 + n]));
    }
  printf("cp+TS UMMA max err %g (%s); cp(32KB)+8 MMAs %llu cycles; 64 cps (256 KB) %llu cycles\n", err,
         cudaGetErrorString(e), cy[0], cy[1]);
  return 0;
}
