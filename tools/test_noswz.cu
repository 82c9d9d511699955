// Check (not product code): UMMA SWIZZLE_NONE K-major descriptor semantics for a K=16 slice.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../paper_2604_13847_b200/csrc/kernels/sm100.cuh"
using namespace sbk::sm100;

__device__ __forceinline__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;
  return d;
}

// A, B: [128][16] bf16 row-major in global. Layout in smem: core matrix (rg, kc) at rg*256 + kc*128,
// inside (r%8)*16 + (k%8)*2.
__global__ void k(const __nv_bfloat16* A, const __nv_bfloat16* B, float* C, int variant) {
  __shared__ __align__(1024) uint8_t sa[4096];
  __shared__ __align__(1024) uint8_t sb[4096];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 128 * 16; i += blockDim.x) {
    const int r = i / 16, kk = i % 16;
    const int off = (r / 8) * 256 + (kk / 8) * 128 + (r % 8) * 16 + (kk % 8) * 2;
    *reinterpret_cast<__nv_bfloat16*>(sa + off) = A[i];
    *reinterpret_cast<__nv_bfloat16*>(sb + off) = B[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<128>(&tbase);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    const uint32_t lbo = variant == 0 ? 128 : 256, sbo = variant == 0 ? 256 : 128;
    mma_ss(tmem, desc_none(smem_u32(sa), lbo, sbo), desc_none(smem_u32(sb), lbo, sbo),
           idesc_bf16_f32(128, 128, false, false), 0u);
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < 4; ++c) {
    uint32_t v[32];
    tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c * 32, v);
    tmem_wait_ld();
    for (int e = 0; e < 32; ++e) C[(warp * 32 + lane) * 128 + c * 32 + e] = __uint_as_float(v[e]);
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<128>(tmem); }
}

int main() {
  __nv_bfloat16 ha[128 * 16], hb[128 * 16];
  float fa[128 * 16], fb[128 * 16];
  for (int i = 0; i < 128 * 16; ++i) {
    fa[i] = __bfloat162float(__float2bfloat16(((i * 37) % 17 - 8) / 8.0f));
    fb[i] = __bfloat162float(__float2bfloat16(((i * 53) % 13 - 6) / 4.0f));
    ha[i] = __float2bfloat16(fa[i]); hb[i] = __float2bfloat16(fb[i]);
  }
  __nv_bfloat16 *da, *db; float* dc;
  cudaMalloc(&da, sizeof(ha)); cudaMalloc(&db, sizeof(hb)); cudaMalloc(&dc, 128 * 128 * 4);
  cudaMemcpy(da, ha, sizeof(ha), cudaMemcpyHostToDevice); cudaMemcpy(db, hb, sizeof(hb), cudaMemcpyHostToDevice);
  static float hc[128 * 128];
  for (int variant = 0; variant < 2; ++variant) {
    k<<<1, 128>>>(da, db, dc, variant);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hc, dc, sizeof(hc), cudaMemcpyDeviceToHost);
    double err = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 128; ++n) {
        double ref = 0;
        for (int kk = 0; kk < 16; ++kk) ref += fa[m * 16 + kk] * fb[n * 16 + kk];
        err = fmax(err, fabs(ref - hc[m * 128 + n]));
      }
    printf("variant %d (LBO %d SBO %d): max err %g (%s)\n", variant, variant == 0 ? 128 : 256, variant == 0 ? 256 : 128,
           err, cudaGetErrorString(e));
  }
  return 0;
}
