// Microbenchmark (not product code): per-SM throughput of the softmax instruction mix on B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../paper_2604_13847_b200/csrc/kernels/fastmath.cuh"
using namespace sbk;

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b));
  return r;
}

__device__ __forceinline__ void ex2_h2(float a, float b, float& ra, float& rb) {
  uint32_t h, r;
  asm("cvt.rn.f16x2.f32 %0, %2, %1;" : "=r"(h) : "f"(a), "f"(b));
  asm("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(h));
  asm("{\n\t.reg .f16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\tcvt.f32.f16 %0, lo;\n\tcvt.f32.f16 %1, hi;\n\t}"
      : "=f"(ra), "=f"(rb) : "r"(r));
}

template <int MODE>
__global__ void k(int iters, float seed, unsigned long long* out, float* sink) {
  float x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = seed * (threadIdx.x + i) * -1e-3f;
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (MODE == 0) {  // MUFU ex2
        x[i] = ex2_sfu(x[i]) - 1.0f;
        x[i + 1] = ex2_sfu(x[i + 1]) - 1.0f;
      } else if (MODE == 1) {  // polynomial pair
        f2 p = ex2_poly2(mk2(x[i], x[i + 1]));
        x[i] = p.x - 1.0f;
        x[i + 1] = p.y - 1.0f;
      } else if (MODE == 2) {  // cvt bf16x2
        acc += pack2(x[i], x[i + 1]);
        x[i] += 1.0f;
      } else if (MODE == 3) {  // FFMA2
        f2 p = ffma2(mk2(x[i], x[i + 1]), mk2(0.999f, 0.999f), mk2(0.001f, 0.001f));
        x[i] = p.x;
        x[i + 1] = p.y;
      } else if (MODE == 5) {  // f16x2 MUFU exp2 pair with f32 in/out
        float a, b;
        ex2_h2(x[i], x[i + 1], a, b);
        x[i] = a - 1.0f;
        x[i + 1] = b - 1.0f;
      } else if (MODE == 4) {  // the softmax mix per pair: FFMA2, 2 MUFU (5/8) or poly (3/8), FADD2, cvt
        const int e = i / 2 + it;
        f2 p = ex2_pair(ffma2(mk2(x[i], x[i + 1]), mk2(0.5f, 0.5f), mk2(-1.f, -1.f)), i / 2);
        acc += pack2(p.x, p.y);
        f2 s = fadd2(mk2(x[i], x[i + 1]), p);
        x[i] = s.x - 1.0f;
        x[i + 1] = s.y - 1.0f;
        (void)e;
      }
    }
  }
  const unsigned long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 1234.5f || acc == 77) sink[threadIdx.x] = s + acc;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int warps) {
  unsigned long long* d; float* sink;
  cudaMalloc(&d, 8); cudaMalloc(&sink, 4096);
  const int iters = 4096;
  k<MODE><<<1, warps * 32>>>(iters, 1.0f, d, sink);
  cudaDeviceSynchronize();
  unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double elems = double(iters) * 16 * warps * 32;
  printf("%-28s warps=%2d  %.2f elements/cycle/SM\n", name, warps, elems / c);
}

int main() {
  for (int w : {4, 8, 16}) run<0>("MUFU ex2.approx", w);
  for (int w : {4, 8, 16}) run<1>("poly ex2 (pair)", w);
  for (int w : {4, 8, 16}) run<2>("cvt.rn.bf16x2 (per elem)", w);
  for (int w : {4, 8, 16}) run<3>("FFMA2 (per elem)", w);
  for (int w : {4, 8, 16}) run<4>("softmax mix (per elem)", w);
  for (int w : {4, 8, 16}) run<5>("ex2.approx.f16x2 (f32 io)", w);
  return 0;
}
