// Elementwise math for the softmax stages, written for the sm_100 issue budget.
//
// The softmax warps are issue-bound (one warp per SM sub-partition streams 128 columns per
// key block), so the hot loops use the packed fp32x2 FMA-pipe instructions (FFMA2 / FADD2 /
// FMUL2), the 3-input FMNMX3 for row maxima, and split the exponentials between the SFU
// (MUFU.EX2, 16/clk/SM on B200 -- exactly the UMMA time of a 128x128 tile) and a
// Cody-Waite + degree-3 polynomial on the FMA pipe (max relative error 2.1e-4, far below the
// bf16 rounding of P).
#pragma once

#include <stdint.h>

namespace sbk {

struct f2 {
  float x, y;
};

__device__ __forceinline__ f2 mk2(float a, float b) { return f2{a, b}; }

__device__ __forceinline__ f2 ffma2(f2 a, f2 b, f2 c) {
  f2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

__device__ __forceinline__ f2 fadd2(f2 a, f2 b) {
  f2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

__device__ __forceinline__ f2 fmul2(f2 a, f2 b) {
  f2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

__device__ __forceinline__ float ex2_sfu(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x for a pair: x = j + f, j = rint(x) via the 1.5*2^23 magic-number add (the low mantissa
// bits of x + magic hold j in two's complement), f in [-0.5, 0.5], 2^f by a degree-3
// polynomial, j folded into the exponent field with one shift + add. x is clamped to >= -126
// first so the exponent never wraps: the polynomial is 0.99998866 < 1 at f = 0, so j = -127
// would take the bits below zero (0xffffff42, a NaN) -- every x <= -127 (a score 127 log2
// units under the row max, or a masked -inf) came out NaN. With j >= -126 the result is a
// non-negative float <= 2^-126 (~0 for softmax).
__device__ __forceinline__ f2 ex2_poly2(f2 x) {
  x.x = fmaxf(x.x, -126.0f);
  x.y = fmaxf(x.y, -126.0f);
  const f2 t = fadd2(x, mk2(12582912.0f, 12582912.0f));
  const f2 jf = fadd2(t, mk2(-12582912.0f, -12582912.0f));
  const f2 f = ffma2(jf, mk2(-1.0f, -1.0f), x);
  f2 p = ffma2(mk2(0.054848f, 0.054848f), f, mk2(0.24180661f, 0.24180661f));
  p = ffma2(p, f, mk2(0.6932482f, 0.6932482f));
  p = ffma2(p, f, mk2(0.99998866f, 0.99998866f));
  return mk2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
             __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// Pair e of a row (columns 2e, 2e+1): 3 of every 8 pairs on the FMA pipe. `e` must be a
// compile-time constant after unrolling so the branch disappears.
#ifndef SB_POLY_OF_8
#define SB_POLY_OF_8 3  // exp2 pairs (of every 8) evaluated on the FMA pipe
#endif
__device__ __forceinline__ f2 ex2_pair(f2 x, int e) {
  if ((e & 7) >= 8 - SB_POLY_OF_8) return ex2_poly2(x);
  return mk2(ex2_sfu(x.x), ex2_sfu(x.y));
}
// Same with a per-kernel split: kPoly of every 8 pairs on the FMA pipe. Measured on C2: the
// fwd is fastest at 3 (2: +0.4 %, 4: +2.8 %), the dkv / dq passes at 2 (-0.6 % each vs 3).
template <int kPoly>
__device__ __forceinline__ f2 ex2_pair_n(f2 x, int e) {
  if ((e & 7) >= 8 - kPoly) return ex2_poly2(x);
  return mk2(ex2_sfu(x.x), ex2_sfu(x.y));
}

// Scalar variant used by the (rare) masked paths.
__device__ __forceinline__ float ex2_mixed(float x, int col) {
  if (((col >> 1) & 7) >= 5) return ex2_poly2(mk2(x, x)).x;
  return ex2_sfu(x);
}

}  // namespace sbk
