// exp2 for the softmax stages, split between the MUFU (SFU) pipe and the FMA pipe.
//
// On B200 the SFU retires 16 ex2/clk/SM, so exponentiating a 128x128 score tile costs exactly
// as many cycles as the two 128x128x128 UMMAs it sits between. Evaluating a fraction of the
// exponentials with a Cody-Waite + degree-3 polynomial on the FMA pipe (max relative error
// 2.1e-4, far below the bf16 rounding of P) takes the SFU off the critical path.
#pragma once

namespace sbk {

__device__ __forceinline__ float ex2_sfu(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x for x in [-125, 64]: x = j + f with j = rint(x) (via the 1.5*2^23 magic-number add) and
// f in [-0.5, 0.5]; 2^f by a degree-3 polynomial; j folded into the exponent field with one
// shift + add (the low mantissa bits of x + magic hold j in two's complement).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -125.0f);  // keeps the result a normal float (2^-125 ~ 0 for softmax)
  const float magic = 12582912.0f;
  const float t = x + magic;
  const float f = x - (t - magic);
  float p = fmaf(0.054848f, f, 0.24180661f);
  p = fmaf(p, f, 0.6932482f);
  p = fmaf(p, f, 0.99998866f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// Column-interleaved split: 3 of every 8 columns on the FMA pipe. `col` must be a
// compile-time constant after unrolling so the branch disappears.
__device__ __forceinline__ float ex2_mixed(float x, int col) {
  return ((col & 7) >= 5) ? ex2_poly(x) : ex2_sfu(x);
}

}  // namespace sbk
