// Per-pair arithmetic shared by the dense (k_update.cu) and gated (k_gate.cu)
// update kernels, so both evaluate bitwise-identical terms
//   u = 2^(-alpha q + log2(p_D c w)) = p_D g(z|x) w          (Eqs 7, 12)
// with packed f32x2 FFMA2/FADD2/FMUL2 and MUFU.EX2 (ex2.approx.ftz).
#pragma once
#include "phd_internal.h"

// pass 2 (dense and gated) folds 1/D_s into the exponent (expo_fold); 0 = multiply by
// d_s (A/B builds)
#ifndef PHD_FOLD_D
#define PHD_FOLD_D 1
#endif

namespace phd {

__device__ __forceinline__ float ex2a(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float2 ex2v(float2 a) { return make_float2(ex2a(a.x), ex2a(a.y)); }
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// Pass-1 exponent: a = -(alpha0 d0^2 + alpha1 d1^2) (log2 units).
// Pass-2 exponent: the same plus lw = log2(p_D c w_i) folded into the last FFMA,
// so that 2^a is directly u = p_D g w (one FMUL per pair saved).
template <int MODEL>
__device__ __forceinline__ float2 expo(float2 d0, float2 d1, float2 na0, float2 na1, float2 base) {
  if (MODEL == kPosIso) {
    float2 q = __fmul2_rn(d0, d0);
    q = __ffma2_rn(d1, d1, q);
    return __ffma2_rn(q, na0, base);
  } else {
    float2 q = __ffma2_rn(__fmul2_rn(d0, d0), na0, base);
    return __ffma2_rn(__fmul2_rn(d1, d1), na1, q);
  }
}

// Pass-2 exponent with 1/D_s folded in (dense pass 2): c = log2(d_s)/na0
// is added to the first squared residual, so 2^e = u d_s = p_D g w / (kappa + C_s) and
// the per-particle weight sum needs one FADD2 instead of an FFMA2 (no d_s operand);
// d_s = 0 (padding, D = 0) gives c = +inf and a term of exactly 0.
template <int MODEL>
__device__ __forceinline__ float2 expo_fold(float2 d0, float2 d1, float2 na0, float2 na1, float2 base, float2 c) {
  if (MODEL == kPosIso) {
    float2 q = __ffma2_rn(d0, d0, c);
    q = __ffma2_rn(d1, d1, q);
    return __ffma2_rn(q, na0, base);
  } else {
    float2 q = __ffma2_rn(__ffma2_rn(d0, d0, c), na0, base);
    return __ffma2_rn(__fmul2_rn(d1, d1), na1, q);
  }
}

// Sum of v[0..7] over the 32 lanes of a warp; lane l ends with the total of
// particle l >> 2 (transposed butterfly: 9 SHFL + 9 FADD for 8 values).
__device__ __forceinline__ float transpose_reduce8(float (&v)[8], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float keep = b4 ? v[i + 4] : v[i];
    float send = b4 ? v[i] : v[i + 4];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    float keep = b3 ? v[i + 2] : v[i];
    float send = b3 ? v[i] : v[i + 2];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  {
    float keep = b2 ? v[1] : v[0];
    float send = b2 ? v[0] : v[1];
    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  return v[0];
}

}  // namespace phd
