// Bit-exact device restatement of the host libm's tanhf, for the fp32 parity
// tier.  The reference's MLP forward calls std::tanh on float
// (train.cpp:68-79), i.e. glibc's tanhf; glibc 2.39 (this image) implements it
// with the fdlibm algorithm (tanh via expm1f, s_tanhf.c / s_expm1f.c), which
// is not correctly rounded (it differs from round(tanh(x)) on ~5 % of floats
// below 11), so CUDA's tanhf — a different approximation — left a last-ulp
// difference per activation that Adam amplified.  Restated here with every
// operation separately rounded (__fmul_rn / __fadd_rn / __fdiv_rn: no FMA
// contraction) it matches glibc on all 2^32 inputs (checked exhaustively on
// the host against libm, tools/check_tanhf.c).
#pragma once
#include <cstdint>

namespace hzp {

__device__ __forceinline__ float f_of(uint32_t u) { return __uint_as_float(u); }

// fdlibm expm1f restricted to what tanhf calls it with: |x| < 44.
__device__ __forceinline__ float expm1f_fdlibm(float x) {
  const float ln2_hi = f_of(0x3f317180u), ln2_lo = f_of(0x3717f7d1u), invln2 = f_of(0x3fb8aa3bu);
  const float Q1 = f_of(0xbd088889u), Q2 = f_of(0x3ad00d01u), Q3 = f_of(0xb8a670cdu), Q4 = f_of(0x36867e54u),
              Q5 = f_of(0xb457edbbu);
  uint32_t hx = __float_as_uint(x);
  const uint32_t xsb = hx & 0x80000000u;
  hx &= 0x7fffffffu;
  if (hx >= 0x4195b844u && xsb) return -1.0f;  // x <= -27 ln2 (tiny - one rounds to -1)
  float hi, lo, c = 0.f, t;
  int k;
  if (hx > 0x3eb17218u) {  // |x| > ln2 / 2: reduce by k ln2
    if (hx < 0x3f851592u) {
      if (!xsb) { hi = __fsub_rn(x, ln2_hi); lo = ln2_lo; k = 1; }
      else { hi = __fadd_rn(x, ln2_hi); lo = -ln2_lo; k = -1; }
    } else {
      k = __float2int_rz(__fadd_rn(__fmul_rn(invln2, x), xsb ? -0.5f : 0.5f));
      t = static_cast<float>(k);
      hi = __fsub_rn(x, __fmul_rn(t, ln2_hi));
      lo = __fmul_rn(t, ln2_lo);
    }
    x = __fsub_rn(hi, lo);
    c = __fsub_rn(__fsub_rn(hi, x), lo);
  } else if (hx < 0x33000000u) {
    return x;  // |x| < 2^-25
  } else {
    k = 0;
  }
  const float hfx = __fmul_rn(0.5f, x);
  const float hxs = __fmul_rn(x, hfx);
  float r1 = __fmul_rn(hxs, Q5);
  r1 = __fmul_rn(hxs, __fadd_rn(Q4, r1));
  r1 = __fmul_rn(hxs, __fadd_rn(Q3, r1));
  r1 = __fmul_rn(hxs, __fadd_rn(Q2, r1));
  r1 = __fadd_rn(1.f, __fmul_rn(hxs, __fadd_rn(Q1, r1)));
  t = __fsub_rn(3.0f, __fmul_rn(r1, hfx));
  float e = __fmul_rn(hxs, __fdiv_rn(__fsub_rn(r1, t), __fsub_rn(6.0f, __fmul_rn(x, t))));
  if (k == 0) return __fsub_rn(x, __fsub_rn(__fmul_rn(x, e), hxs));
  e = __fsub_rn(__fmul_rn(x, __fsub_rn(e, c)), c);
  e = __fsub_rn(e, hxs);
  if (k == -1) return __fsub_rn(__fmul_rn(0.5f, __fsub_rn(x, e)), 0.5f);
  if (k == 1) {
    if (x < -0.25f) return __fmul_rn(-2.0f, __fsub_rn(e, __fadd_rn(x, 0.5f)));
    return __fadd_rn(1.f, __fmul_rn(2.0f, __fsub_rn(x, e)));
  }
  float y;
  if (k <= -2 || k > 56) {
    y = __fsub_rn(1.f, __fsub_rn(e, x));
    y = f_of(__float_as_uint(y) + (uint32_t(k) << 23));
    return __fsub_rn(y, 1.f);
  }
  if (k < 23) {
    t = f_of(0x3f800000u - (0x1000000u >> k));  // 1 - 2^-k
    y = __fsub_rn(t, __fsub_rn(e, x));
  } else {
    t = f_of(uint32_t(0x7f - k) << 23);  // 2^-k
    y = __fadd_rn(__fsub_rn(x, __fadd_rn(e, t)), 1.f);
  }
  return f_of(__float_as_uint(y) + (uint32_t(k) << 23));
}

// fdlibm tanhf (finite inputs; the GEMM epilogue never sees inf / nan on a
// healthy step, and both return nan for nan).
__device__ __forceinline__ float tanhf_fdlibm(float x) {
  const uint32_t jx = __float_as_uint(x), ix = jx & 0x7fffffffu;
  if (ix >= 0x7f800000u) return ix > 0x7f800000u ? x + x : ((jx >> 31) ? -1.f : 1.f);
  float z;
  if (ix < 0x41b00000u) {  // |x| < 22
    if (ix == 0) return x;
    if (ix < 0x24000000u) return __fmul_rn(x, __fadd_rn(1.f, x));  // |x| < 2^-55
    const float ax = fabsf(x);
    if (ix >= 0x3f800000u) {  // |x| >= 1
      const float t = expm1f_fdlibm(__fmul_rn(2.f, ax));
      z = __fsub_rn(1.f, __fdiv_rn(2.f, __fadd_rn(t, 2.f)));
    } else {
      const float t = expm1f_fdlibm(__fmul_rn(-2.f, ax));
      z = __fdiv_rn(-t, __fadd_rn(t, 2.f));
    }
  } else {
    z = 1.f;  // one - tiny
  }
  return (jx >> 31) ? -z : z;
}

}  // namespace hzp
