// tagg_e4m3.cuh -- e4m3 codes of fp32 quotients x / s without a division per element
// (fp8.py:54-80: q = fl(x / s), then e4m3 round-to-nearest-even, saturating), shared by the
// column-block quantizer (tagg_wgrad.cu) and quantize + dispatch (tagg_quant.cu).
#pragma once

#include <cstdint>

#include "tagg_ptx.cuh"

namespace tagg {

// Reciprocal bounds of a positive scale s: lo = RD(1/s), hi >= (1/s)(1 + 2^-22) (RU(1/s)
// raised by two ulps, or 1/s overflowing to inf).  For every x, RZ(x * lo) <= |RN(x / s)| <=
// RZ(x * hi) in magnitude.
__device__ __forceinline__ void recip_bracket(float s, float& lo, float& hi) {
  lo = __frcp_rd(s);
  const float ru = __frcp_ru(s);
  hi = isinf(ru) ? ru : __uint_as_float(__float_as_uint(ru) + 2u);
}

// e4m3 codes of four quotients x / s (fp8.py:54-80: fp32 x / s, then round to e4m3).  The
// exact fp32 quotient lies between RZ(x * RD(1/s)) and RZ(x * r_hi) with r_hi >= (1/s)(1 + 2^-22)
// (both bounds toward zero, so the bracket holds for either sign); fp32 rounding and the e4m3
// conversion (rn, satfinite) are monotonic, so when both bounds give the same codes those ARE
// the codes of RN(x / s).  Otherwise -- a bound pair straddling an e4m3 rounding midpoint: a few
// per thousand bf16 elements, whose quotients land on a midpoint exactly -- the IEEE division decides.  Two multiplies and a conversion per element
// instead of the ~10-instruction __fdiv_rn.
__device__ __forceinline__ uint32_t e4m3x4_bracket(const float (&v)[4], const float (&rlo)[4],
                                                   const float (&rhi)[4], uint32_t& hi_codes) {
  float l[4], u[4];  // packed FMUL2.RZ: one instruction per pair
  fmul2_rz(l[0], l[1], v[0], v[1], rlo[0], rlo[1]);
  fmul2_rz(l[2], l[3], v[2], v[3], rlo[2], rlo[3]);
  fmul2_rz(u[0], u[1], v[0], v[1], rhi[0], rhi[1]);
  fmul2_rz(u[2], u[3], v[2], v[3], rhi[2], rhi[3]);
  uint16_t a, b, c, d;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(a) : "f"(l[1]), "f"(l[0]));
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(b) : "f"(l[3]), "f"(l[2]));
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(c) : "f"(u[1]), "f"(u[0]));
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(d) : "f"(u[3]), "f"(u[2]));
  hi_codes = static_cast<uint32_t>(c) | (static_cast<uint32_t>(d) << 16);
  return static_cast<uint32_t>(a) | (static_cast<uint32_t>(b) << 16);
}
// Codes of four exact quotients x * (1/s) for a power-of-two s (the MXFP8 recipe).
__device__ __forceinline__ uint32_t e4m3x4_pow2(const float (&v)[4], const float (&r)[4]) {
  float l[4];
  fmul2_rz(l[0], l[1], v[0], v[1], r[0], r[1]);
  fmul2_rz(l[2], l[3], v[2], v[3], r[2], r[3]);
  uint16_t a, b;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(a) : "f"(l[1]), "f"(l[0]));
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(b) : "f"(l[3]), "f"(l[2]));
  return static_cast<uint32_t>(a) | (static_cast<uint32_t>(b) << 16);
}
// The bracket's undecided case (a few per thousand elements: bf16 data over a bf16 column
// maximum puts x / s on or next to an e4m3 midpoint that often): the IEEE division decides.
__device__ __forceinline__ uint32_t e4m3x4_div(const float4 v, const float* s) {
  uint16_t a, b;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(a) : "f"(__fdiv_rn(v.y, s[1])), "f"(__fdiv_rn(v.x, s[0])));
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(b) : "f"(__fdiv_rn(v.w, s[3])), "f"(__fdiv_rn(v.z, s[2])));
  return static_cast<uint32_t>(a) | (static_cast<uint32_t>(b) << 16);
}

}  // namespace tagg
