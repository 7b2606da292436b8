// Exhaustive check of the quantizers' division shortcut: for every bf16 column maximum a
// (positive, finite) -> s = RN(a / 448), r = RN(1 / s), and every bf16 x with |x| <= a,
//   q0 = RN(x * r), e = RN(x - q0 s) (one FMA: exact), q1 = RN(q0 + e r) (one FMA)
// must equal RN(x / s) (__fdiv_rn) -- Markstein's correction step.  Counts fp32 mismatches and
// e4m3 code mismatches; then a random sample of fp32 x / fp32 maxima.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ unsigned long long d_bad32, d_badcode, d_pairs;

__device__ __forceinline__ uint16_t code(float q) {
  uint16_t c;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(c) : "f"(0.0f), "f"(q));
  return c & 0xFF;
}
__device__ __forceinline__ float markstein(float x, float s, float r) {
  const float q0 = __fmul_rn(x, r);
  const float e = __fmaf_rn(-q0, s, x);
  return __fmaf_rn(e, r, q0);
}

__global__ void bf16_all(int a_lo) {
  const uint32_t ab = a_lo + blockIdx.x;  // bf16 bits of the maximum
  const float a = __uint_as_float(ab << 16);
  if (!(a > 0.0f) || isinf(a)) return;
  const float s = __fdiv_rn(a, 448.0f);
  const float r = __frcp_rn(s);
  unsigned long long b32 = 0, bc = 0, n = 0;
  for (uint32_t xb = threadIdx.x; xb < 65536; xb += blockDim.x) {
    const float x = __uint_as_float(xb << 16);
    if (!(fabsf(x) <= a)) continue;
    const float q1 = markstein(x, s, r), qe = __fdiv_rn(x, s);
    b32 += __float_as_uint(q1) != __float_as_uint(qe);
    bc += code(q1) != code(qe);
    ++n;
  }
  atomicAdd(&d_bad32, b32);
  atomicAdd(&d_badcode, bc);
  atomicAdd(&d_pairs, n);
}

__device__ __forceinline__ uint32_t hash(uint32_t v) {
  v ^= v >> 16; v *= 0x7feb352dU; v ^= v >> 15; v *= 0x846ca68bU; v ^= v >> 16;
  return v;
}
__global__ void f32_random(uint32_t seed, int iters) {
  unsigned long long b32 = 0, bc = 0, n = 0;
  uint32_t st = hash(seed ^ (blockIdx.x * 1024 + threadIdx.x));
  for (int i = 0; i < iters; ++i) {
    st = hash(st + 0x9e3779b9u);
    const uint32_t abits = 0x01000000u + (st % 0x7E000000u);  // positive normal
    const float a = __uint_as_float(abits);
    st = hash(st + 0x9e3779b9u);
    // x: uniform bits below a, or a "simple" multiple of a (ratio of small integers)
    float x;
    if (st & 1) {
      x = __uint_as_float(st % (abits + 1u)) * ((st & 2) ? -1.0f : 1.0f);
    } else {
      const float num = static_cast<float>((st >> 2) & 1023), den = 1024.0f;
      x = __fmul_rn(a, num / den);
    }
    const float s = __fdiv_rn(a, 448.0f);
    if (!(s > 1.17549435e-38f)) continue;
    const float r = __frcp_rn(s);
    const float q1 = markstein(x, s, r), qe = __fdiv_rn(x, s);
    b32 += __float_as_uint(q1) != __float_as_uint(qe);
    bc += code(q1) != code(qe);
    ++n;
  }
  atomicAdd(&d_bad32, b32);
  atomicAdd(&d_badcode, bc);
  atomicAdd(&d_pairs, n);
}

int main() {
  unsigned long long z = 0, h[3];
  cudaMemcpyToSymbol(d_bad32, &z, 8); cudaMemcpyToSymbol(d_badcode, &z, 8); cudaMemcpyToSymbol(d_pairs, &z, 8);
  bf16_all<<<0x7F80, 256>>>(0);
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&h[0], d_bad32, 8); cudaMemcpyFromSymbol(&h[1], d_badcode, 8); cudaMemcpyFromSymbol(&h[2], d_pairs, 8);
  printf("bf16 exhaustive: %llu pairs, fp32 mismatches %llu, e4m3 code mismatches %llu\n", h[2], h[0], h[1]);
  cudaMemcpyToSymbol(d_bad32, &z, 8); cudaMemcpyToSymbol(d_badcode, &z, 8); cudaMemcpyToSymbol(d_pairs, &z, 8);
  for (int rep = 0; rep < 8; ++rep) f32_random<<<148 * 16, 256>>>(rep * 7919u + 1u, 4096);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&h[0], d_bad32, 8); cudaMemcpyFromSymbol(&h[1], d_badcode, 8); cudaMemcpyFromSymbol(&h[2], d_pairs, 8);
  printf("fp32 random: %llu pairs, fp32 mismatches %llu, e4m3 code mismatches %llu %s\n", h[2], h[0], h[1],
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  return 0;
}
