// Throughput of the epilogue's fp32 -> bf16x2 conversion on one SM: F2FP.BF16.F32.PACK_AB
// (cvt.rn.bf16x2.f32) against the reference's integer RNE (engine.py:46-50) built from IADD3 /
// LOP3 / PRMT, and a 50/50 mix.  8 warps per CTA, one CTA per SM; clk per conversion pair.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ uint32_t cvt_f2fp(float lo, float hi) {
  uint32_t r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint32_t cvt_int(float lo, float hi) {
  const uint32_t a = __float_as_uint(lo), b = __float_as_uint(hi);
  const uint32_t ra = a + 0x7FFFu + ((a >> 16) & 1u);
  const uint32_t rb = b + 0x7FFFu + ((b >> 16) & 1u);
  return __byte_perm(ra, rb, 0x7632);
}

template <int kMode>
__global__ void kern(const float* in, uint32_t* out, long long* clk, int iters) {
  float x[16];
  for (int i = 0; i < 16; ++i) x[i] = in[threadIdx.x * 16 + i];
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      uint32_t r;
      if (kMode == 0) r = cvt_f2fp(x[i], x[i + 1]);
      else if (kMode == 1) r = cvt_int(x[i], x[i + 1]);
      else r = (i & 2) ? cvt_int(x[i], x[i + 1]) : cvt_f2fp(x[i], x[i + 1]);
      acc ^= r;
      x[i] = __uint_as_float(__float_as_uint(x[i]) + 1u);  // new input each iteration
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
  float* in; uint32_t* out; long long* clk;
  cudaMalloc(&in, 1024 * 16 * 4); cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&clk, 148 * 8);
  cudaMemset(in, 0x3f, 1024 * 16 * 4);
  const int iters = 4096;
  const char* names[3] = {"F2FP (cvt.rn.bf16x2.f32)", "integer RNE (IADD3/LOP3/PRMT)", "50/50 mix"};
  for (int warps : {8, 16}) {
    for (int mode = 0; mode < 3; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) kern<0><<<148, 32 * warps>>>(in, out, clk, iters);
        if (mode == 1) kern<1><<<148, 32 * warps>>>(in, out, clk, iters);
        if (mode == 2) kern<2><<<148, 32 * warps>>>(in, out, clk, iters);
      }
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      const double pairs = double(iters) * 8 * 32 * warps;
      printf("%2d warps  %-32s %7.2f pairs/clk/SM\n", warps, names[mode], pairs / c);
    }
  }
  return 0;
}
