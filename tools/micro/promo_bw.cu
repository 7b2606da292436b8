// Microbenchmark: the promotion drain in isolation.  W warps per CTA read a
// 128-lane x 256-column fp32 TMEM buffer per "k-block" (128 KB, what one CTA of
// the 256x256 pair tile drains per 128-K block) and fold it into independent
// fp32 accumulators with FFMA2, exactly like the GEMM's promotion warps.
// Variants: DEPTH x32 loads issued before each tcgen05.wait::ld, optionally
// software-pipelined (next group in flight while the current one is promoted).
// Target: <= 512 clk per k-block (the MMA time of a 256x256x128 pair step).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2508_16584_b200/csrc/tagg_ptx.cuh"
using namespace tagg;

template <int W, int CPT, int DEPTH, bool PIPE>
__global__ void __launch_bounds__(32 * W, 1) promo(int iters, unsigned long long* cycles, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<1>(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = slot + ((32 * (warp & 3)) << 16) + (warp >> 2) * CPT;
  float acc[CPT];
#pragma unroll
  for (int i = 0; i < CPT; ++i) acc[i] = 0.f;
  __syncthreads();
  const unsigned long long t0 = clock64();
  constexpr int kGroups = CPT / (32 * DEPTH);
  for (int it = 0; it < iters; ++it) {
    const uint32_t taddr = base + (it & 1) * 256;
    const float s = 1.0f + 1e-7f * it;
    if constexpr (!PIPE) {
#pragma unroll
      for (int g = 0; g < kGroups; ++g) {
        uint32_t v[DEPTH][32];
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) tmem_ld_32x32b_x32(taddr + 32 * (g * DEPTH + d), v[d]);
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) tmem_wait_ld_dep(v[d]);
#pragma unroll
        for (int d = 0; d < DEPTH; ++d)
#pragma unroll
          for (int i = 0; i < 32; i += 2)
            ffma2(acc[32 * (g * DEPTH + d) + i], acc[32 * (g * DEPTH + d) + i + 1], __uint_as_float(v[d][i]),
                  __uint_as_float(v[d][i + 1]), s);
      }
    } else {
      uint32_t va[DEPTH][32], vb[DEPTH][32];
#pragma unroll
      for (int d = 0; d < DEPTH; ++d) tmem_ld_32x32b_x32(taddr + 32 * d, va[d]);
#pragma unroll
      for (int d = 0; d < DEPTH; ++d) tmem_wait_ld_dep(va[d]);
#pragma unroll
      for (int g = 0; g < kGroups; ++g) {
        uint32_t(&cur)[DEPTH][32] = (g & 1) ? vb : va;
        uint32_t(&nxt)[DEPTH][32] = (g & 1) ? va : vb;
        if (g + 1 < kGroups) {
#pragma unroll
          for (int d = 0; d < DEPTH; ++d) tmem_ld_32x32b_x32(taddr + 32 * ((g + 1) * DEPTH + d), nxt[d]);
        }
#pragma unroll
        for (int d = 0; d < DEPTH; ++d)
#pragma unroll
          for (int i = 0; i < 32; i += 2)
            ffma2(acc[32 * (g * DEPTH + d) + i], acc[32 * (g * DEPTH + d) + i + 1], __uint_as_float(cur[d][i]),
                  __uint_as_float(cur[d][i + 1]), s);
        if (g + 1 < kGroups) {
#pragma unroll
          for (int d = 0; d < DEPTH; ++d) tmem_wait_ld_dep(nxt[d]);
        }
      }
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  float x = 0.f;
#pragma unroll
  for (int i = 0; i < CPT; ++i) x += acc[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = x;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<1>(slot, 512);
  }
}

// single-warp latency of one x32 load + wait
__global__ void lat(int iters, unsigned long long* cycles, float* sink) {
  __shared__ uint32_t slot;
  tmem_alloc<1>(&slot, 512);
  tc_fence_before();
  __syncwarp();
  tc_fence_after();
  float acc = 0.f;
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t v[32];
    tmem_ld_32x32b_x32(slot + (it & 7) * 32 + (__float_as_uint(acc) & 0), v);
    tmem_wait_ld_dep(v);
    acc += __uint_as_float(v[it & 31]) * 0.f;
  }
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  sink[threadIdx.x] = acc;
  tc_fence_before();
  __syncwarp();
  tc_fence_after();
  tmem_dealloc<1>(slot, 512);
}

static unsigned long long* g_cyc;
static float* g_sink;

template <int W, int CPT, int DEPTH, bool PIPE>
void run(const char* name) {
  const int iters = 4096;
  promo<W, CPT, DEPTH, PIPE><<<148, 32 * W>>>(iters, g_cyc, g_sink);
  cudaDeviceSynchronize();
  promo<W, CPT, DEPTH, PIPE><<<148, 32 * W>>>(iters, g_cyc, g_sink);
  const cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, g_cyc, sizeof(h), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double bytes = 32.0 * W * CPT * 4;  // per iteration per CTA
  const double per = double(mx) / iters * (131072.0 / bytes);
  printf("%-34s W=%2d CPT=%3d depth=%d pipe=%d : %7.1f clk per 128 KB  %6.1f B/clk/SM %s\n", name, W, CPT, DEPTH, PIPE,
         per, 131072.0 / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  cudaMalloc(&g_cyc, 148 * 8);
  cudaMalloc(&g_sink, 148 * 1024 * 4);
  {
    lat<<<1, 32>>>(1024, g_cyc, g_sink);
    cudaDeviceSynchronize();
    lat<<<1, 32>>>(1024, g_cyc, g_sink);
    cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, g_cyc, 8, cudaMemcpyDeviceToHost);
    printf("x32 ld+wait latency (1 warp): %.1f clk\n", double(h) / 1024);
  }
  run<8, 128, 1, false>("8 warps x32 serial");
  run<8, 128, 1, true>("8 warps x32 pipelined (kernel today)");
  run<8, 128, 2, false>("8 warps 2x x32 per wait");
  run<8, 128, 2, true>("8 warps 2x x32 pipelined");
  run<8, 128, 4, false>("8 warps 4x x32 per wait");
  run<16, 64, 1, false>("16 warps x32 serial");
  run<16, 64, 1, true>("16 warps x32 pipelined");
  run<16, 64, 2, false>("16 warps 2x x32 per wait");
  run<16, 64, 2, true>("16 warps 2x x32 pipelined");
  run<12, 64, 1, true>("12 warps x 64 cols pipelined");
  run<12, 64, 2, false>("12 warps x 64 cols 2 per wait");
  run<4, 128, 1, true>("4 warps x32 pipelined");
  run<4, 128, 2, true>("4 warps 2x x32 pipelined");
  return 0;
}
