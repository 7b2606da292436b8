// Microbenchmark: TMEM -> register read throughput per SM (tcgen05.ld 32x32b, various widths).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2508_16584_b200/csrc/tagg_ptx.cuh"
using namespace tagg;

template <int X>
__device__ __forceinline__ void ld_x(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void ld_x<32>(uint32_t taddr, uint32_t* r) {
  uint32_t (&v)[32] = *reinterpret_cast<uint32_t(*)[32]>(r);
  tmem_ld_32x32b_x32(taddr, v);
}

__global__ void __launch_bounds__(384, 1) tmem_read(int iters, unsigned long long* cycles, float* sink, int nwarps) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<1>(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = slot;
  float acc = 0.f;
  unsigned long long t0 = clock64();
  if (warp < nwarps) {
    const uint32_t q = warp & 3;
    const uint32_t taddr = base + ((32 * q) << 16) + ((warp / 4) * 128) % 512;
    for (int it = 0; it < iters; ++it) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(taddr + (it & 3) * 32, v);
      tmem_wait_ld_dep(v);
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += __uint_as_float(v[i]);
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<1>(base, 512); }
}

int main() {
  unsigned long long* cyc; float* sink;
  cudaMalloc(&cyc, 148 * 8); cudaMalloc(&sink, 148 * 384 * 4);
  const int iters = 4096;
  for (int nw : {4, 8, 12}) {
    tmem_read<<<148, 384>>>(iters, cyc, sink, nw);
    cudaDeviceSynchronize();
    tmem_read<<<148, 384>>>(iters, cyc, sink, nw);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double bytes = double(nw) * iters * 32 * 32 * 4;  // per SM
    printf("warps=%2d  %s  cycles=%llu  TMEM read = %.1f B/clk/SM\n", nw, cudaGetErrorString(e), h[0], bytes / h[0]);
  }
  return 0;
}
