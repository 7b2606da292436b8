// Microbenchmark: TMEM -> register read throughput per SM.
// tcgen05.ld.32x32b.x{32,64,128}, W warps per CTA (W/4 per SMSP), D loads in flight per warp.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2508_16584_b200/csrc/tagg_ptx.cuh"
using namespace tagg;

__device__ __forceinline__ void ld64(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
      "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
        "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]),
        "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]),
        "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]),
        "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
}

// MODE 0: x32, one in flight.  MODE 1: x32, two in flight (pipelined).  MODE 2: x64, one in flight.
// MODE 3: x32 x4 issued back to back, one wait (4 in flight).
template <int MODE>
__global__ void __launch_bounds__(512, 1) tmem_read(int iters, unsigned long long* cycles, float* sink, int nwarps) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<1>(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = slot;
  float acc = 0.f;
  __syncthreads();
  unsigned long long t0 = clock64();
  if (warp < nwarps) {
    const uint32_t taddr = base + ((32 * (warp & 3)) << 16) + ((warp >> 2) * 128) % 512;
    if (MODE == 0) {
      for (int it = 0; it < iters; ++it) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(taddr + (it & 3) * 32, v);
        tmem_wait_ld_dep(v);
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += __uint_as_float(v[i]);
      }
    } else if (MODE == 1) {
      uint32_t va[32], vb[32];
      tmem_ld_32x32b_x32(taddr, va);
      tmem_wait_ld_dep(va);
      for (int it = 0; it < iters; it += 2) {
        tmem_ld_32x32b_x32(taddr + 32, vb);
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += __uint_as_float(va[i]);
        tmem_wait_ld_dep(vb);
        tmem_ld_32x32b_x32(taddr + 64, va);
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += __uint_as_float(vb[i]);
        tmem_wait_ld_dep(va);
      }
    } else if (MODE == 2) {
      for (int it = 0; it < iters; it += 2) {
        uint32_t v[64];
        ld64(taddr + (it & 2) * 32, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 64; ++i) acc += __uint_as_float(v[i]);
      }
    } else {
      for (int it = 0; it < iters; it += 4) {
        uint32_t v0[32], v1[32], v2[32], v3[32];
        tmem_ld_32x32b_x32(taddr, v0);
        tmem_ld_32x32b_x32(taddr + 32, v1);
        tmem_ld_32x32b_x32(taddr + 64, v2);
        tmem_ld_32x32b_x32(taddr + 96, v3);
        tmem_wait_ld_dep(v0); tmem_wait_ld_dep(v1); tmem_wait_ld_dep(v2); tmem_wait_ld_dep(v3);
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += __uint_as_float(v0[i]) + __uint_as_float(v1[i]) + __uint_as_float(v2[i]) + __uint_as_float(v3[i]);
      }
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

template <int MODE>
void run(const char* name) {
  unsigned long long* cyc; float* sink;
  cudaMalloc(&cyc, 148 * 8); cudaMalloc(&sink, 148 * 512 * 4);
  const int iters = 2048;
  for (int nw : {4, 8, 12, 16}) {
    tmem_read<MODE><<<148, 512>>>(iters, cyc, sink, nw);
    cudaDeviceSynchronize();
    tmem_read<MODE><<<148, 512>>>(iters, cyc, sink, nw);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double bytes = double(nw) * iters * 32 * 32 * 4;
    printf("%-18s warps=%2d %s  TMEM read = %6.1f B/clk/SM\n", name, nw, e == cudaSuccess ? "" : cudaGetErrorString(e), bytes / h[0]);
  }
  cudaFree(cyc); cudaFree(sink);
}

int main() {
  run<0>("x32 depth1");
  run<1>("x32 depth2");
  run<2>("x64 depth1");
  run<3>("x32x4 one wait");
  return 0;
}
