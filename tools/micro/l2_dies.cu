// Does B200's L2 cache a line once chip-wide, or once per die?  Every CTA streams the same
// buffer (all CTAs read all of it, ld.global.cg: L2 only).  ncu dram__bytes_read.sum then
// reads ~1x the buffer if the two dies' L2 halves share a line, ~2x if each die fetches its own
// copy.  Mode 1: only CTAs on SMs with %smid < 74 read; mode 2: only %smid even.  Also prints
// the %smid of each CTA's first and the GPC layout hint (%nsmid).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void stream_all(const uint4* __restrict__ buf, size_t n16, uint4* sink, int mode, int* smids) {
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) smids[blockIdx.x] = static_cast<int>(smid);
  if (mode == 1 && smid >= 74) return;
  if (mode == 2 && (smid & 1)) return;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (size_t i = threadIdx.x; i < n16; i += blockDim.x) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(buf + i));
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x12345678) sink[blockIdx.x] = acc;
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const size_t bytes = static_cast<size_t>(argc > 2 ? atoi(argv[2]) : 32) << 20;
  uint4 *buf, *sink;
  int* smids;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 148 * sizeof(uint4));
  cudaMalloc(&smids, 148 * sizeof(int));
  cudaMemset(buf, 1, bytes);
  // evict: touch a 512 MB buffer
  void* big;
  cudaMalloc(&big, 512u << 20);
  cudaMemset(big, 0, 512u << 20);
  cudaDeviceSynchronize();
  stream_all<<<148, 512>>>(buf, bytes / 16, sink, mode, smids);
  cudaDeviceSynchronize();
  int h[148];
  cudaMemcpy(h, smids, sizeof(h), cudaMemcpyDeviceToHost);
  printf("mode %d, %zu MB buffer; smid of blocks 0..15:", mode, bytes >> 20);
  for (int i = 0; i < 16; ++i) printf(" %d", h[i]);
  printf("\n");
  return 0;
}
