// Minimal reproducer for the only compute-sanitizer racecheck report on the product kernels: a
// cluster of 2 CTAs, one warp per CTA executes tcgen05.alloc.cta_group::2 (the allocated TMEM
// address is written to the smem slot), then a cluster barrier, then every thread reads the
// slot, then dealloc.  No other shared-memory access exists, so any hazard racecheck reports
// here is the pair-collective alloc's own slot write versus itself.  Mode 1 is the same with
// tcgen05.alloc.cta_group::1 in 1-CTA clusters (reported clean).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int kCG>
__global__ void __cluster_dims__(kCG, 1, 1) alloc_kernel(uint32_t* out) {
  extern __shared__ uint64_t dyn[];  // mode 3: the product kernel's layout -- barriers, then the slot
  __shared__ uint32_t static_slot;
  uint32_t& slot = (out[7] == 3) ? *reinterpret_cast<uint32_t*>(dyn + 16) : static_slot;
  const int warp = threadIdx.x >> 5;
  if (out[7] == 3 && threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dyn + i))));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == (out[7] == 3 ? 1 : 0)) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(&slot));
    if constexpr (kCG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(a) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(a) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = slot;
  if (threadIdx.x == 0) out[blockIdx.x] = t;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == (out[7] == 3 ? 1 : 0)) {
    if constexpr (kCG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 128;" ::"r"(t) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(t) : "memory");
  }
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 2;
  uint32_t* out;
  cudaMalloc(&out, 8 * sizeof(uint32_t));
  cudaMemset(out, 0, 8 * sizeof(uint32_t));
  const uint32_t m3 = static_cast<uint32_t>(mode);
  cudaMemcpy(out + 7, &m3, 4, cudaMemcpyHostToDevice);
  if (mode == 3) {
    cudaFuncSetAttribute(alloc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    alloc_kernel<2><<<2, 384, 200 * 1024>>>(out);
  } else if (mode == 2) {
    alloc_kernel<2><<<2, 128>>>(out);
  } else {
    alloc_kernel<1><<<2, 128>>>(out);
  }
  cudaError_t e = cudaDeviceSynchronize();
  uint32_t h[2];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  printf("cta_group::%d alloc: %s, tmem addresses %u %u\n", mode, cudaGetErrorString(e), h[0], h[1]);
  return e != cudaSuccess;
}
