// Where does tcgen05.mma.cta_group::2 with M=128 put its rows in TMEM?
// Each CTA's A tile (K-major, SW128) encodes its local row m in two one-hot K
// positions: k = m % 16 and k = 16 + m / 16.  B[k][n] = k + 1 for k < 16 and
// 16 * (k - 15) for 16 <= k < 24 (exact e4m3), so D = (m % 16 + 1) + 16 * (m / 16 + 1).
// Prints, per CTA and TMEM lane, the decoded local A row of column 0 (or '.' for 0).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../paper_2508_16584_b200/csrc/tagg_ptx.cuh"
using namespace tagg;

__device__ uint8_t e4m3(float v) {  // exact small values only
  if (v == 0.f) return 0;
  int e = 0;
  float m = v;
  while (m >= 2.f) { m *= 0.5f; ++e; }
  const int mant = static_cast<int>((m - 1.f) * 8.f + 0.5f);
  return static_cast<uint8_t>(((e + 7) << 3) | mant);
}

template <int M>
__global__ void __launch_bounds__(128, 1) probe(float* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;           // 128 rows x 128 B (K-major SW128)
  uint8_t* sB = smem + 16384;   // MN-major: 128 K-rows x 128 B (this CTA's 128 N columns), SW128
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t rank = cluster_ctarank();
  const int tid = threadIdx.x;
  // A: row m, 128 bytes (k = 0..127); SW128: 16-byte chunk c of row m lands at chunk c ^ (m & 7)
  for (int i = tid; i < 128 * 128; i += 128) {
    const int m = i / 128, k = i % 128;
    uint8_t v = 0;
    if (k == m % 16 || k == 16 + m / 16 || k == 24) v = e4m3(1.f);
    const int chunk = k / 16, w = k % 16;
    sA[m * 128 + ((chunk ^ (m & 7)) * 16) + w] = v;
  }
  // B MN-major: K-row k holds this CTA's 128 columns n; value depends on k only
  for (int i = tid; i < 128 * 128; i += 128) {
    const int k = i / 128, n = i % 128;
    float f = 0.f;
    if (k < 16) f = k + 1;
    else if (k < 24) f = 16 * (k - 15);
    else if (k == 24) f = rank ? 256.f : 0.f;  // marks tile columns [128, 256) (this CTA's share)
    const int chunk = n / 16, w = n % 16;
    sB[k * 128 + ((chunk ^ (k & 7)) * 16) + w] = e4m3(f);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (tid < 32) tmem_alloc<2>(&slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (rank == 0 && tid == 0) {
    const uint32_t idesc = idesc_e4m3_f32(M, 256, true);
    const uint64_t ad = umma_desc_sw128(smem_u32(sA), 16, 1024);
    const uint64_t bd = umma_desc_sw128(smem_u32(sB), 16384, 1024);
    mma_f8f6f4<2>(tmem, ad, bd, idesc, 0);  // K = 32: k in [0, 32)
    mma_commit<2>(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  // every warp reads its lane quarter, column 0 and column 128
  uint32_t v[32];
  tmem_ld_32x32b_x32(tmem + ((32 * (tid / 32)) << 16), v);
  tmem_wait_ld_dep(v);
  out[(rank * 128 + tid) * 2 + 0] = __uint_as_float(v[0]);
  tmem_ld_32x32b_x32(tmem + ((32 * (tid / 32)) << 16) + 128, v);
  tmem_wait_ld_dep(v);
  out[(rank * 128 + tid) * 2 + 1] = __uint_as_float(v[0]);
  tc_fence_before();
  cluster_sync();
  if (tid < 32) {
    tc_fence_after();
    tmem_dealloc<2>(tmem, 512);
  }
}

template <int M>
void run() {
  float* d;
  cudaMalloc(&d, 256 * 2 * 4);
  cudaMemset(d, 0, 256 * 2 * 4);
  cudaFuncSetAttribute(probe<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 40000;
  cudaLaunchAttribute attr[1] = {};
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, probe<M>, d);
  const cudaError_t e = cudaDeviceSynchronize();
  float h[512];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("M=%d cta_group::2 %s\n", M, cudaGetErrorString(e));
  for (int r = 0; r < 2; ++r) {
    for (int c = 0; c < 2; ++c) {
      printf("CTA %d col %3d lanes 0..127 -> local A row:", r, c * 128);
      for (int l = 0; l < 128; ++l) {
        const float x = h[(r * 128 + l) * 2 + c];
        if (x == 0.f) { printf(" ."); continue; }
        int xi = static_cast<int>(x);
        const bool upper = xi >= 256;
        if (upper) xi -= 256;
        const int lo = ((xi - 1) % 16), hi = (xi - 1 - lo) / 16 - 1;  // x = lo + 1 + 16 (hi + 1)
        printf(" %d%s", hi * 16 + lo, upper ? "u" : "");
      }
      printf("\n");
    }
  }
  cudaFree(d);
}

int main() {
  run<256>();
  run<128>();
  return 0;
}
