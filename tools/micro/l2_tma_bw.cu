// L2 -> SM throughput through TMA, the operand path of the GEMM kernels: one CTA per SM, one
// thread keeping S 2-D box loads (128 rows x 128 B, SWIZZLE_128B: a K1 / K6 operand box) in
// flight into a ring of shared-memory stages, over a buffer small enough to stay in L2.
//   mode 0: every CTA walks the same boxes (shared operand tiles, as in a GEMM wave)
//   mode 1: CTA c starts at box 97 c (mostly distinct boxes at any moment)
//   mode 2: as 1, over a [rows, 7168 B] matrix: each box row is a 128-B piece of a 7168-B row (the
//           GEMMs' operand boxes: K-major A rows, token rows of X and dY)
// Prints TB/s and bytes per SM clock (chip-wide).  Build: see tools/micro/README or
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o l2_tma_bw l2_tma_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

constexpr int kBox = 128 * 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int S>
__global__ void __launch_bounds__(32, 1) stream_boxes(const __grid_constant__ CUtensorMap map, int iters, int nbox,
                                                      int mode, unsigned long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[S];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < S; ++i)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int start = mode == 0 ? 0 : (97 * blockIdx.x) % nbox;
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters + S; ++i) {
    const int st = i % S;
    if (i >= S) {  // the load issued S iterations ago has landed
      const uint32_t par = ((i / S) - 1) & 1;
      asm volatile(
          "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
              smem_u32(&full[st])),
          "r"(par)
          : "memory");
    }
    if (i < iters) {
      const int box = (start + i) % nbox;
      const int bx = mode == 2 ? (box % 56) * 128 : 0, by = mode == 2 ? (box / 56) * 128 : box * 128;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[st])), "r"(kBox)
                   : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              smem_u32(ring + st * kBox)),
          "l"(&map), "r"(bx), "r"(by), "r"(smem_u32(&full[st]))
          : "memory");
    }
  }
  cyc[blockIdx.x] = clock64() - t0;
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int mb = argc > 2 ? atoi(argv[2]) : 32;  // buffer MB (L2-resident when well under 126)
  const int iters = 4096;
  int nbox = (mb << 20) / kBox;
  if (mode == 2) nbox -= nbox % 56;  // whole 7168-B rows
  uint8_t* buf;
  cudaMalloc(&buf, static_cast<size_t>(nbox) * kBox);
  cudaMemset(buf, 1, static_cast<size_t>(nbox) * kBox);
  // the buffer as a [nbox * 128 rows, 128 B] u8 matrix, boxes of 128 x 128 B, 128B swizzle
  CUtensorMap map;
  const cuuint64_t dims[2] = {mode == 2 ? 7168u : 128u,
                              static_cast<cuuint64_t>(nbox) * 128 / (mode == 2 ? 56 : 1)};
  const cuuint64_t strides[1] = {mode == 2 ? 7168u : 128u};
  const cuuint32_t box[2] = {128, 128}, es[2] = {1, 1};
  if (cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * sizeof(unsigned long long));
  auto run = [&](auto kern, int stages) {
    const int smem = stages * kBox + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int w = 0; w < 2; ++w) kern<<<sms, 32, smem>>>(map, iters, nbox, mode, cyc);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<sms, 32, smem>>>(map, iters, nbox, mode, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long* h = new unsigned long long[sms];
    cudaMemcpy(h, cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
    const double bytes = static_cast<double>(sms) * iters * kBox;
    printf("mode %d buffer %3d MB stages %2d: %6.2f TB/s, %6.0f B/clk chip-wide (SM clock %4.0f MHz from clock64)%s\n",
           mode, mb, stages, bytes / (ms * 1e-3) / 1e12, bytes / mx, mx / (ms * 1e3),
           cudaGetLastError() == cudaSuccess ? "" : " ERROR");
    delete[] h;
  };
  run(stream_boxes<4>, 4);
  run(stream_boxes<8>, 8);
  run(stream_boxes<12>, 12);
  return 0;
}
