// tagg_pad.cu -- the pad + padded-GEMM baseline's data-movement kernels.
//
// K2 pad (engine.py:369-373): every group is copied into a slot of
// ceil(M_g/128)*128 rows.  Pad rows of A are zero and pad rows of S_A are 1.0.
// K3 unpad (engine.py:399-401): the valid rows of each group are gathered back
// from the padded C.  Both kernels are HBM-bound byte movers: one warp per row,
// 16-byte vector accesses, with the group tables built by a warp prefix sum
// over the DEVICE group sizes (no host sync).
#include <cuda_runtime.h>

#include <cstdint>

#include "tagg.h"

namespace tagg {

// Block-wide tables: row_off[G+1] (unpadded), pad_off[G+1] (padded), size[G].
__device__ void build_pad_tables(const int32_t* gs, int G, int32_t* row_off, int32_t* pad_off,
                                 int32_t* size) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int cr = 0, cp = 0;
    for (int base = 0; base < G; base += 32) {
      const int g = base + lane;
      const int m = (g < G) ? max(0, gs[g]) : 0;
      const int mp = (m + 127) / 128 * 128;
      int im = m, ip = mp;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, im, o);
        const int y = __shfl_up_sync(0xffffffffu, ip, o);
        if (lane >= o) { im += x; ip += y; }
      }
      if (g < G) {
        row_off[g] = cr + im - m;
        pad_off[g] = cp + ip - mp;
        size[g] = m;
      }
      cr += __shfl_sync(0xffffffffu, im, 31);
      cp += __shfl_sync(0xffffffffu, ip, 31);
    }
    if (lane == 0) {
      row_off[G] = cr;
      pad_off[G] = cp;
    }
  }
  __syncthreads();
}

// A row copy by one warp: 4 16-byte vectors per lane in flight (loads first, then stores), so a
// warp keeps 2 KB of reads outstanding instead of one 512-byte wave at a time.
__device__ __forceinline__ void copy_row(uint4* __restrict__ dst, const uint4* __restrict__ src, int vec, int lane) {
  int i = lane;
  for (; i + 96 < vec; i += 128) {
    const uint4 v0 = __ldg(src + i), v1 = __ldg(src + i + 32), v2 = __ldg(src + i + 64), v3 = __ldg(src + i + 96);
    dst[i] = v0;
    dst[i + 32] = v1;
    dst[i + 64] = v2;
    dst[i + 96] = v3;
  }
  for (; i < vec; i += 32) dst[i] = __ldg(src + i);
}

__device__ __forceinline__ int find_group(const int32_t* off, int G, int x) {
  int lo = 0, hi = G - 1;  // largest g with off[g] <= x
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (off[mid] <= x) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(256) pad_groups_kernel(const uint8_t* __restrict__ a, int64_t lda,
                                                         const float* __restrict__ sa,
                                                         const int32_t* __restrict__ gs, int G, int K,
                                                         int kbc, uint8_t* __restrict__ a_pad,
                                                         float* __restrict__ sa_pad,
                                                         int32_t* __restrict__ padded_sizes,
                                                         int64_t m_pad_alloc) {
  extern __shared__ int32_t tabs[];
  int32_t* row_off = tabs;
  int32_t* pad_off = row_off + (G + 1);
  int32_t* size = pad_off + (G + 1);
  build_pad_tables(gs, G, row_off, pad_off, size);
  if (blockIdx.x == 0)
    for (int g = threadIdx.x; g < G; g += blockDim.x) padded_sizes[g] = (size[g] + 127) / 128 * 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int64_t total = pad_off[G] < m_pad_alloc ? pad_off[G] : m_pad_alloc;
  const int vec = K / 16;  // K % 16 == 0
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * nw + warp; p < total; p += static_cast<int64_t>(gridDim.x) * nw) {
    const int g = find_group(pad_off, G, static_cast<int>(p));
    const int local = static_cast<int>(p) - pad_off[g];
    uint4* dst = reinterpret_cast<uint4*>(a_pad + p * K);
    float* dsa = sa_pad + p * kbc;
    if (local < size[g]) {
      const int64_t src_row = row_off[g] + local;
      copy_row(dst, reinterpret_cast<const uint4*>(a + src_row * lda), vec, lane);
      const float* ssa = sa + src_row * kbc;
      for (int i = lane; i < kbc; i += 32) dsa[i] = __ldg(ssa + i);
    } else {
      const uint4 z = make_uint4(0, 0, 0, 0);
      for (int i = lane; i < vec; i += 32) dst[i] = z;
      for (int i = lane; i < kbc; i += 32) dsa[i] = 1.0f;
    }
  }
}

__global__ void __launch_bounds__(256) unpad_rows_kernel(const uint16_t* __restrict__ c_pad,
                                                         const int32_t* __restrict__ gs, int G, int N,
                                                         uint16_t* __restrict__ c, int64_t m_alloc) {
  extern __shared__ int32_t tabs[];
  int32_t* row_off = tabs;
  int32_t* pad_off = row_off + (G + 1);
  int32_t* size = pad_off + (G + 1);
  build_pad_tables(gs, G, row_off, pad_off, size);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int64_t total = row_off[G] < m_alloc ? row_off[G] : m_alloc;
  const int vec = N / 8;  // N % 64 == 0: 2N bytes is a multiple of 16
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * nw + warp; r < total; r += static_cast<int64_t>(gridDim.x) * nw) {
    const int g = find_group(row_off, G, static_cast<int>(r));
    const int64_t src_row = pad_off[g] + (r - row_off[g]);
    const uint4* src = reinterpret_cast<const uint4*>(c_pad + src_row * N);
    copy_row(reinterpret_cast<uint4*>(c + r * N), src, vec, lane);
  }
  (void)size;
}

// 4 CTAs (32 warps) per SM, but no more CTAs than the rows give warps to (one warp per row):
// a launch over a few rows then does not spend its time building 592 CTAs' group tables.
static int grid_for_rows(int64_t rows) {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (rows + 7) / 8;
  return static_cast<int>(want < 1 ? 1 : (want < 4 * n ? want : 4 * n));
}

}  // namespace tagg

extern "C" int64_t tagg_padded_rows_bound(int64_t m_alloc, int G) {
  return m_alloc + static_cast<int64_t>(G) * 127;
}

extern "C" int tagg_pad_groups(const void* a, int64_t lda, const float* sa, const int32_t* group_sizes,
                               int G, int K, void* a_pad, float* sa_pad, int32_t* padded_sizes,
                               int64_t m_pad_alloc, void* stream) {
  if (G < 1 || K < 16 || K % 16 != 0) return TAGG_ERR_CONFIG;
  if (!a || !sa || !group_sizes || !a_pad || !sa_pad || !padded_sizes) return TAGG_ERR_SHAPE;
  if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(a_pad)) & 15u || lda % 16)
    return TAGG_ERR_ALIGNMENT;
  const int kbc = (K + 127) / 128;
  const size_t shm = sizeof(int32_t) * (3 * G + 2);
  if (shm > 48 * 1024) return TAGG_ERR_UNSUPPORTED;
  tagg::pad_groups_kernel<<<tagg::grid_for_rows(m_pad_alloc), 256, shm, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(a), lda, sa, group_sizes, G, K, kbc, static_cast<uint8_t*>(a_pad), sa_pad,
      padded_sizes, m_pad_alloc);
  return cudaGetLastError() == cudaSuccess ? TAGG_OK : TAGG_ERR_CUDA;
}

extern "C" int tagg_unpad_rows(const void* c_pad, const int32_t* group_sizes, int G, int N, void* c,
                               int64_t m_alloc, void* stream) {
  if (G < 1 || N < 64 || N % 64 != 0) return TAGG_ERR_CONFIG;
  if (!c_pad || !group_sizes || !c) return TAGG_ERR_SHAPE;
  if ((reinterpret_cast<uintptr_t>(c_pad) | reinterpret_cast<uintptr_t>(c)) & 15u) return TAGG_ERR_ALIGNMENT;
  const size_t shm = sizeof(int32_t) * (3 * G + 2);
  if (shm > 48 * 1024) return TAGG_ERR_UNSUPPORTED;
  tagg::unpad_rows_kernel<<<tagg::grid_for_rows(m_alloc), 256, shm, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(c_pad), group_sizes, G, N, static_cast<uint16_t*>(c), m_alloc);
  return cudaGetLastError() == cudaSuccess ? TAGG_OK : TAGG_ERR_CUDA;
}
