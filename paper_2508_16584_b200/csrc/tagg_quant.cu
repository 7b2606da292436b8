// tagg_quant.cu -- the producer side of the padding-free grouped GEMM (SURVEY.md §8f,
// rank 1): 1x128 activation quantization fused with the MoE dispatch permutation,
// writing A / S_A directly in the expert-contiguous, padding-free layout the GEMM
// consumes (no pad rows, no intermediate copy).
//
//   route plan (stable counting sort of the routed rows by expert):
//     Q1 route_hist_kernel  : per chunk of 1024 rows, per-expert counts
//     Q2 route_scan_kernel  : per expert, exclusive prefix over chunks; group sizes
//     Q3 route_rank_kernel  : expert offsets + stable rank inside the chunk
//                             (warp __match_any) -> dest row
//   Q4 quantize_dispatch_kernel: one warp per token; per 128-column tile
//     amax -> s = fl(amax / 448) (1.0 for an all-zero tile) -> codes = e4m3(fl(x / s)),
//     RNE and saturating (fp8.py:54-80, 132-151); the codes and s go to all topk
//     destination rows of the token.
//
// All kernels are HBM- or latency-bound integer/byte work: 16-byte or 8-byte
// vector accesses, warp reductions, no tensor cores.
#include <cuda_runtime.h>

#include <cstdint>

#include "tagg.h"

namespace tagg {

constexpr int kRouteChunk = 256;  // rows per route chunk (one warp ranks a chunk in order)
constexpr int kMaxExperts = 1024;

__global__ void __launch_bounds__(256) route_hist_kernel(const int32_t* __restrict__ eid, int64_t R, int E,
                                                         int32_t* __restrict__ counts, int32_t* __restrict__ err) {
  __shared__ int32_t h[kMaxExperts];
  for (int i = threadIdx.x; i < E; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kRouteChunk;
  for (int i = threadIdx.x; i < kRouteChunk; i += blockDim.x) {
    const int64_t r = r0 + i;
    if (r >= R) break;
    const int e = eid[r];
    if (e < 0 || e >= E) {
      atomicOr(err, 1);
      continue;
    }
    atomicAdd(&h[e], 1);
  }
  __syncthreads();
  // expert-major [E][nchunks]: the per-expert scan reads a contiguous column
  for (int i = threadIdx.x; i < E; i += blockDim.x) counts[static_cast<int64_t>(i) * gridDim.x + blockIdx.x] = h[i];
}

// One warp per expert: lane l owns chunks [l*cpl, (l+1)*cpl) of the expert's contiguous
// count column; a warp scan of the lane sums gives each lane's starting offset and the
// column becomes an exclusive prefix (the expert's rows before each chunk).
// group_sizes[e] = the expert's total.
__global__ void __launch_bounds__(256) route_scan_kernel(int32_t* __restrict__ counts, int nchunks, int E,
                                                         int32_t* __restrict__ group_sizes) {
  const int lane = threadIdx.x & 31;
  const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (e >= E) return;
  int32_t* col = counts + static_cast<int64_t>(e) * nchunks;
  // segments of 1024 chunks: lane l holds chunks [32 l, 32 l + 32) of the segment in
  // registers (all loads in flight at once), one warp scan, then the prefix goes back
  constexpr int kPer = 32;
  int carry = 0;
  for (int seg = 0; seg < nchunks; seg += 32 * kPer) {
    const int c0 = seg + lane * kPer;
    int v[kPer];
    int sum = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      v[i] = c0 + i < nchunks ? col[c0 + i] : 0;
      sum += v[i];
    }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int run = carry + incl - sum;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      if (c0 + i < nchunks) col[c0 + i] = run;
      run += v[i];
    }
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) group_sizes[e] = carry;
}

// One warp per chunk, 32 rows at a time in order: lanes with the same expert find
// each other with __match_any_sync; a lane's rank among them plus the chunk's running
// count for that expert is its stable position.
__global__ void __launch_bounds__(32) route_rank_kernel(const int32_t* __restrict__ eid, int64_t R, int E,
                                                        const int32_t* __restrict__ base,
                                                        const int32_t* __restrict__ group_sizes,
                                                        int32_t* __restrict__ dest) {
  __shared__ int32_t run[kMaxExperts];
  const int lane = threadIdx.x;
  const int c = blockIdx.x;
  // expert offsets: exclusive scan of the group sizes (lane l sums experts [l*epl, (l+1)*epl))
  {
    const int epl = (E + 31) / 32;
    const int e0 = min(E, lane * epl), e1 = min(E, e0 + epl);
    int sum = 0;
    for (int e = e0; e < e1; ++e) sum += group_sizes[e];
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int off = incl - sum;
    for (int e = e0; e < e1; ++e) {
      run[e] = off + base[static_cast<int64_t>(e) * gridDim.x + c];
      off += group_sizes[e];
    }
  }
  __syncwarp();
  const int64_t r0 = static_cast<int64_t>(c) * kRouteChunk;
  // every id of the chunk is loaded up front (8 loads in flight per lane), then ranked in order
  constexpr int kSteps = kRouteChunk / 32;
  int ids[kSteps];
#pragma unroll
  for (int i = 0; i < kSteps; ++i) {
    const int64_t r = r0 + 32 * i + lane;
    ids[i] = r < R ? eid[r] : -1;
  }
#pragma unroll
  for (int i = 0; i < kSteps; ++i) {
    const int64_t r = r0 + 32 * i + lane;
    const bool ok = r < R;
    int e = ids[i];
    if (e >= E) e = -1;  // invalid ids were flagged by route_hist_kernel
    const uint32_t same = __match_any_sync(0xffffffffu, e);
    const int rank = __popc(same & ((1u << lane) - 1u));
    const int leader = __ffs(same) - 1;
    int pos = 0;
    if (ok && e >= 0) pos = run[e] + rank;
    __syncwarp();
    if (ok && e >= 0) {
      dest[r] = pos;
      if (lane == leader) run[e] += __popc(same);
    } else if (ok) {
      dest[r] = -1;  // an id outside [0, E) (e.g. a router's -1 for a dropped token): no row
    }
    __syncwarp();
  }
}

// fp8.py:54-80 encode for one f32 pair: RNE, saturating at +-448, -0 keeps its sign.
__device__ __forceinline__ uint16_t e4m3x2(float lo, float hi) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}

template <bool kBf16>
__global__ void __launch_bounds__(256) quantize_dispatch_kernel(const void* __restrict__ x, int64_t ldx, int64_t T,
                                                                int K, int topk, const int32_t* __restrict__ dest,
                                                                uint8_t* __restrict__ a, int64_t lda,
                                                                float* __restrict__ sa, int32_t* __restrict__ err,
                                                                bool vec, const int32_t* __restrict__ gidx = nullptr,
                                                                const float* __restrict__ gw = nullptr) {
  const int lane = threadIdx.x & 31;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= T) return;
  // gather form (Q5): row t quantizes bf16(gw[t] * x[gidx[t]]) -- K10's rows, never written out
  const int64_t xr = gidx ? static_cast<int64_t>(gidx[t]) : t;
  const float wrow = (gidx && gw) ? gw[t] : 1.0f;
  const bool scaled = gidx != nullptr && gw != nullptr;
  const int kb = (K + 127) / 128;
  int32_t d[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) d[k] = (k < topk) ? (dest ? dest[t * topk + k] : static_cast<int32_t>(t)) : -1;
  bool bad = false;
  // A warp covers 4 tiles per step: lane l holds 16 consecutive columns of tile
  // 4 step + l / 8 (8 lanes per 128-column tile): 32-B loads, 16-B code stores.
  const int sub = lane >> 3, part = lane & 7;
  // Raw 16-byte loads of the next step are issued before the current step is quantized
  // and scattered (2 steps of loads in flight per warp: the kernel is bound by memory
  // parallelism, not bandwidth, at one step).
  constexpr int kRaw = kBf16 ? 2 : 4;
  auto full_at = [&](int tile0) { return vec && (tile0 + sub) * 128 + 16 * part + 15 < K; };
  auto load_raw = [&](int tile0, uint4 (&r)[kRaw]) {
    const int c0 = (tile0 + sub) * 128 + 16 * part;
    const uint4* src = kBf16 ? reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(x) + xr * ldx + c0)
                             : reinterpret_cast<const uint4*>(reinterpret_cast<const float*>(x) + xr * ldx + c0);
#pragma unroll
    for (int j = 0; j < kRaw; ++j) r[j] = __ldcs(src + j);  // read once: stream past L2
  };
  uint4 nxt[kRaw];
  bool nxt_full = full_at(0);
  if (nxt_full) load_raw(0, nxt);
  for (int tile0 = 0; tile0 < kb; tile0 += 4) {
    const int tile = tile0 + sub;
    const int c0 = tile * 128 + 16 * part;
    const bool full16 = nxt_full;
    uint4 cur[kRaw];
#pragma unroll
    for (int j = 0; j < kRaw; ++j) cur[j] = nxt[j];
    nxt_full = tile0 + 4 < kb && full_at(tile0 + 4);
    if (nxt_full) load_raw(tile0 + 4, nxt);
    float v[16];
    if (full16) {
      if constexpr (kBf16) {
        const uint32_t w[8] = {cur[0].x, cur[0].y, cur[0].z, cur[0].w, cur[1].x, cur[1].y, cur[1].z, cur[1].w};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          v[2 * j] = __uint_as_float(w[j] << 16);
          v[2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          v[4 * j] = __uint_as_float(cur[j].x);
          v[4 * j + 1] = __uint_as_float(cur[j].y);
          v[4 * j + 2] = __uint_as_float(cur[j].z);
          v[4 * j + 3] = __uint_as_float(cur[j].w);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        v[j] = 0.0f;
        if (tile < kb && c0 + j < K) {
          if constexpr (kBf16)
            v[j] = __uint_as_float(static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(x)[xr * ldx + c0 + j]) << 16);
          else
            v[j] = reinterpret_cast<const float*>(x)[xr * ldx + c0 + j];
        }
      }
    }
    if (scaled) {
      // K10's value: bf16(fl(w * x)), round to nearest even (cvt.rn.bf16x2)
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        uint32_t pr;
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(pr) : "f"(__fmul_rn(wrow, v[j + 1])), "f"(__fmul_rn(wrow, v[j])));
        v[j] = __uint_as_float(pr << 16);
        v[j + 1] = __uint_as_float(pr & 0xFFFF0000u);
      }
    }
    float amax = 0.0f;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float m = fabsf(v[j]);
      bad |= !(m <= 3.402823466e38f);  // inf or nan: the reference raises InvalidInput
      amax = fmaxf(amax, m);
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const float s = amax > 0.0f ? __fdiv_rn(amax, 448.0f) : 1.0f;
    uint32_t word[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint16_t lo = e4m3x2(__fdiv_rn(v[4 * j], s), __fdiv_rn(v[4 * j + 1], s));
      const uint16_t hi = e4m3x2(__fdiv_rn(v[4 * j + 2], s), __fdiv_rn(v[4 * j + 3], s));
      word[j] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
    }
    if (tile < kb) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (k >= topk) break;
        const int64_t row = d[k];
        if (row < 0) continue;  // dropped / invalid route (route_rank_kernel wrote -1)
        if (full16) {
          *reinterpret_cast<uint4*>(a + row * lda + c0) = make_uint4(word[0], word[1], word[2], word[3]);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (c0 + j < K) a[row * lda + c0 + j] = static_cast<uint8_t>(word[j >> 2] >> (8 * (j & 3)));
        }
        if (part == 0) sa[row * kb + tile] = s;
      }
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, 2);
}

// fp8.py:154-176: one scale per 128x128 block.  One CTA per block (grid: column
// blocks x row blocks x batch), 8 warps x 16 rows, 4 columns per lane: 64 values per
// thread held in registers across the block-wide amax.
template <bool kBf16>
__global__ void __launch_bounds__(256) quantize_blocks_kernel(const void* __restrict__ x, int64_t ldx,
                                                              int64_t batch_stride, int rows, int cols,
                                                              uint8_t* __restrict__ codes, int64_t ldc,
                                                              int64_t codes_batch_stride, float* __restrict__ scales,
                                                              int32_t* __restrict__ err) {
  __shared__ float wmax[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int cb = gridDim.x, rb = gridDim.y;
  const int c = blockIdx.x * 128 + 4 * lane;
  const int r0 = blockIdx.y * 128 + 16 * w;
  const int64_t bx = static_cast<int64_t>(blockIdx.z) * batch_stride;
  float v[16][4];
  float amax = 0.0f;
  bool bad = false;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int r = r0 + i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float f = 0.0f;
      if (r < rows && c + j < cols) {
        const int64_t idx = bx + static_cast<int64_t>(r) * ldx + c + j;
        if constexpr (kBf16)
          f = __uint_as_float(static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(x)[idx]) << 16);
        else
          f = reinterpret_cast<const float*>(x)[idx];
      }
      v[i][j] = f;
      const float m = fabsf(f);
      bad |= !(m <= 3.402823466e38f);
      amax = fmaxf(amax, m);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if (lane == 0) wmax[w] = amax;
  __syncthreads();
  amax = wmax[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) amax = fmaxf(amax, wmax[i]);
  const float s = amax > 0.0f ? __fdiv_rn(amax, 448.0f) : 1.0f;
  const int64_t cbase = static_cast<int64_t>(blockIdx.z) * codes_batch_stride;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int r = r0 + i;
    if (r >= rows) break;
    const uint16_t lo = e4m3x2(__fdiv_rn(v[i][0], s), __fdiv_rn(v[i][1], s));
    const uint16_t hi = e4m3x2(__fdiv_rn(v[i][2], s), __fdiv_rn(v[i][3], s));
    const uint32_t word = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
    uint8_t* dst = codes + cbase + static_cast<int64_t>(r) * ldc + c;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (c + j < cols) dst[j] = static_cast<uint8_t>(word >> (8 * j));
  }
  if (threadIdx.x == 0)
    scales[(static_cast<int64_t>(blockIdx.z) * rb + blockIdx.y) * cb + blockIdx.x] = s;
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, 2);
}

}  // namespace tagg

using namespace tagg;

extern "C" int tagg_quantize_blocks(const void* x, int x_dtype, int64_t batch, int64_t rows, int64_t cols,
                                    int64_t ldx, int64_t x_batch_stride, void* codes, int64_t ldc,
                                    int64_t codes_batch_stride, float* scales, int32_t* err_flag, void* stream) {
  if (x_dtype != TAGG_DTYPE_BF16 && x_dtype != TAGG_DTYPE_F32) return TAGG_ERR_CONFIG;
  if (batch < 0 || rows < 0 || cols < 0 || ldx < cols || ldc < cols) return TAGG_ERR_SHAPE;
  if (batch == 0 || rows == 0 || cols == 0) return TAGG_OK;
  if (!x || !codes || !scales || !err_flag) return TAGG_ERR_SHAPE;
  const int64_t rb = (rows + 127) / 128, cb = (cols + 127) / 128;
  if (rb > 65535 || batch > 65535 || cb >= (int64_t(1) << 31) || rows >= (int64_t(1) << 31)) return TAGG_ERR_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const dim3 grid(static_cast<unsigned>(cb), static_cast<unsigned>(rb), static_cast<unsigned>(batch));
  if (x_dtype == TAGG_DTYPE_BF16)
    quantize_blocks_kernel<true><<<grid, 256, 0, st>>>(x, ldx, x_batch_stride, static_cast<int>(rows),
                                                       static_cast<int>(cols), static_cast<uint8_t*>(codes), ldc,
                                                       codes_batch_stride, scales, err_flag);
  else
    quantize_blocks_kernel<false><<<grid, 256, 0, st>>>(x, ldx, x_batch_stride, static_cast<int>(rows),
                                                        static_cast<int>(cols), static_cast<uint8_t*>(codes), ldc,
                                                        codes_batch_stride, scales, err_flag);
  return cudaGetLastError() == cudaSuccess ? TAGG_OK : TAGG_ERR_CUDA;
}

extern "C" int64_t tagg_route_workspace_ints(int64_t rows, int num_experts) {
  if (rows < 0 || num_experts < 1) return 0;
  return ((rows + kRouteChunk - 1) / kRouteChunk) * num_experts + 1;
}

extern "C" int tagg_route_plan(const int32_t* expert_ids, int64_t rows, int num_experts, int32_t* group_sizes,
                               int32_t* dest_rows, int32_t* workspace, void* stream) {
  if (rows < 0 || num_experts < 1 || num_experts > kMaxExperts) return TAGG_ERR_CONFIG;
  if (!group_sizes || !workspace || (rows > 0 && (!expert_ids || !dest_rows))) return TAGG_ERR_SHAPE;
  if (rows >= (int64_t(1) << 31)) return TAGG_ERR_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nchunks = static_cast<int>((rows + kRouteChunk - 1) / kRouteChunk);
  int32_t* err = workspace + static_cast<int64_t>(nchunks) * num_experts;
  if (cudaMemsetAsync(err, 0, sizeof(int32_t), st) != cudaSuccess) return TAGG_ERR_CUDA;
  if (nchunks == 0) {
    return cudaMemsetAsync(group_sizes, 0, sizeof(int32_t) * num_experts, st) == cudaSuccess ? TAGG_OK
                                                                                           : TAGG_ERR_CUDA;
  }
  route_hist_kernel<<<nchunks, 256, 0, st>>>(expert_ids, rows, num_experts, workspace, err);
  route_scan_kernel<<<num_experts, 32, 0, st>>>(workspace, nchunks, num_experts, group_sizes);
  route_rank_kernel<<<nchunks, 32, 0, st>>>(expert_ids, rows, num_experts, workspace, group_sizes, dest_rows);
  return cudaGetLastError() == cudaSuccess ? TAGG_OK : TAGG_ERR_CUDA;
}

extern "C" int tagg_route_error(const int32_t* workspace, int64_t rows, int num_experts, int32_t* host_flag) {
  if (!workspace || !host_flag || num_experts < 1) return TAGG_ERR_SHAPE;
  const int64_t nchunks = (rows + kRouteChunk - 1) / kRouteChunk;
  return cudaMemcpy(host_flag, workspace + nchunks * num_experts, sizeof(int32_t), cudaMemcpyDeviceToHost) ==
                 cudaSuccess
             ? TAGG_OK
             : TAGG_ERR_CUDA;
}

extern "C" int tagg_quantize_gather_rows(const void* x, int x_dtype, int64_t ldx, const int32_t* index,
                                         const float* row_weights, int64_t rows, int K, void* a, int64_t lda,
                                         float* sa, int32_t* err_flag, void* stream) {
  if (K < 1 || rows < 0) return TAGG_ERR_CONFIG;
  if (x_dtype != TAGG_DTYPE_BF16 && x_dtype != TAGG_DTYPE_F32) return TAGG_ERR_CONFIG;
  if (ldx < K || lda < K) return TAGG_ERR_SHAPE;
  if (rows == 0) return TAGG_OK;
  if (!x || !index || !a || !sa || !err_flag) return TAGG_ERR_SHAPE;
  const int esz = x_dtype == TAGG_DTYPE_BF16 ? 2 : 4;
  const bool vec = !(reinterpret_cast<uintptr_t>(x) % 16) && !((ldx * esz) % 16) &&
                   !(reinterpret_cast<uintptr_t>(a) % 16) && !(lda % 16);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int warps = 8;
  const int64_t blocks = (rows + warps - 1) / warps;
  if (blocks >= (int64_t(1) << 31)) return TAGG_ERR_UNSUPPORTED;
  if (x_dtype == TAGG_DTYPE_BF16)
    quantize_dispatch_kernel<true><<<static_cast<unsigned>(blocks), 32 * warps, 0, st>>>(
        x, ldx, rows, K, 1, nullptr, static_cast<uint8_t*>(a), lda, sa, err_flag, vec, index, row_weights);
  else
    quantize_dispatch_kernel<false><<<static_cast<unsigned>(blocks), 32 * warps, 0, st>>>(
        x, ldx, rows, K, 1, nullptr, static_cast<uint8_t*>(a), lda, sa, err_flag, vec, index, row_weights);
  return cudaGetLastError() == cudaSuccess ? TAGG_OK : TAGG_ERR_CUDA;
}

extern "C" int tagg_quantize_dispatch(const void* x, int x_dtype, int64_t ldx, int64_t tokens, int K, int topk,
                                      const int32_t* dest_rows, void* a, int64_t lda, float* sa, int32_t* err_flag,
                                      void* stream) {
  if (K < 1 || tokens < 0 || topk < 1 || topk > 8) return TAGG_ERR_CONFIG;
  if (x_dtype != TAGG_DTYPE_BF16 && x_dtype != TAGG_DTYPE_F32) return TAGG_ERR_CONFIG;
  if (ldx < K || lda < K) return TAGG_ERR_SHAPE;
  if (tokens == 0) return TAGG_OK;
  if (!x || !a || !sa || !err_flag || (topk > 1 && !dest_rows)) return TAGG_ERR_SHAPE;
  const int esz = x_dtype == TAGG_DTYPE_BF16 ? 2 : 4;
  // vector path: 16-byte loads and 16-byte code stores at column multiples of 16;
  // any other alignment takes the element-wise path
  const bool vec = !(reinterpret_cast<uintptr_t>(x) % 16) && !((ldx * esz) % 16) &&
                   !(reinterpret_cast<uintptr_t>(a) % 16) && !(lda % 16);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int warps = 8;
  const int64_t blocks = (tokens + warps - 1) / warps;
  if (blocks >= (int64_t(1) << 31)) return TAGG_ERR_UNSUPPORTED;
  if (x_dtype == TAGG_DTYPE_BF16)
    quantize_dispatch_kernel<true><<<static_cast<unsigned>(blocks), 32 * warps, 0, st>>>(
        x, ldx, tokens, K, topk, dest_rows, static_cast<uint8_t*>(a), lda, sa, err_flag, vec);
  else
    quantize_dispatch_kernel<false><<<static_cast<unsigned>(blocks), 32 * warps, 0, st>>>(
        x, ldx, tokens, K, topk, dest_rows, static_cast<uint8_t*>(a), lda, sa, err_flag, vec);
  return cudaGetLastError() == cudaSuccess ? TAGG_OK : TAGG_ERR_CUDA;
}
