// tagg_moe.cu -- the two HBM-bound steps that close an MoE FFN around the padding-free GEMM:
//
//   K7 swiglu_quantize_kernel: gate|up GEMM output (grouped rows, bf16 [M, 2I]) ->
//      h = silu(gate) * up in fp32 (fast exp / division, a few ulp) -> the 1x128 FP8 recipe
//      of fp8.py:132-151 (amax -> s = fl(amax/448) -> e4m3(h * fl(1/s)), RNE, saturating;
//      the reciprocal in place of the recipe's division) -> the down GEMM's A and S_A, in the
//      same padding-free grouped rows (no permutation, no pad rows).  Rows past sum(M_g)
//      are not touched (the group sizes stay on the device).
//   K8 combine_kernel: down GEMM output (grouped rows, bf16 [R, N]) -> per token
//      out[t] = bf16( sum_k fl(w[t,k] * c[dest[t*topk+k]]) ) accumulated in fp32 in k order,
//      separately rounded (no FMA), so a CPU restatement reproduces it bit for bit.
//
// Both are memory-bound byte/float work: 16-byte vector accesses, one warp per row (K7) or
// one CTA per token (K8), no tensor cores.
#include <cuda_runtime.h>

#include <cstdint>

#include "tagg.h"

namespace tagg {
namespace moe {

__device__ __forceinline__ uint16_t e4m3x2(float lo, float hi) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// silu(g) * u in fp32: g / (1 + e^-g) with the fast ex2-based exp and an approximate
// division (a few ulp; the result is quantized to 3 mantissa bits next).  The accurate
// expf + IEEE division made the kernel compute-bound at 6x its HBM time.
__device__ __forceinline__ float swiglu(float g, float u) { return __fdividef(g, 1.0f + __expf(-g)) * u; }

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// One warp per row; lane l holds 16 consecutive columns of tile 4 step + l / 8.
__global__ void __launch_bounds__(256) swiglu_quantize_kernel(const uint16_t* __restrict__ h, int64_t ldh,
                                                              const int32_t* __restrict__ group_sizes, int G,
                                                              int64_t m_alloc, int I, uint8_t* __restrict__ a,
                                                              int64_t lda, float* __restrict__ sa,
                                                              int32_t* __restrict__ err, uint16_t* __restrict__ vout,
                                                              int64_t ldv) {
  const int lane = threadIdx.x & 31;
  // rows in use = sum of the device group sizes (every warp reduces them; G is small)
  int64_t total = 0;
  for (int g = lane; g < G; g += 32) total += max(0, group_sizes[g]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
  total = min(total, m_alloc);
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= total) return;
  const int kb = (I + 127) / 128;
  const int sub = lane >> 3, part = lane & 7;
  const uint16_t* hg = h + row * ldh;  // gate: columns [0, I)
  const uint16_t* hu = hg + I;         // up:   columns [I, 2I)
  bool bad = false;
  for (int tile0 = 0; tile0 < kb; tile0 += 4) {
    const int tile = tile0 + sub;
    const int c0 = tile * 128 + 16 * part;
    float v[16];
    if (tile < kb && c0 + 15 < I) {
      const uint4* pg = reinterpret_cast<const uint4*>(hg + c0);
      const uint4* pu = reinterpret_cast<const uint4*>(hu + c0);
      const uint4 g0 = pg[0], g1 = pg[1], u0 = pu[0], u1 = pu[1];
      const uint32_t gw[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
      const uint32_t uw[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        v[2 * j] = swiglu(bf16_lo(gw[j]), bf16_lo(uw[j]));
        v[2 * j + 1] = swiglu(bf16_hi(gw[j]), bf16_hi(uw[j]));
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        v[j] = (tile < kb && c0 + j < I) ? swiglu(__uint_as_float(static_cast<uint32_t>(hg[c0 + j]) << 16),
                                                  __uint_as_float(static_cast<uint32_t>(hu[c0 + j]) << 16))
                                         : 0.0f;
    }
    float amax = 0.0f;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float m = fabsf(v[j]);
      bad |= !(m <= 3.402823466e38f);
      amax = fmaxf(amax, m);
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const float s = amax > 0.0f ? __fdiv_rn(amax, 448.0f) : 1.0f;
    // v * (1/s) instead of the recipe's IEEE v / s: v is itself a few ulp off (fast exp),
    // and the IEEE division sequence made this kernel issue-bound (79 instructions per
    // element); the two differ by at most one fp32 ulp before the 3-bit rounding
    const float inv = __frcp_rn(s);
    uint32_t word[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint16_t lo = e4m3x2(__fmul_rn(v[4 * j], inv), __fmul_rn(v[4 * j + 1], inv));
      const uint16_t hi = e4m3x2(__fmul_rn(v[4 * j + 2], inv), __fmul_rn(v[4 * j + 3], inv));
      word[j] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
    }
    if (vout && tile < kb && c0 + 15 < I) {  // v itself, bf16 (saved for the backward's wgrad)
      uint32_t o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = pack_bf16(v[2 * j], v[2 * j + 1]);
      uint4* q = reinterpret_cast<uint4*>(vout + row * ldv + c0);
      q[0] = make_uint4(o[0], o[1], o[2], o[3]);
      q[1] = make_uint4(o[4], o[5], o[6], o[7]);
    }
    if (tile < kb) {
      uint8_t* dst = a + row * lda + c0;
      if (c0 + 15 < I) {
        *reinterpret_cast<uint4*>(dst) = make_uint4(word[0], word[1], word[2], word[3]);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (c0 + j < I) dst[j] = static_cast<uint8_t>(word[j >> 2] >> (8 * (j & 3)));
      }
      if (part == 0) sa[row * kb + tile] = s;
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, 2);
}

// K9 (backward of K7): from the saved gate|up rows h = [g | u] and the gradient dh of
// v = silu(g) * u:  dg = dh * u * sig(g) * (1 + g * (1 - sig(g))),  du = dh * silu(g).
// Writes d[g | u] as bf16 (for the wgrad column quantizer) and row-quantized 1x128 FP8
// (codes + scales: the A operand of the gate|up dgrad GEMM).  One warp per row; the
// dg and du halves are quantized as separate 128-column tiles (I % 128 == 0).
__device__ __forceinline__ void quantize16(const float (&v)[16], float& s, uint32_t (&word)[4], bool& bad) {
  float amax = 0.0f;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const float m = fabsf(v[j]);
    bad |= !(m <= 3.402823466e38f);
    amax = fmaxf(amax, m);
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  s = amax > 0.0f ? __fdiv_rn(amax, 448.0f) : 1.0f;
  const float inv = __frcp_rn(s);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint16_t lo = e4m3x2(__fmul_rn(v[4 * j], inv), __fmul_rn(v[4 * j + 1], inv));
    const uint16_t hi = e4m3x2(__fmul_rn(v[4 * j + 2], inv), __fmul_rn(v[4 * j + 3], inv));
    word[j] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
  }
}

__global__ void __launch_bounds__(256) swiglu_backward_kernel(const uint16_t* __restrict__ h, int64_t ldh,
                                                              const uint16_t* __restrict__ dh, int64_t lddh,
                                                              const int32_t* __restrict__ group_sizes, int G,
                                                              int64_t m_alloc, int I, uint16_t* __restrict__ dgu,
                                                              int64_t lddgu, uint8_t* __restrict__ a, int64_t lda,
                                                              float* __restrict__ sa, int32_t* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  int64_t total = 0;
  for (int g = lane; g < G; g += 32) total += max(0, group_sizes[g]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
  total = min(total, m_alloc);
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= total) return;
  const int kbi = I / 128;  // tiles per half
  const int sub = lane >> 3, part = lane & 7;
  bool bad = false;
  for (int tile0 = 0; tile0 < kbi; tile0 += 4) {
    const int tile = tile0 + sub;
    // an 8-lane group past the last tile computes on zeros and stores nothing (the warp's
    // shuffles need every lane)
    const bool active = tile < kbi;
    const int c0 = (active ? tile : 0) * 128 + 16 * part;
    const uint4* pg = reinterpret_cast<const uint4*>(h + row * ldh + c0);
    const uint4* pu = reinterpret_cast<const uint4*>(h + row * ldh + I + c0);
    const uint4* pd = reinterpret_cast<const uint4*>(dh + row * lddh + c0);
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
    const uint4 g0 = active ? pg[0] : z, g1 = active ? pg[1] : z, u0 = active ? pu[0] : z,
                u1 = active ? pu[1] : z, d0 = active ? pd[0] : z, d1 = active ? pd[1] : z;
    const uint32_t gw[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    const uint32_t uw[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
    const uint32_t dw[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
    float vg[16], vu[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float g = (j & 1) ? bf16_hi(gw[j >> 1]) : bf16_lo(gw[j >> 1]);
      const float u = (j & 1) ? bf16_hi(uw[j >> 1]) : bf16_lo(uw[j >> 1]);
      const float d = (j & 1) ? bf16_hi(dw[j >> 1]) : bf16_lo(dw[j >> 1]);
      const float sig = __fdividef(1.0f, 1.0f + __expf(-g));
      vg[j] = d * u * sig * (1.0f + g * (1.0f - sig));
      vu[j] = d * g * sig;
    }
    float sg, su;
    uint32_t wg[4], wu[4];
    quantize16(vg, sg, wg, bad);
    quantize16(vu, su, wu, bad);
    if (!active) continue;
    *reinterpret_cast<uint4*>(a + row * lda + c0) = make_uint4(wg[0], wg[1], wg[2], wg[3]);
    *reinterpret_cast<uint4*>(a + row * lda + I + c0) = make_uint4(wu[0], wu[1], wu[2], wu[3]);
    if (part == 0) {
      sa[row * (2 * kbi) + tile] = sg;
      sa[row * (2 * kbi) + kbi + tile] = su;
    }
    if (dgu) {
      uint32_t og[8], ou[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        og[j] = pack_bf16(vg[2 * j], vg[2 * j + 1]);
        ou[j] = pack_bf16(vu[2 * j], vu[2 * j + 1]);
      }
      uint4* qg = reinterpret_cast<uint4*>(dgu + row * lddgu + c0);
      uint4* qu = reinterpret_cast<uint4*>(dgu + row * lddgu + I + c0);
      qg[0] = make_uint4(og[0], og[1], og[2], og[3]);
      qg[1] = make_uint4(og[4], og[5], og[6], og[7]);
      qu[0] = make_uint4(ou[0], ou[1], ou[2], ou[3]);
      qu[1] = make_uint4(ou[4], ou[5], ou[6], ou[7]);
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, 2);
}

// K10: out[r] = bf16(w[r] * src[idx[r]]) -- rows of a token matrix gathered into the grouped
// layout and scaled (the backward's dL/dc = w[t,k] * dy[t]); one warp per row, 16-B vectors.
__global__ void __launch_bounds__(256) gather_scale_rows_kernel(const uint16_t* __restrict__ src, int64_t lds,
                                                                const int32_t* __restrict__ idx,
                                                                const float* __restrict__ w, int64_t R, int H,
                                                                uint16_t* __restrict__ out, int64_t ldo) {
  const int lane = threadIdx.x & 31;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= R) return;
  const uint16_t* s = src + static_cast<int64_t>(idx[r]) * lds;
  const float wr = w ? w[r] : 1.0f;
  for (int c = 8 * lane; c < H; c += 256) {
    const uint4 q = *reinterpret_cast<const uint4*>(s + c);
    const uint32_t qw[4] = {q.x, q.y, q.z, q.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = pack_bf16(__fmul_rn(wr, bf16_lo(qw[j])), __fmul_rn(wr, bf16_hi(qw[j])));
    *reinterpret_cast<uint4*>(out + r * ldo + c) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// K11: g[t, k] = <dy[t], c[dest[t*topk + k]]> in fp32 (the router-weight gradient); one warp
// per (t, k) pair.
__global__ void __launch_bounds__(256) router_grad_kernel(const uint16_t* __restrict__ dy, int64_t lddy,
                                                          const uint16_t* __restrict__ c, int64_t ldc,
                                                          const int32_t* __restrict__ dest, int64_t pairs, int topk,
                                                          int H, float* __restrict__ g) {
  const int lane = threadIdx.x & 31;
  const int64_t p = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (p >= pairs) return;
  if (dest[p] < 0) {  // dropped route (tagg_route_plan wrote -1): no expert output, no gradient
    if (lane == 0) g[p] = 0.0f;
    return;
  }
  const uint16_t* a = dy + (p / topk) * lddy;
  const uint16_t* b = c + static_cast<int64_t>(dest[p]) * ldc;
  float acc = 0.0f;
  for (int col = 8 * lane; col < H; col += 256) {
    const uint4 qa = *reinterpret_cast<const uint4*>(a + col);
    const uint4 qb = *reinterpret_cast<const uint4*>(b + col);
    const uint32_t wa[4] = {qa.x, qa.y, qa.z, qa.w}, wb[4] = {qb.x, qb.y, qb.z, qb.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      acc = fmaf(bf16_lo(wa[j]), bf16_lo(wb[j]), acc);
      acc = fmaf(bf16_hi(wa[j]), bf16_hi(wb[j]), acc);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) g[p] = acc;
}

// One CTA per token; thread i owns 8-column groups i, i + blockDim, ...
__global__ void __launch_bounds__(128) combine_kernel(const uint16_t* __restrict__ c, int64_t ldc,
                                                      const int32_t* __restrict__ dest,
                                                      const float* __restrict__ w, int topk, int N,
                                                      uint16_t* __restrict__ out, int64_t ldo) {
  const int64_t t = blockIdx.x;
  __shared__ int32_t rows[8];
  __shared__ float ws[8];
  if (threadIdx.x < topk) {
    rows[threadIdx.x] = dest[t * topk + threadIdx.x];
    ws[threadIdx.x] = w[t * topk + threadIdx.x];
  }
  __syncthreads();
  for (int c8 = threadIdx.x; c8 * 8 < N; c8 += blockDim.x) {
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0f;
    for (int k = 0; k < topk; ++k) {
      if (rows[k] < 0) continue;  // dropped route (tagg_route_plan wrote -1) contributes nothing
      const uint4 q = *reinterpret_cast<const uint4*>(c + static_cast<int64_t>(rows[k]) * ldc + 8 * c8);
      const uint32_t qw[4] = {q.x, q.y, q.z, q.w};
      const float wk = ws[k];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[2 * j] = __fadd_rn(acc[2 * j], __fmul_rn(wk, bf16_lo(qw[j])));
        acc[2 * j + 1] = __fadd_rn(acc[2 * j + 1], __fmul_rn(wk, bf16_hi(qw[j])));
      }
    }
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t r;
      asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(acc[2 * j + 1]), "f"(acc[2 * j]));
      o[j] = r;
    }
    *reinterpret_cast<uint4*>(out + t * ldo + 8 * c8) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

}  // namespace moe
}  // namespace tagg

using namespace tagg;

extern "C" int tagg_swiglu_quantize(const void* h, int64_t ldh, const int32_t* group_sizes, int G, int64_t m_alloc,
                                    int I, void* a, int64_t lda, float* sa, int32_t* err_flag, void* v_out,
                                    int64_t ldv, void* stream) {
  if (I < 1 || G < 1 || m_alloc < 0) return TAGG_ERR_CONFIG;
  if (ldh < 2 * static_cast<int64_t>(I) || lda < I) return TAGG_ERR_SHAPE;
  if (m_alloc == 0) return TAGG_OK;
  if (!h || !group_sizes || !a || !sa || !err_flag) return TAGG_ERR_SHAPE;
  // 16-byte vectors: row pitches and both halves' starts on 16-byte boundaries
  if ((reinterpret_cast<uintptr_t>(h) % 16) || ((ldh * 2) % 16) || ((I * 2) % 16) ||
      (reinterpret_cast<uintptr_t>(a) % 16) || (lda % 16) ||
      (v_out && ((reinterpret_cast<uintptr_t>(v_out) % 16) || (ldv * 2) % 16 || ldv < I)))
    return TAGG_ERR_ALIGNMENT;
  const int warps = 8;
  const int64_t blocks = (m_alloc + warps - 1) / warps;
  if (blocks >= (int64_t(1) << 31)) return TAGG_ERR_UNSUPPORTED;
  moe::swiglu_quantize_kernel<<<static_cast<unsigned>(blocks), 32 * warps, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(h), ldh, group_sizes, G, m_alloc, I, static_cast<uint8_t*>(a), lda, sa, err_flag,
      static_cast<uint16_t*>(v_out), ldv);
  return cudaGetLastError() == cudaSuccess ? TAGG_OK : TAGG_ERR_CUDA;
}

extern "C" int tagg_swiglu_backward_quantize(const void* h, int64_t ldh, const void* dh, int64_t lddh,
                                             const int32_t* group_sizes, int G, int64_t m_alloc, int I, void* dgu,
                                             int64_t lddgu, void* a, int64_t lda, float* sa, int32_t* err_flag,
                                             void* stream) {
  if (I < 128 || I % 128 || G < 1 || m_alloc < 0) return TAGG_ERR_CONFIG;
  if (ldh < 2 * static_cast<int64_t>(I) || lddh < I || lda < 2 * static_cast<int64_t>(I) ||
      (dgu && lddgu < 2 * static_cast<int64_t>(I)))
    return TAGG_ERR_SHAPE;
  if (m_alloc == 0) return TAGG_OK;
  if (!h || !dh || !group_sizes || !a || !sa || !err_flag) return TAGG_ERR_SHAPE;
  auto mis = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) % 16) != 0; };
  if (mis(h) || mis(dh) || mis(a) || (dgu && mis(dgu)) || (ldh * 2) % 16 || (lddh * 2) % 16 || lda % 16 ||
      (dgu && (lddgu * 2) % 16))
    return TAGG_ERR_ALIGNMENT;
  const int warps = 8;
  const int64_t blocks = (m_alloc + warps - 1) / warps;
  if (blocks >= (int64_t(1) << 31)) return TAGG_ERR_UNSUPPORTED;
  moe::swiglu_backward_kernel<<<static_cast<unsigned>(blocks), 32 * warps, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(h), ldh, static_cast<const uint16_t*>(dh), lddh, group_sizes, G, m_alloc, I,
      static_cast<uint16_t*>(dgu), lddgu, static_cast<uint8_t*>(a), lda, sa, err_flag);
  return cudaGetLastError() == cudaSuccess ? TAGG_OK : TAGG_ERR_CUDA;
}

extern "C" int tagg_combine(const void* c, int64_t ldc, const int32_t* dest_rows, const float* weights, int64_t tokens,
                            int topk, int N, void* out, int64_t ldo, void* stream) {
  if (tokens < 0 || topk < 1 || topk > 8 || N < 8 || N % 8) return TAGG_ERR_CONFIG;
  if (ldc < N || ldo < N) return TAGG_ERR_SHAPE;
  if (tokens == 0) return TAGG_OK;
  if (!c || !dest_rows || !weights || !out) return TAGG_ERR_SHAPE;
  if ((reinterpret_cast<uintptr_t>(c) % 16) || ((ldc * 2) % 16) || (reinterpret_cast<uintptr_t>(out) % 16) ||
      ((ldo * 2) % 16))
    return TAGG_ERR_ALIGNMENT;
  if (tokens >= (int64_t(1) << 31)) return TAGG_ERR_UNSUPPORTED;
  moe::combine_kernel<<<static_cast<unsigned>(tokens), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(c), ldc, dest_rows, weights, topk, N, static_cast<uint16_t*>(out), ldo);
  return cudaGetLastError() == cudaSuccess ? TAGG_OK : TAGG_ERR_CUDA;
}

extern "C" int tagg_gather_scale_rows(const void* src, int64_t lds, const int32_t* index, const float* row_weights,
                                      int64_t rows, int H, void* out, int64_t ldo, void* stream) {
  if (rows < 0 || H < 8 || H % 8) return TAGG_ERR_CONFIG;
  if (lds < H || ldo < H) return TAGG_ERR_SHAPE;
  if (rows == 0) return TAGG_OK;
  if (!src || !index || !out) return TAGG_ERR_SHAPE;
  if ((reinterpret_cast<uintptr_t>(src) % 16) || (reinterpret_cast<uintptr_t>(out) % 16) || (lds * 2) % 16 ||
      (ldo * 2) % 16)
    return TAGG_ERR_ALIGNMENT;
  const int64_t blocks = (rows + 7) / 8;
  if (blocks >= (int64_t(1) << 31)) return TAGG_ERR_UNSUPPORTED;
  moe::gather_scale_rows_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(src), lds, index, row_weights, rows, H, static_cast<uint16_t*>(out), ldo);
  return cudaGetLastError() == cudaSuccess ? TAGG_OK : TAGG_ERR_CUDA;
}

extern "C" int tagg_router_grad(const void* dy, int64_t lddy, const void* c, int64_t ldc, const int32_t* dest_rows,
                                int64_t tokens, int topk, int H, float* out, void* stream) {
  if (tokens < 0 || topk < 1 || H < 8 || H % 8) return TAGG_ERR_CONFIG;
  if (lddy < H || ldc < H) return TAGG_ERR_SHAPE;
  if (tokens == 0) return TAGG_OK;
  if (!dy || !c || !dest_rows || !out) return TAGG_ERR_SHAPE;
  if ((reinterpret_cast<uintptr_t>(dy) % 16) || (reinterpret_cast<uintptr_t>(c) % 16) || (lddy * 2) % 16 ||
      (ldc * 2) % 16)
    return TAGG_ERR_ALIGNMENT;
  const int64_t pairs = tokens * topk;
  const int64_t blocks = (pairs + 7) / 8;
  if (blocks >= (int64_t(1) << 31)) return TAGG_ERR_UNSUPPORTED;
  moe::router_grad_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(dy), lddy, static_cast<const uint16_t*>(c), ldc, dest_rows, pairs, topk, H, out);
  return cudaGetLastError() == cudaSuccess ? TAGG_OK : TAGG_ERR_CUDA;
}
