// Microbenchmark: mma_vs_ld's pipeline (CTA pair, 256x256 tile, 2 TMEM buffers,
// 8 promotion warps) fed by REAL TMA loads of A [rows, K] and MN-major B [K, N]
// from global memory, the way tagg_gemm_kernel feeds it.  Prints the k-block
// period; MODE selects the promotion work.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "../../paper_2508_16584_b200/csrc/tagg_ptx.cuh"
using namespace tagg;

constexpr int kPromo = 8;
constexpr int kThreads = 32 * (4 + kPromo);
constexpr int KB = 64;  // k-blocks per tile (K = 8192)

struct P {
  CUtensorMap ta, tb, tc;
};

// MODE 0: no drain.  1: drain + FFMA2 (late release).  2: drain + FFMA2 (early release)
// 3: the kernel's drain (two 32x32b.x64 loads, release after the second, math between)
// LOAD 0: producer only arrives (no TMA).  1: TMA A + B.
// X bit 0: scale s from two ld.shared one k-block ahead; bit 1: epilogue (bf16 -> smem
// staging -> TMA store) every KB k-blocks; bit 2: MMA waits full before tempty;
// bit 4: pair cid reads B n-tile cid % 16 of a [K, 4096] B (distinct B per pair)
template <int MODE, int LOAD, int X = 0, int NS = 4>
__global__ void __launch_bounds__(kThreads, 1) gemm(const __grid_constant__ P p, int reps, unsigned long long* out,
                                                    float* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                 // NS x 16 KB
  uint8_t* sB = smem + NS * 16384;    // NS x 16 KB (this CTA's 128 columns x 128 K, SW128)
  uint8_t* sC = smem + 2 * NS * 16384;  // 2 x 16 KB staging
  __shared__ uint64_t tfull[2], tempty[2], full[NS], empty[NS];
  __shared__ float s_sa[128 * KB], s_sb[2 * KB];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const int cid = blockIdx.x / 2;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kPromo * 2);
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<2>(&slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const int nk = reps * KB;
  const unsigned long long t0 = clock64();
  if (warp < 4) {
    setmaxnreg_dec<72>();
    if (warp == 0 && lane == 0) {
      for (int i = 0; i < nk; ++i) {
        const int s = i % NS;
        mbar_wait(&empty[s], ((i / NS) & 1) ^ 1);
        if (LOAD) {
          if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * (16384 + 16384));
          const int kb = i % KB;
          tma_load_2d_cg2(&p.ta, &full[s], sA + s * 16384, kb * 128, cid * 256 + rank * 128);
          tma_load_3d_cg2(&p.tb, &full[s], sB + s * 16384, ((X & 16) ? (cid % 16) * 256 : 0) + rank * 128, kb * 128, 0);
        } else if (rank == 0) {
          mbar_arrive(&full[s]);
        }
      }
      for (int i = nk; i < nk + NS; ++i) mbar_wait(&empty[i % NS], ((i / NS) & 1) ^ 1);
    } else if (warp == 1 && rank == 0 && lane == 0) {
      const uint32_t tmem = slot;
      const uint32_t idesc = idesc_e4m3_f32(256, 256, true);
      const uint64_t ad0 = umma_desc_sw128(smem_u32(sA), 16, 1024);
      const uint64_t bd0 = umma_desc_sw128(smem_u32(sB), 16384, 1024);
      for (int i = 0; i < nk; ++i) {
        const int b = i & 1, s = i % NS;
        if (X & 4) {
          mbar_wait(&full[s], (i / NS) & 1);
          mbar_wait(&tempty[b], ((i >> 1) & 1) ^ 1);
        } else {
          mbar_wait(&tempty[b], ((i >> 1) & 1) ^ 1);
          mbar_wait(&full[s], (i / NS) & 1);
        }
        tc_fence_after();
        const uint64_t ad = ad0 + ((s * 16384) >> 4), bd = bd0 + ((s * 16384) >> 4);
#pragma unroll
        for (int k = 0; k < 4; ++k) mma_f8f6f4<2>(tmem + b * 256, ad + 2 * k, bd + 256 * k, idesc, k > 0);
        mma_commit<2>(&empty[s]);
        mma_commit<2>(&tfull[b]);
      }
    }
  } else {
    setmaxnreg_inc<216>();
    const uint32_t tmem = slot;
    const int pw = warp - 4, q = warp & 3, half = pw >> 2;
    const uint32_t ta0 = tmem + (static_cast<uint32_t>(32 * q) << 16) + half * 128;
    float acc[128];
#pragma unroll
    for (int i = 0; i < 128; ++i) acc[i] = 0.f;
    const int r = 32 * q + lane;
    const int ptid = threadIdx.x - 128;
    // X & 8: S_A transposed [kb][row] (conflict-free); else [row][kb] (32-way conflict)
    const uint32_t sa_row = (X & 8) ? smem_u32(s_sa) + 4u * r : smem_u32(s_sa) + 4u * KB * r;
    const uint32_t sa_step = (X & 8) ? 4u * 128 : 4u;
    const uint32_t sb_col = smem_u32(s_sb) + 4u * KB * half;
    float s_next = (X & 1) ? __fmul_rn(ld_shared_f32(sa_row), ld_shared_f32(sb_col)) : 1.0f;
    for (int i = 0; i < nk; ++i) {
      const int b = i & 1;
      float s = 1.0f + 1e-7f * i;
      if (X & 1) {
        s = s_next;
        const int kn = (i + 1) % KB;
        s_next = __fmul_rn(ld_shared_f32(sa_row + sa_step * kn), ld_shared_f32(sb_col + 4u * kn));
      }
      mbar_wait(&tfull[b], (i >> 1) & 1);
      tc_fence_after();
      if (MODE == 3) {
        const uint32_t ta = ta0 + b * 256;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t v[64];
          tmem_ld_32x32b_x64(ta + 64 * c, v);
          tmem_wait_ld_dep64(v);
          if (c == 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_leader(&tempty[b]);
          }
#pragma unroll
          for (int j = 0; j < 64; j += 2)
            ffma2(acc[64 * c + j], acc[64 * c + j + 1], __uint_as_float(v[j]), __uint_as_float(v[j + 1]), s);
        }
      } else if (MODE != 0) {
        const uint32_t ta = ta0 + b * 256;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(ta + 32 * c, v);
          tmem_wait_ld_dep(v);
          if (MODE == 2 && c == 3) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_leader(&tempty[b]);
          }
#pragma unroll
          for (int j = 0; j < 32; j += 2)
            ffma2(acc[32 * c + j], acc[32 * c + j + 1], __uint_as_float(v[j]), __uint_as_float(v[j + 1]), s);
        }
      }
      if (MODE != 2 && MODE != 3) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(&tempty[b]);
      }
      if ((X & 2) && (i % KB) == KB - 1) {
        // epilogue: 2 passes of 128 columns, 2 chunks of 64 bf16 columns each
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
          if (ptid == 0) bulk_wait_read0();
          named_bar_sync(1, 256);
          if (half == pass) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int chunk = j >> 3, pc = j & 7;
              const uint32_t w0 = pack_bf16x2(acc[8 * j + 0], acc[8 * j + 1]);
              const uint32_t w1 = pack_bf16x2(acc[8 * j + 2], acc[8 * j + 3]);
              const uint32_t w2 = pack_bf16x2(acc[8 * j + 4], acc[8 * j + 5]);
              const uint32_t w3 = pack_bf16x2(acc[8 * j + 6], acc[8 * j + 7]);
              st_shared_v4(smem_u32(sC + chunk * 16384) + r * 128u + ((pc ^ (r & 7)) * 16u), w0, w1, w2, w3);
            }
            fence_proxy_async_smem();
          }
          named_bar_sync(1, 256);
          if (ptid == 0) {
            for (int ch = 0; ch < 2; ++ch)
              tma_store_2d(&p.tc, sC + ch * 16384, 128 * pass + 64 * ch, cid * 256 + rank * 128);
            bulk_commit();
          }
        }
#pragma unroll
        for (int j = 0; j < 128; ++j) acc[j] = 0.f;
      }
    }
    if (ptid == 0) bulk_wait0();
    float x = 0.f;
#pragma unroll
    for (int i = 0; i < 128; ++i) x += acc[i];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = x;
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<2>(slot, 512);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* ptr = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
}

template <int MODE, int LOAD, int X = 0, int NS = 4>
void run(const char* name, const P& p, unsigned long long* d_out, float* sink) {
  const int reps = 32;
  const int smem = 2 * NS * 16384 + 32768 + 1024;
  cudaFuncSetAttribute(gemm<MODE, LOAD, X, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1] = {};
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, gemm<MODE, LOAD, X, NS>, p, reps, d_out, sink);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int it = 0; it < 5; ++it) cudaLaunchKernelEx(&cfg, gemm<MODE, LOAD, X, NS>, p, reps, d_out, sink);
  cudaEventRecord(e1);
  const cudaError_t e = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 5;
  const double tflops = 74.0 * reps * KB * 2.0 * 256 * 256 * 128 / (ms * 1e-3) / 1e12;
  std::vector<unsigned long long> h(148);
  cudaMemcpy(h.data(), d_out, 148 * 8, cudaMemcpyDeviceToHost);
  const double mx = *std::max_element(h.begin(), h.end());
  printf("%-40s k-block period %7.1f clk  %7.1f TFLOP/s  (%.0f MHz) %s\n", name, mx / (reps * KB), tflops,
         mx / (ms * 1e3), e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  const int M = 256 * 74, K = 8192, N = 4096;
  uint8_t *a, *b;
  cudaMalloc(&a, size_t(M) * K);
  cudaMalloc(&b, size_t(K) * N);
  std::vector<uint8_t> h(size_t(M) * K);
  uint32_t x = 12345;
  for (auto& v : h) {
    x = x * 1664525u + 1013904223u;
    v = static_cast<uint8_t>(x >> 24) & 0xFE;
  }
  cudaMemcpy(a, h.data(), size_t(M) * K, cudaMemcpyHostToDevice);
  cudaMemcpy(b, h.data(), size_t(K) * N, cudaMemcpyHostToDevice);  // K*N <= M*K
  P p;
  auto fn = enc();
  {
    cuuint64_t d[2] = {cuuint64_t(K), cuuint64_t(M)}, s[1] = {cuuint64_t(K)};
    cuuint32_t box[2] = {128, 128}, e[2] = {1, 1};
    fn(&p.ta, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, a, d, s, box, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    cuuint64_t d[3] = {cuuint64_t(N), cuuint64_t(K), 1}, s[2] = {cuuint64_t(N), cuuint64_t(N) * K};
    cuuint32_t box[3] = {128, 128, 1}, e[3] = {1, 1, 1};
    fn(&p.tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, b, d, s, box, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    uint16_t* c;
    cudaMalloc(&c, size_t(M) * N * 2);
    cuuint64_t d[2] = {cuuint64_t(N), cuuint64_t(M)}, s[1] = {cuuint64_t(N) * 2};
    cuuint32_t box[2] = {64, 128}, e[2] = {1, 1};
    fn(&p.tc, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, c, d, s, box, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  unsigned long long* d_out;
  float* sink;
  cudaMalloc(&d_out, 148 * 8);
  cudaMalloc(&sink, 148 * kThreads * 4);
  run<0, 1>("TMA, no drain", p, d_out, sink);
  run<2, 1>("TMA, drain x32 (early release)", p, d_out, sink);
  run<3, 1>("TMA, drain x64 kernel-style", p, d_out, sink);
  run<3, 1, 0, 3>("TMA, drain x64, 3 stages", p, d_out, sink);
  run<3, 1, 1>("TMA, drain x64, s from smem", p, d_out, sink);
  run<3, 1, 16>("TMA, drain x64, distinct B", p, d_out, sink);
  run<3, 1, 2>("TMA, drain x64, epilogue", p, d_out, sink);
  run<3, 1, 19, 3>("TMA, drain x64, all, 3 stages", p, d_out, sink);
  run<2, 1, 19, 3>("TMA, drain x32, all, 3 stages", p, d_out, sink);
  return 0;
}
