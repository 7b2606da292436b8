// Microbenchmark: does the promotion drain (tcgen05.ld) run concurrently with
// tcgen05.mma, or do they serialise on TMEM?  One CTA per SM, cta_group::1,
// M=128 N=256 K=32 kind::f8f6f4 (4 MMAs per 128-K "k-block" into a fresh
// 256-column TMEM buffer, 2 buffers), 8 promotion warps drain each buffer
// (128 lanes x 256 cols fp32 = 128 KB) with the load shape under test and fold
// it into fp32 registers with FFMA2, then free it.
#include <cstdio>
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2508_16584_b200/csrc/tagg_ptx.cuh"
using namespace tagg;

#define R4(i) "=r"(r[i]), "=r"(r[i + 1]), "=r"(r[i + 2]), "=r"(r[i + 3])
#define R16(i) R4(i), R4(i + 4), R4(i + 8), R4(i + 12)
#define R32(i) R16(i), R16(i + 16)

__device__ __forceinline__ void ld_16x256b_x8(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : R32(0)
      : "r"(taddr));
}
__device__ __forceinline__ void ld_16x128b_x16(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x128b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : R32(0)
      : "r"(taddr));
}
__device__ __forceinline__ void ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : R16(0)
      : "r"(taddr));
}
__device__ __forceinline__ void wait_dep16(uint32_t (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15])::"memory");
}

constexpr int kPromo = 8;
constexpr int kThreads = 32 * (4 + kPromo);

// MODE: 0 no drain; 1 32x32b.x32 pipelined; 2 16x256b.x8; 3 16x128b.x16; 4 32x32b.x16 pipelined;
//       5 32x32b.x32 but only half the columns (64 KB); 6 x32, drain issued only after the MMA
//       for the NEXT buffer completed (no overlap by construction: measures serialised cost)
template <int MODE, int CG, int BMN = 0, int EXTRA = 0>
__global__ void __launch_bounds__(kThreads, 1) bench(int nk, unsigned long long* out, float* sink, int fill, unsigned long long* tr) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // ROT stages of [A 16 KB | B 32 KB]; EXTRA & 8 rotates the MMA operands through them
  constexpr int ROT = (EXTRA & 8) ? 4 : 1;
  constexpr int NS = (EXTRA & 32) ? 4 : 6;   // ring depth
  uint8_t* sA = smem;           // 128 x 128 B, K-major SW128
  uint8_t* sB = smem + 16384;   // 256 x 128 B, K-major SW128
  __shared__ uint64_t tfull[2], tempty[2], full[6], empty[6];
  __shared__ float s_sa[128 * 56];
  __shared__ uint32_t slot;
  __shared__ unsigned long long drain_clk;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < ROT * 49152 / 4; i += blockDim.x) {
    uint32_t v = 0x38383838u;
    if (fill) {  // random e4m3 codes, never NaN
      v = (i + 1) * 2654435761u ^ (blockIdx.x * 97u);
      v ^= v >> 13; v *= 0x5bd1e995u; v ^= v >> 15;
      v &= 0xFEFEFEFEu;  // clear bit 0 of each byte: 0x7F / 0xFF cannot occur
    }
    reinterpret_cast<uint32_t*>(smem)[i] = v;
  }
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kPromo * CG);
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    drain_clk = 0;
    fence_mbar_init();
  }
  if (warp == 3) tmem_alloc<CG>(&slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const unsigned long long t0 = clock64();
  if (warp < 4) {
   if (EXTRA & 4) setmaxnreg_dec<72>();
   if (warp == ((EXTRA & 16) ? 1 : 0) && rank == 0) {
    // EXTRA & 64: A MN-major too (128 K-rows of 128 B = this CTA's 128 M rows, K step 4 KB),
    // the wgrad kernel's operand layout
    constexpr bool AMN = (EXTRA & 64) != 0;
    const uint32_t idesc = idesc_e4m3_f32_ab(128 * CG, 256, AMN, BMN != 0);
    const uint64_t ad = umma_desc_sw128(smem_u32(sA), AMN ? 16384 : 16, 1024);
    const uint32_t astep = AMN ? 256 : 2;
    // B K-major: 256/CG N-rows of 128 B.  MN-major: 128 K-rows of 128 B (this CTA's 128 N columns), K step 4 KB.
    const uint64_t bd = umma_desc_sw128(smem_u32(sB), BMN ? 16384 : 16, 1024);
    const uint32_t bstep = BMN ? 256 : 2;
    const bool el = elect_one();
    for (int i = 0; i < nk; ++i) {
      const int b = i & 1;
      mbar_wait(&tempty[b], ((i >> 1) & 1) ^ 1);
      if (lane == 0 && blockIdx.x == 0 && i < 1024) tr[0 * 1024 + i] = clock64();
      if (EXTRA & 1) mbar_wait(&full[i % NS], (i / NS) & 1);
      if (lane == 0 && blockIdx.x == 0 && i < 1024) tr[1 * 1024 + i] = clock64();
      tc_fence_after();
      if (el) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma_f8f6f4<CG>(tmem + b * 256, ad + 3072 * (i % ROT) + astep * k, bd + 3072 * (i % ROT) + bstep * k, idesc, k > 0);
        if (EXTRA & 1) mma_commit<CG>(&empty[i % NS]);
        mma_commit<CG>(&tfull[b]);
      }
      __syncwarp();
      if (lane == 0 && blockIdx.x == 0 && i < 1024) tr[2 * 1024 + i] = clock64();
    }
   } else if (warp == ((EXTRA & 16) ? 0 : 2) && (EXTRA & 1)) {
    // producer stand-in: waits for the slot, then arrives on the leader's full barrier (no loads)
    for (int i = 0; i < nk; ++i) {
      mbar_wait(&empty[i % NS], ((i / NS) & 1) ^ 1);
      if (lane == 0 && rank == 0) mbar_arrive(&full[i % NS]);
      __syncwarp();
    }
    for (int i = nk; i < nk + NS; ++i) mbar_wait(&empty[i % NS], ((i / NS) & 1) ^ 1);
   }
  } else {
    if (EXTRA & 4) setmaxnreg_inc<216>();
    const int pw = warp - 4, q = warp & 3, half = pw >> 2;
    const uint32_t lanebase = static_cast<uint32_t>(32 * q) << 16;
    float acc[128];
#pragma unroll
    for (int i = 0; i < 128; ++i) acc[i] = 0.f;
    unsigned long long dsum = 0;
    const float* sbp = sink + 4096 + (blockIdx.x & 7) * 64;
    float sb_next = (EXTRA & 2) ? __ldg(sbp) : 1.0f;
    for (int i = 0; i < nk; ++i) {
      const int b = i & 1;
      float s = 1.0f + 1e-7f * i;
      if (EXTRA & 2) {
        const float sbv = sb_next;
        sbp += 1;
        sb_next = __ldg(sbp);
        s = __fmul_rn(s_sa[(q * 32 + lane) * 56 + (i % 56)], sbv);
      }
      mbar_wait(&tfull[b], (i >> 1) & 1);
      if (pw == 0 && lane == 0 && blockIdx.x == 0 && i < 1024) tr[4 * 1024 + i] = clock64();
      if (MODE == 6) {  // wait until the next k-block's MMA has finished too (serialised drain)
        if (i + 1 < nk) mbar_wait(&tfull[b ^ 1], ((i + 1) >> 1) & 1);
      }
      tc_fence_after();
      const unsigned long long d0 = clock64();
      const uint32_t ta = tmem + lanebase + b * 256 + half * 128;
      if (MODE == 1 || MODE == 5 || MODE == 6) {
        constexpr int kCh = (MODE == 5) ? 2 : 4;
        uint32_t va[32], vb[32];
        tmem_ld_32x32b_x32(ta, va);
        tmem_wait_ld_dep(va);
#pragma unroll
        for (int c = 0; c < kCh; ++c) {
          uint32_t(&cur)[32] = (c & 1) ? vb : va;
          uint32_t(&nxt)[32] = (c & 1) ? va : vb;
          if (c + 1 < kCh) tmem_ld_32x32b_x32(ta + 32 * (c + 1), nxt);
#pragma unroll
          for (int j = 0; j < 32; j += 2)
            ffma2(acc[32 * c + j], acc[32 * c + j + 1], __uint_as_float(cur[j]), __uint_as_float(cur[j + 1]), s);
          if (c + 1 < kCh) tmem_wait_ld_dep(nxt);
        }
      } else if (MODE == 2 || MODE == 3) {
        // 16-lane shapes: two lane halves (+0, +16) x 2 column halves of 64
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t v[32];
          const uint32_t a2 = ta + (static_cast<uint32_t>(16 * (c & 1)) << 16) + 64 * (c >> 1);
          if (MODE == 2) ld_16x256b_x8(a2, v); else ld_16x128b_x16(a2, v);
          tmem_wait_ld_dep(v);
#pragma unroll
          for (int j = 0; j < 32; j += 2)
            ffma2(acc[32 * c + j], acc[32 * c + j + 1], __uint_as_float(v[j]), __uint_as_float(v[j + 1]), s);
        }
      } else if (MODE == 4) {
        uint32_t va[16], vb[16];
        ld_32x32b_x16(ta, va);
        wait_dep16(va);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint32_t(&cur)[16] = (c & 1) ? vb : va;
          uint32_t(&nxt)[16] = (c & 1) ? va : vb;
          if (c + 1 < 8) ld_32x32b_x16(ta + 16 * (c + 1), nxt);
#pragma unroll
          for (int j = 0; j < 16; j += 2)
            ffma2(acc[16 * c + j], acc[16 * c + j + 1], __uint_as_float(cur[j]), __uint_as_float(cur[j + 1]), s);
          if (c + 1 < 8) wait_dep16(nxt);
        }
      }
      dsum += clock64() - d0;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2) mbar_arrive_leader(&tempty[b]); else mbar_arrive(&tempty[b]);
      }
      if (pw == 0 && lane == 0 && blockIdx.x == 0 && i < 1024) tr[5 * 1024 + i] = clock64();
    }
    float x = 0.f;
#pragma unroll
    for (int i = 0; i < 128; ++i) x += acc[i];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = x;
    if (pw == 0 && lane == 0) drain_clk = dsum;
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = t1 - t0;
    out[2 * blockIdx.x + 1] = drain_clk;
  }
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 3) {
    tc_fence_after();
    tmem_dealloc<CG>(tmem, 512);
  }
}

static unsigned long long* g_out;
static float* g_sink;
static unsigned long long* g_tr;

template <int MODE, int CG, int BMN, int EXTRA>
void launch(int nk, int smem, int fill) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1] = {};
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, bench<MODE, CG, BMN, EXTRA>, nk, g_out, g_sink, fill, g_tr);
}

template <int MODE, int CG = 1, int BMN = 0, int EXTRA = 0>
void run(const char* name, int fill = 0, int smem_override = 0) {
  const int nk = 2048;
  const int smem = smem_override ? smem_override : ((EXTRA & 8) ? 4 : 1) * 49152 + 1024;
  cudaFuncSetAttribute(bench<MODE, CG, BMN, EXTRA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  cudaFuncSetAttribute(bench<MODE, CG, BMN, EXTRA>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  launch<MODE, CG, BMN, EXTRA>(nk, smem, fill);
  cudaDeviceSynchronize();
  launch<MODE, CG, BMN, EXTRA>(nk, smem, fill);
  const cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[296];
  cudaMemcpy(h, g_out, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0, dr = 0;
  for (int i = 0; i < 148; ++i) {
    mx = h[2 * i] > mx ? h[2 * i] : mx;
    dr += h[2 * i + 1];
  }
  {
    static unsigned long long t[6 * 1024];
    cudaMemcpy(t, g_tr, sizeof(t), cudaMemcpyDeviceToHost);
    auto med = [&](int a, int b, int sh) {
      static double v[1024];
      int n = 0;
      for (int i = 100; i < 900; ++i) v[n++] = double(t[a * 1024 + i]) - double(t[b * 1024 + i - sh]);
      std::sort(v, v + n);
      return v[n / 2];
    };
    printf("   issue period %.0f | tempty wait %.0f | full wait %.0f | issue %.0f | issue->promo full %.0f | promo full->arrive %.0f | arrive(i-2)->tempty(i) %.0f\n",
           med(2, 2, 1), med(0, 2, 1), med(1, 0, 0), med(2, 1, 0), med(4, 2, 0), med(5, 4, 0), med(0, 5, 2));
  }
  printf("%-44s fill=%d k-block period %7.1f clk (MMA-only ideal 512)   drain %6.1f clk/k-block %s\n", name, fill, mx / nk,
         dr / 148 / nk, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  cudaMalloc(&g_out, 296 * 8);
  cudaMalloc(&g_tr, 6 * 1024 * 8);
  cudaMalloc(&g_sink, (148 * kThreads + 8192) * 4);
  cudaMemset(g_sink, 0, (148 * kThreads + 8192) * 4);
  run<0, 2, 0, 0>("cg2: no drain, A K-major, B K-major");
  run<0, 2, 1, 0>("cg2: no drain, A K-major, B MN-major");
  run<0, 2, 1, 64>("cg2: no drain, A MN-major, B MN-major");
  run<1, 2, 1, 0>("cg2: 32x32b.x32 drain, A K, B MN");
  run<1, 2, 1, 64>("cg2: 32x32b.x32 drain, A MN, B MN");
  run<0, 2, 1, 0>("cg2: no drain, A K, B MN", 1);
  run<1, 2, 1, 0>("cg2: 32x32b.x32 drain, A K, B MN", 1);
  return 0;
}
