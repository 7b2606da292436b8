// Microbenchmark: per-128-K promotion pipeline (MMA -> TMEM drain -> FFMA2) at several MMA
// widths N and TMEM buffer counts.  CTA pair (cta_group::2, M=256), K-major A and B resident in
// smem (4 rotating operand sets, random e4m3), 8 promotion warps; each thread drains its row's
// N/2 columns (32x32b.x32 chunks + an x16 remainder) and folds them into fp32 registers with
// FFMA2.  Prints clk per k-block and its ratio to the MMA floor (2N clk: 128 x N x 128 MACs per
// CTA at 8192 FP8 MAC/clk).  Question answered: does a third accumulation buffer (N=160 x 3)
// get closer to its floor than the kernel's N=256 x 2?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o nbuf nbuf.cu
#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <cuda_runtime.h>
#include "../../paper_2508_16584_b200/csrc/tagg_ptx.cuh"
using namespace tagg;

__device__ __forceinline__ void ld_x16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void wait16(uint32_t* r) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15])::"memory");
}

constexpr int kPromo = 8;
constexpr int kThreads = 32 * (4 + kPromo);
constexpr int kRot = 4;                 // operand sets the MMAs rotate through
constexpr int kSetBytes = 16384 + 16384;  // A 128 x 128 B, B up to 128 rows x 128 B

// DRAIN: 0 none, 1 full, 2 drain but no math
template <int N, int NBUF, int DRAIN, int HI = 0, int PROD = 0, int PAD = 1>
__global__ void __launch_bounds__(kThreads, 1) bench(int nk, unsigned long long* out, float* sink, unsigned long long* tr) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int CPT = N / 2;
  __shared__ uint64_t tfull[NBUF], tempty[NBUF], tfull2[NBUF], tempty2[NBUF];
  __shared__ __align__(128) uint64_t sbar[2 * 4 * 16];
  uint64_t* sfull = sbar;            // stride PAD barriers
  uint64_t* sempty = sbar + 4 * 16;
  constexpr bool SPLIT = DRAIN >= 5;  // two N/2 MMAs per k-block, each half of the buffer its own barriers
  __shared__ float s_sa[128 * 56];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < kRot * kSetBytes / 4; i += blockDim.x) {
    uint32_t v = (i + 1) * 2654435761u ^ (blockIdx.x * 97u);
    v ^= v >> 13; v *= 0x5bd1e995u; v ^= v >> 15;
    reinterpret_cast<uint32_t*>(smem)[i] = v & 0xFEFEFEFEu;  // never a NaN code
  }
  for (int i = threadIdx.x; i < 128 * 56; i += blockDim.x) s_sa[i] = 1.0f + 1e-6f * (i & 63);
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kPromo * 2);
      mbar_init(&tfull2[i], 1);
      mbar_init(&tempty2[i], kPromo * 2);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&sfull[i * PAD], 1);
      mbar_init(&sempty[i * PAD], 1);
    }
    fence_mbar_init();
  }
  constexpr int kCtl0 = HI ? kPromo : 0;  // first control warp (HI: control warps after the promotion warps)
  constexpr int kPro0 = HI ? 0 : 4;
  if (warp == kCtl0 + 3) tmem_alloc<2>(&slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp >= kCtl0 && warp < kCtl0 + 4) {
    setmaxnreg_dec<72>();
    if (PROD && warp == kCtl0 && rank == 0) {
      uint32_t st = 0, sph = 0;
      for (int i = 0; i < nk; ++i) {
        mbar_wait(&sempty[st * PAD], sph ^ 1);
        if (elect_one()) mbar_arrive(&sfull[st * PAD]);
        __syncwarp();
        if (++st == 4) { st = 0; sph ^= 1; }
      }
    }
    if (warp == kCtl0 + 1 && rank == 0) {
      uint32_t st = 0, sph = 0;
      const uint32_t idesc = idesc_e4m3_f32_ab(256, N, false, false);
      const uint64_t ad = umma_desc_sw128(smem_u32(smem), 16, 1024);
      const uint64_t bd = umma_desc_sw128(smem_u32(smem + 16384), 16, 1024);
      uint32_t b = 0, ph = 0;
      for (int i = 0; i < nk; ++i) {
        if (SPLIT) {
          const uint32_t idesc2 = idesc_e4m3_f32_ab(256, N / 2, false, false);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            mbar_wait(hh ? &tempty2[b] : &tempty[b], ph ^ 1);
            tc_fence_after();
            if (hh == 0 && lane == 0 && blockIdx.x == 0 && i < 1024) tr[0 * 1024 + i] = clock64();
            if (elect_one()) {
              const uint64_t off = (kSetBytes >> 4) * (i % kRot);
              const uint64_t boff = static_cast<uint64_t>(hh * (N / 4) * 128) >> 4;  // this CTA's N/4 B rows
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_f8f6f4<2>(tmem + b * N + hh * (N / 2), ad + off + 2 * k, bd + off + boff + 2 * k, idesc2, k > 0);
              mma_commit<2>(hh ? &tfull2[b] : &tfull[b]);
            }
            __syncwarp();
          }
        } else {
        if (PROD == 2) mbar_wait(&sfull[st * PAD], sph);  // operands first: usually long complete
        mbar_wait(&tempty[b], ph ^ 1);
        if (lane == 0 && blockIdx.x == 0 && i < 1024) tr[4 * 1024 + i] = clock64();
        if (PROD == 1) mbar_wait(&sfull[st * PAD], sph);
        tc_fence_after();
        if (lane == 0 && blockIdx.x == 0 && i < 1024) tr[0 * 1024 + i] = clock64();
        if (elect_one()) {
          const uint64_t off = (kSetBytes >> 4) * (i % kRot);
#pragma unroll
          for (int k = 0; k < 4; ++k) mma_f8f6f4<2>(tmem + b * N, ad + off + 2 * k, bd + off + 2 * k, idesc, k > 0);
          if (PROD) mma_commit<2>(&sempty[st * PAD]);
          mma_commit<2>(&tfull[b]);
        }
        __syncwarp();
        if (++st == 4) { st = 0; sph ^= 1; }
        }
        if (++b == NBUF) { b = 0; ph ^= 1; }
      }
    }
  } else {
    setmaxnreg_inc<216>();
    const int pw = warp - kPro0, q = warp & 3, half = pw >> 2;
    const uint32_t lanebase = static_cast<uint32_t>(32 * q) << 16;
    float acc[CPT];
#pragma unroll
    for (int i = 0; i < CPT; ++i) acc[i] = 0.f;
    uint32_t b = 0, ph = 0;
    unsigned long long tstart = 0;
    for (int i = 0; i < nk; ++i) {
      const float s = s_sa[(q * 32 + lane) * 56 + (i % 56)];
      mbar_wait(&tfull[b], ph);
      if (SPLIT && DRAIN != 5) mbar_wait(&tfull2[b], ph);
      tc_fence_after();
      const bool trc = pw == 0 && lane == 0 && blockIdx.x == 0 && i < 1024;
      if (trc) tr[1 * 1024 + i] = clock64();
      if (pw == 0 && lane == 0 && i == 0) tstart = clock64();
      const uint32_t ta = tmem + lanebase + b * N + half * CPT;
      if (DRAIN == 5) {  // split halves: this warp's 64 columns of each half; lo half freed first
        static_assert(DRAIN != 5 || N == 256, "split drain written for N = 256");
        const uint32_t tl = tmem + lanebase + b * N + half * 64;  // lo: cols [64h, 64h+64); hi: +128
        uint32_t va[32], vb[32];
        tmem_ld_32x32b_x32(tl, va);
        tmem_wait_ld_dep(va);
        tmem_ld_32x32b_x32(tl + 32, vb);
#pragma unroll
        for (int j = 0; j < 32; j += 2) ffma2(acc[j], acc[j + 1], __uint_as_float(va[j]), __uint_as_float(va[j + 1]), s);
        tmem_wait_ld_dep(vb);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(&tempty[b]);
        if (trc) tr[2 * 1024 + i] = clock64();
        mbar_wait(&tfull2[b], ph);
        tc_fence_after();
        tmem_ld_32x32b_x32(tl + 128, va);
#pragma unroll
        for (int j = 0; j < 32; j += 2) ffma2(acc[32 + j], acc[33 + j], __uint_as_float(vb[j]), __uint_as_float(vb[j + 1]), s);
        tmem_wait_ld_dep(va);
        tmem_ld_32x32b_x32(tl + 160, vb);
#pragma unroll
        for (int j = 0; j < 32; j += 2) ffma2(acc[64 + j], acc[65 + j], __uint_as_float(va[j]), __uint_as_float(va[j + 1]), s);
        tmem_wait_ld_dep(vb);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(&tempty2[b]);
#pragma unroll
        for (int j = 0; j < 32; j += 2) ffma2(acc[96 + j], acc[97 + j], __uint_as_float(vb[j]), __uint_as_float(vb[j + 1]), s);
      } else if (DRAIN == 7) {  // split MMAs, no drain
        tc_fence_before();
        __syncwarp();
        if (lane == 0) { mbar_arrive_leader(&tempty[b]); mbar_arrive_leader(&tempty2[b]); }
        if (trc) tr[2 * 1024 + i] = clock64();
        acc[0] += s;
      } else if (DRAIN == 3 || DRAIN == 6) {  // pipelined: chunk c+1's load in flight during chunk c's math
        static_assert(DRAIN != 3 || (CPT % 32) == 0, "x32 chunks");
        constexpr int n32 = CPT / 32;
        uint32_t va[32], vb[32];
        tmem_ld_32x32b_x32(ta, va);
        tmem_wait_ld_dep(va);
#pragma unroll
        for (int c = 0; c < n32; ++c) {
          uint32_t(&cur)[32] = (c & 1) ? vb : va;
          uint32_t(&nxt)[32] = (c & 1) ? va : vb;
          if (c + 1 < n32) tmem_ld_32x32b_x32(ta + 32 * (c + 1), nxt);
#pragma unroll
          for (int j = 0; j < 32; j += 2)
            ffma2(acc[32 * c + j], acc[32 * c + j + 1], __uint_as_float(cur[j]), __uint_as_float(cur[j + 1]), s);
          if (c + 1 < n32) tmem_wait_ld_dep(nxt);
          if (c + 2 == n32) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_leader(&tempty[b]);
            if (SPLIT && lane == 0) mbar_arrive_leader(&tempty2[b]);
            if (trc) tr[2 * 1024 + i] = clock64();
          }
        }
      } else if (DRAIN == 4) {  // math only, no TMEM load
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(&tempty[b]);
        if (trc) tr[2 * 1024 + i] = clock64();
#pragma unroll
        for (int j = 0; j < CPT; j += 2) ffma2(acc[j], acc[j + 1], s * 0.5f, s * 0.25f, s);
      } else if (DRAIN) {
        constexpr int n32 = CPT / 32;
#pragma unroll
        for (int c = 0; c < n32; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(ta + 32 * c, v);
          tmem_wait_ld_dep(v);
          if (c + 1 == n32 && (CPT % 32) == 0) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_leader(&tempty[b]);
            if (trc) tr[2 * 1024 + i] = clock64();
          }
          if (DRAIN == 1) {
#pragma unroll
            for (int j = 0; j < 32; j += 2)
              ffma2(acc[32 * c + j], acc[32 * c + j + 1], __uint_as_float(v[j]), __uint_as_float(v[j + 1]), s);
          } else {
            acc[c] += __uint_as_float(v[c]);
          }
        }
        if constexpr ((CPT % 32) != 0) {
          uint32_t v[16];
          ld_x16(ta + 32 * n32, v);
          wait16(v);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_leader(&tempty[b]);
            if (trc) tr[2 * 1024 + i] = clock64();
          if (DRAIN == 1) {
#pragma unroll
            for (int j = 0; j < 16; j += 2)
              ffma2(acc[32 * n32 + j], acc[32 * n32 + j + 1], __uint_as_float(v[j]), __uint_as_float(v[j + 1]), s);
          } else {
            acc[1] += __uint_as_float(v[1]);
          }
        }
      } else {
        acc[0] += s;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(&tempty[b]);
            if (trc) tr[2 * 1024 + i] = clock64();
      }
      if (trc) tr[3 * 1024 + i] = clock64();
      if (++b == NBUF) { b = 0; ph ^= 1; }
    }
    if (pw == 0 && lane == 0) out[blockIdx.x] = clock64() - tstart;
    float x = 0.f;
#pragma unroll
    for (int i = 0; i < CPT; ++i) x += acc[i];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = x;
  }
  __syncthreads();
  tc_fence_before();
  cluster_sync();
  if (warp == kCtl0 + 3) {
    tc_fence_after();
    tmem_dealloc<2>(tmem, 512);
  }
}

static unsigned long long* g_out;
static float* g_sink;
static unsigned long long* g_tr;

template <int N, int NBUF, int DRAIN, int HI = 0, int PROD = 0, int PAD = 1>
void run(const char* name) {
  static_assert(N * NBUF <= 512, "TMEM");
  const int nk = 4096;
  const int smem = kRot * kSetBytes + 1024;
  cudaFuncSetAttribute(bench<N, NBUF, DRAIN, HI, PROD, PAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
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
  float best = 1e30f;
  double mx_best = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, bench<N, NBUF, DRAIN, HI, PROD, PAD>, nk, g_out, g_sink, g_tr);
    cudaEventRecord(e1);
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[148];
    cudaMemcpy(h, g_out, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    if (ms < best) { best = ms; mx_best = mx; }
  }
  static unsigned long long t[5 * 1024];
  cudaMemcpy(t, g_tr, sizeof(t), cudaMemcpyDeviceToHost);
  auto med = [&](int a, int b, int sh) {
    static double v[1024];
    int n = 0;
    for (int i = 100; i < 1000; ++i) v[n++] = double(t[a * 1024 + i]) - double(t[b * 1024 + i - sh]);
    std::sort(v, v + n);
    return v[n / 2];
  };
  const double flops = 148.0 * 128 * N * 128 * 2.0 * nk;
  printf("%-34s HI=%d N=%3d x%d  %7.1f clk/k-block  floor %4d  eff %.3f  %7.1f TFLOP/s  (%.0f MHz)\n", name, HI, N, NBUF,
         mx_best / nk, 2 * N, 2.0 * N / (mx_best / nk), flops / (best * 1e-3) / 1e12, mx_best / (best * 1e3));
  printf("     issue period %.0f | issue->promo full %.0f | full->freed %.0f | freed->done %.0f | done->next full %.0f | freed(i-NBUF)->issue(i) %.0f | tempty seen->issue %.0f\n",
         med(0, 0, 1), med(1, 0, 0), med(2, 1, 0), med(3, 2, 0), med(1, 3, 1), med(0, 2, NBUF), med(0, 4, 0));
}

int main() {
  cudaMalloc(&g_out, 148 * 8);
  cudaMalloc(&g_sink, 148 * kThreads * 4);
  cudaMalloc(&g_tr, 5 * 1024 * 8);
  for (int pass = 0; pass < 2; ++pass) {
    run<256, 2, 0, 0, 1, 1>("no drain, producer ring");
    run<256, 2, 0, 0, 1, 16>("no drain, producer ring, padded bars");
    run<256, 2, 0, 0, 2, 1>("no drain, producer ring, full first");
    run<256, 2, 3, 0, 1, 1>("drain+ffma2, producer ring");
    run<256, 2, 3, 0, 1, 16>("drain+ffma2, ring, padded bars");
    run<256, 2, 3, 0, 2, 1>("drain+ffma2, ring, full first");
    run<256, 2, 3, 0, 0, 1>("drain+ffma2, no ring");
  }
  return 0;
}
