// Microbenchmark: K1's k-block loop transplanted (producer without loads, MMA issuer, promotion
// with smem scales, s one k-block ahead, the x32 two-in-flight drain), on smem-resident random
// operands, one "tile" of nk k-blocks per CTA pair.  Variants switch single features off to find
// what separates the kernel (~970 clk per k-block) from tools/micro/nbuf.cu (~660).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o kloop kloop.cu
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2508_16584_b200/csrc/tagg_ptx.cuh"
using namespace tagg;

constexpr int kThreads = 384;
constexpr int kS = 4;  // stages, each A 16 KB + B 16 KB (MN-major)
// V bits: 1 = scales from smem (else constant), 2 = trace stamps off, 4 = release before math (x64),
//         8 = MMA waits stage full, 16 = MMA warp tempty-first
template <int V, int CG = 2>
__global__ void __launch_bounds__(kThreads, 1) kloop(int nk, unsigned long long* out, float* sink,
                                                   unsigned long long* tr, float one) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr uint32_t kStB = CG == 2 ? 16384 : 32768;  // B per stage: this CTA's 128 columns, or all 256 (CG 1)
  uint8_t* sA = smem;
  uint8_t* sB = smem + kS * 16384;
  constexpr int kKb = 56;  // scale window depth (the DeepSeek-V3 gate+up tile); k-block kb reads column kb % 56
  float* sSA = reinterpret_cast<float*>(smem + kS * (16384 + kStB));  // [128 rows][56] (rb = 224 B)
  float* sSB = sSA + 128 * kKb;                                   // [2][56]
  __shared__ uint64_t full[kS], empty[kS], tfull[2], tempty[2];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < kS * (16384 + kStB) / 4; i += blockDim.x) {
    uint32_t v = (i + 1) * 2654435761u ^ (blockIdx.x * 97u);
    v ^= v >> 13; v *= 0x5bd1e995u; v ^= v >> 15;
    reinterpret_cast<uint32_t*>(smem)[i] = v & 0xFEFEFEFEu;
  }
  for (int i = threadIdx.x; i < 130 * kKb; i += blockDim.x) sSA[i] = 0.001f * (1 + (i & 7));
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 8 * CG); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<CG>(&slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const bool trace = !(V & 2) && blockIdx.x == 0;
  if (warp < 4) {
    setmaxnreg_dec<72>();
    if (warp == 0 && rank == 0) {
      uint32_t stage = 0, phase = 0;
      const uint32_t full0 = smem_u32(&full[0]), empty0 = smem_u32(&empty[0]);
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait_addr(empty0 + 8 * stage, phase ^ 1);
        if (elect_one()) mbar_arrive_addr(full0 + 8 * stage);
        __syncwarp();
        if (++stage == kS) { stage = 0; phase ^= 1; }
      }
    } else if (warp == 1 && rank == 0) {
      const uint32_t tmem_base = ld_shared_u32(smem_u32(&slot));
      const uint32_t idesc = idesc_e4m3_f32(128 * CG, 256, true);
      const uint64_t a_desc0 = umma_desc_sw128(smem_u32(sA), 16, 1024);
      const uint64_t b_desc0 = umma_desc_sw128(smem_u32(sB), 16384, 1024);
      const uint32_t full0 = smem_u32(&full[0]), empty0 = smem_u32(&empty[0]);
      const uint32_t tfull0 = smem_u32(&tfull[0]), tempty0 = smem_u32(&tempty[0]);
      uint32_t stage = 0, phase = 0, acc = 0, accph = 0;
      for (int kb = 0; kb < nk; ++kb) {
        if (V & 16) mbar_wait_addr(tempty0 + 8 * acc, accph ^ 1);
        if (V & 8) mbar_wait_addr(full0 + 8 * stage, phase);
        if (!(V & 16)) mbar_wait_addr(tempty0 + 8 * acc, accph ^ 1);
        tc_fence_after();
        if (trace && lane == 0 && kb < 1024) tr[0 * 1024 + kb] = clock64();
        const uint64_t ad = a_desc0 + ((stage * 16384u) >> 4);
        const uint64_t bd = b_desc0 + ((stage * kStB) >> 4);
        const uint32_t d_tmem = tmem_base + acc * 256;
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_f8f6f4<CG>(d_tmem, ad + static_cast<uint64_t>(k * 2), bd + static_cast<uint64_t>(k * 256), idesc,
                           k > 0 ? 1u : 0u);
          mma_commit_addr<CG>(empty0 + 8 * stage);
          mma_commit_addr<CG>(tfull0 + 8 * acc);
        }
        __syncwarp();
        if (trace && lane == 0 && kb < 1024) tr[1 * 1024 + kb] = clock64();
        if (++stage == kS) { stage = 0; phase ^= 1; }
        if (++acc == 2) { acc = 0; accph ^= 1; }
      }
    }
  } else {
    setmaxnreg_inc<216>();
    const uint32_t tmem_base = opaque_u32(ld_shared_u32(smem_u32(&slot)));
    const int pw = warp - 4, q = warp & 3, half = pw >> 2, r = 32 * q + lane;
    const uint32_t t_lane = static_cast<uint32_t>(32 * q) << 16;
    const uint32_t tfull0 = opaque_u32(smem_u32(&tfull[0])), tempty0 = opaque_u32(smem_u32(&tempty[0]));
    const uint32_t sa_row = smem_u32(sSA) + static_cast<uint32_t>(r) * 4u * kKb;
    const uint32_t sb_colp = smem_u32(sSB) + 4u * static_cast<uint32_t>(half * kKb);
    const bool tr_a = trace && pw == 0 && lane == 0;
    float acc[128];
#pragma unroll
    for (int i = 0; i < 128; ++i) acc[i] = 0.0f;
    uint32_t acc_i = 0, accph = 0;
    float s_next = (V & 1) ? __fmul_rn(ld_shared_f32(sa_row), ld_shared_f32(sb_colp)) : 1.0f;
    for (int kb = 0; kb < nk; ++kb) {
      const float s = s_next;
      if (V & 1) {
        if (kb + 1 < nk) {
          const uint32_t j = 4u * static_cast<uint32_t>((kb + 1) % kKb);
          s_next = __fmul_rn(ld_shared_f32(sa_row + j), ld_shared_f32(sb_colp + j));
        }
      } else {
        s_next = s * one;
      }
      mbar_wait_addr(tfull0 + 8 * acc_i, accph);
      if (tr_a && kb < 1024) tr[2 * 1024 + kb] = clock64();
      tc_fence_after();
      const uint32_t tempty_b = tempty0 + 8 * acc_i;
      const uint32_t taddr = tmem_base + t_lane + acc_i * 256 + half * 128;
      if (V & 4) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t v[64];
          tmem_ld_32x32b_x64(taddr + 64 * c, v);
          tmem_wait_ld_dep64(v);
          if (c == 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) { if (CG == 2) mbar_arrive_leader_addr(tempty_b); else mbar_arrive_addr(tempty_b); }
            if (tr_a && kb < 1024) tr[3 * 1024 + kb] = clock64();
          }
#pragma unroll
          for (int i = 0; i < 64; i += 2)
            ffma2(acc[64 * c + i], acc[64 * c + i + 1], __uint_as_float(v[i]), __uint_as_float(v[i + 1]), s);
        }
      } else {
        uint32_t va[32], vb[32];
        tmem_ld_32x32b_x32(taddr, va);
        tmem_ld_32x32b_x32(taddr + 32, vb);
        tmem_wait_ld_dep2(va, vb);
#pragma unroll
        for (int c = 0; c < 4; c += 2) {
          const bool more = c + 2 < 4;
#pragma unroll
          for (int i = 0; i < 32; i += 2)
            ffma2(acc[32 * c + i], acc[32 * c + i + 1], __uint_as_float(va[i]), __uint_as_float(va[i + 1]), s);
          if (more) tmem_ld_32x32b_x32(taddr + 32 * (c + 2), va);
#pragma unroll
          for (int i = 0; i < 32; i += 2)
            ffma2(acc[32 * c + 32 + i], acc[32 * c + 33 + i], __uint_as_float(vb[i]), __uint_as_float(vb[i + 1]), s);
          if (more) {
            tmem_ld_32x32b_x32(taddr + 32 * (c + 3), vb);
            tmem_wait_ld_dep2(va, vb);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) { if (CG == 2) mbar_arrive_leader_addr(tempty_b); else mbar_arrive_addr(tempty_b); }
            if (tr_a && kb < 1024) tr[3 * 1024 + kb] = clock64();
          }
        }
      }
      if (++acc_i == 2) { acc_i = 0; accph ^= 1; }
    }
    float x = 0.f;
#pragma unroll
    for (int i = 0; i < 128; ++i) x += acc[i];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = x;
  }
  __syncthreads();
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<CG>(ld_shared_u32(smem_u32(&slot)), 512);
  }
}

static unsigned long long* g_out;
static float* g_sink;
static unsigned long long* g_tr;

template <int V, int CG = 2>
void run(const char* name) {
  const int nk = 56;  // the DeepSeek-V3 gate+up tile depth; launched as many "tiles" back to back
  const int smem = kS * (16384 + (CG == 2 ? 16384 : 32768)) + (130 * 56) * 4 + 2048;
  cudaFuncSetAttribute(kloop<V, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
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
  const int nk_run = 1024;  // one long "tile": the loop itself, no tile boundaries
  (void)nk;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, kloop<V, CG>, nk_run, g_out, g_sink, g_tr, 1.0f);
    cudaEventRecord(e1);
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  static unsigned long long t[4 * 1024];
  cudaMemcpy(t, g_tr, sizeof(t), cudaMemcpyDeviceToHost);
  auto med = [&](int a, int b, int sh) {
    static double v[1024];
    int n = 0;
    for (int i = 100; i < 1000; ++i) v[n++] = double(t[a * 1024 + i]) - double(t[b * 1024 + i - sh]);
    std::sort(v, v + n);
    return v[n / 2];
  };
  const double flops = 148.0 * 128 * 256 * 128 * 2.0 * nk_run;  // per SM: 128 rows x 256 columns either way
  printf("%-40s %7.1f TFLOP/s  period %5.0f clk | issue->issued %4.0f | issued->promo full %5.0f | drain %4.0f | "
         "freed->issue(i+2) %4.0f\n",
         name, flops / (best * 1e-3) / 1e12, med(0, 0, 1), med(1, 0, 0), med(2, 1, 0), med(3, 2, 0), med(0, 3, 2));
}

int main() {
  cudaMalloc(&g_out, 148 * 8);
  cudaMalloc(&g_sink, 148 * kThreads * 4);
  cudaMalloc(&g_tr, 4 * 1024 * 8);
  cudaMemset(g_tr, 0, 4 * 1024 * 8);
  for (int pass = 0; pass < 2; ++pass) {
    run<1 | 8, 2>("pair M=256 (kernel-like)");
    run<1 | 8, 1>("1-CTA M=128 N=256");
    run<8, 1>("1-CTA, constant scale");
  }
  return 0;
}
