// tagg_gemm.cu -- B200 (sm_100a) padding-free FP8 grouped GEMM.
//
// Semantics (the reference's run_adaptive, engine.py:184-343):
//   for every group g, row i < M_g, column n:
//     acc = 0
//     for kb ascending: acc = acc + inner_kb(i, n) * fl(SA[row, kb] * SB_g[kb, n / 128])
//     C[c_row0(g) + i, n] = bf16_rne(acc)
//
// One persistent CTA per SM walks a static tile schedule.  The tile -> group
// map comes from a prefix sum over the DEVICE group sizes, computed in each
// CTA's prologue with no host sync.  Warp roles:
//   warp 0 : TMA producer.  A [128 x 128] and B [128 x 128] boxes go into
//            128B-swizzled smem (S-stage mbarrier ring).  The tile's S_A rows
//            arrive by one over-fetching 1-D bulk copy whose start slides back
//            row_prev rows onto a 16-byte boundary (prefetch.py:50-72).
//   warp 1 : TMEM allocator + single-thread tcgen05.mma issuer.  Per 128-K
//            block it issues 4 x kind::f8f6f4 (M=128, N=128, K=32) into a fresh
//            TMEM accumulator (4 buffers x 128 columns = all 512 columns).
//   warps 2-9 : promotion + epilogue.  Each thread owns one row and 64
//            columns.  Per k-block it does tcgen05.ld of the partial,
//            s = fl(sa * sb), acc += partial * s in fp32 registers (FFMA2, or
//            FMUL+FADD with TAGG_FLAG_EXACT_PROMOTION), ascending kb.  At tile
//            end: bf16 -> swizzled smem staging -> TMA store.  Full tiles use
//            the 128-row descriptor.  Residual tiles pick d = 2^floor(log2 res)
//            from the 8-entry store pool and issue the dual-phase store
//            (descriptors.py:95-106), so no row past M_g is ever written.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "tagg.h"
#include "tagg_ptx.cuh"

namespace tagg {

constexpr int BM = 128, BN = 128, BK = 128;
constexpr int kNumAcc = 4;  // TMEM accumulation buffers of BN columns
constexpr uint32_t kTmemCols = 512;
constexpr int kNumPromoWarps = 8;
constexpr int kThreads = 64 + 32 * kNumPromoWarps;
constexpr int kMaxStages = 8;
constexpr uint32_t kStageBytesA = BM * BK;
constexpr uint32_t kStageBytesB = BK * BN;
constexpr uint32_t kChunkBytesC = BM * 128;  // 128 rows x 64 bf16 columns
constexpr uint32_t kCStagingBytes = 2 * kChunkBytesC;
constexpr int kPoolSize = 8;  // heights 1, 2, ..., 128 (descriptors.py:31-35)

struct Params {
  CUtensorMap tmap_a;
  CUtensorMap tmap_b;
  CUtensorMap tmap_c[kPoolSize];
  const float* sa;
  const float* sb;
  const int32_t* group_sizes;
  const int64_t* c_row_offsets;
  int32_t* tile_map;
  int64_t m_alloc;
  int64_t sb_sg, sb_skb, sb_snb;
  int32_t G, N, K, kb_count, n_tiles, sa_rb, b_kmajor, b_shared;
  uint32_t stages, sa_buf_bytes;
  uint32_t off_a, off_b, off_c, off_sa, off_tab, off_bar;
};

struct Tile {
  int g, mt, n0, row0, valid, crow0;
};

__device__ __forceinline__ Tile decode_tile(int t, const int32_t* tab_tile, const int32_t* tab_row,
                                            const int32_t* tab_size, const int32_t* tab_crow, int G) {
  int lo = 0, hi = G - 1;  // largest g with tab_tile[g] <= t
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (tab_tile[mid] <= t) lo = mid; else hi = mid - 1;
  }
  Tile T;
  T.g = lo;
  const int l = t - tab_tile[lo];
  const int m = tab_size[lo];
  const int mtiles = (m + BM - 1) / BM;
  T.mt = l % mtiles;
  T.n0 = (l / mtiles) * BN;
  T.row0 = tab_row[lo] + T.mt * BM;
  T.valid = min(BM, m - T.mt * BM);
  T.crow0 = tab_crow[lo] + T.mt * BM;
  return T;
}

// prefetch.py:50-72: smallest row_prev in [0, 16) that puts the window start
// on a 16-byte boundary (the S_A base itself is 16-byte aligned).
__device__ __forceinline__ int sa_row_prev(int64_t row0, int rb) {
  const int64_t addr = row0 * rb;
  int rp = 0;
  while (((addr - static_cast<int64_t>(rp) * rb) & 15) != 0 && rp < 15) ++rp;
  return rp;
}

template <bool kExact, bool kSwizzleC>
__global__ void __launch_bounds__(kThreads, 1) tagg_gemm_kernel(const __grid_constant__ Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t S = p.stages;
  const int G = p.G;

  uint8_t* sA = smem + p.off_a;
  uint8_t* sB = smem + p.off_b;
  uint8_t* sC = smem + p.off_c;
  uint8_t* sSA = smem + p.off_sa;
  int32_t* tab_tile = reinterpret_cast<int32_t*>(smem + p.off_tab);  // [G+1]
  int32_t* tab_row = tab_tile + (G + 1);                                // [G+1]
  int32_t* tab_size = tab_row + (G + 1);                                // [G]
  int32_t* tab_crow = tab_size + G;                                     // [G]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* tfull = bars + 2 * S;
  uint64_t* tempty = tfull + kNumAcc;
  uint64_t* safull = tempty + kNumAcc;
  uint64_t* saempty = safull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(saempty + 2);

  // ------------------------------------------------------------ prologue
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.tmap_a);
    prefetch_tmap(&p.tmap_b);
    for (uint32_t i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < kNumAcc; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kNumPromoWarps);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&safull[i], 1);
      mbar_init(&saempty[i], kNumPromoWarps);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
  if (warp == 2) {
    // device-side prefix sums over M_g: row offsets and tile offsets
    int carry_r = 0, carry_t = 0;
    for (int base = 0; base < G; base += 32) {
      const int g = base + lane;
      const int m = (g < G) ? max(0, p.group_sizes[g]) : 0;
      const int tl = ((m + BM - 1) / BM) * p.n_tiles;
      int im = m, it = tl;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, im, o);
        const int y = __shfl_up_sync(0xffffffffu, it, o);
        if (lane >= o) { im += x; it += y; }
      }
      if (g < G) {
        tab_row[g] = carry_r + im - m;
        tab_tile[g] = carry_t + it - tl;
        tab_size[g] = m;
        tab_crow[g] = p.c_row_offsets ? static_cast<int32_t>(p.c_row_offsets[g]) : carry_r + im - m;
      }
      carry_r += __shfl_sync(0xffffffffu, im, 31);
      carry_t += __shfl_sync(0xffffffffu, it, 31);
    }
    if (lane == 0) {
      tab_row[G] = carry_r;
      tab_tile[G] = carry_t;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = tab_tile[G];
  const int kbc = p.kb_count;
  const int rb = p.sa_rb;

  if (warp == 0) {
    // ========================================================== TMA producer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, sab = 0, saph = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        const Tile T = decode_tile(t, tab_tile, tab_row, tab_size, tab_crow, G);
        const int gb = p.b_shared ? 0 : T.g;
        // ---- S_A over-fetch window (one 1-D bulk copy per tile)
        mbar_wait(&saempty[sab], saph ^ 1);
        const int rp = sa_row_prev(T.row0, rb);
        const int64_t start_row = static_cast<int64_t>(T.row0) - rp;
        const int64_t want = ((static_cast<int64_t>(rp + BM) * rb) + 15) & ~int64_t(15);
        int64_t avail = (p.m_alloc - start_row) * rb;
        if (avail < 0) avail = 0;
        const int64_t lim = min(want, avail);
        const uint32_t bulk = static_cast<uint32_t>(lim & ~int64_t(15));
        const uint32_t tail = static_cast<uint32_t>(lim) - bulk;
        uint8_t* dst = sSA + sab * p.sa_buf_bytes;
        const uint8_t* src = reinterpret_cast<const uint8_t*>(p.sa) + start_row * rb;
        for (uint32_t i = 0; i < tail; i += 4)  // < 16 B at the very end of S_A
          *reinterpret_cast<float*>(dst + bulk + i) = __ldg(reinterpret_cast<const float*>(src + bulk + i));
        mbar_arrive_expect_tx(&safull[sab], bulk);
        if (bulk) bulk_load_1d(dst, src, bulk, &safull[sab]);
        if (++sab == 2) { sab = 0; saph ^= 1; }
        // ---- A / B k-blocks
        for (int kb = 0; kb < kbc; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], kStageBytesA + kStageBytesB);
          tma_load_2d(&p.tmap_a, &full[stage], sA + stage * kStageBytesA, kb * BK, T.row0);
          if (p.b_kmajor)
            tma_load_3d(&p.tmap_b, &full[stage], sB + stage * kStageBytesB, kb * BK, T.n0, gb);
          else
            tma_load_3d(&p.tmap_b, &full[stage], sB + stage * kStageBytesB, T.n0, kb * BK, gb);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ========================================================== MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_e4m3_f32(BM, BN, p.b_kmajor == 0);
      uint32_t stage = 0, phase = 0, acc = 0, accph = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        for (int kb = 0; kb < kbc; ++kb) {
          mbar_wait(&tempty[acc], accph ^ 1);
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * kStageBytesA);
          const uint32_t b_base = smem_u32(sB + stage * kStageBytesB);
          const uint32_t d_tmem = tmem_base + acc * BN;
#pragma unroll
          for (int k = 0; k < BK / 32; ++k) {
            const uint64_t ad = umma_desc_sw128(a_base + k * 32, 16, 1024);
            const uint64_t bd = p.b_kmajor ? umma_desc_sw128(b_base + k * 32, 16, 1024)
                                           : umma_desc_sw128(b_base + k * 32 * BN, kStageBytesB, 1024);
            mma_f8f6f4(d_tmem, ad, bd, idesc, k > 0 ? 1u : 0u);
          }
          mma_commit(&empty[stage]);  // smem slot free once these MMAs retire
          mma_commit(&tfull[acc]);    // k-block partial ready for promotion
          if (++stage == S) { stage = 0; phase ^= 1; }
          if (++acc == kNumAcc) { acc = 0; accph ^= 1; }
        }
      }
    }
  } else {
    // ========================================================== promotion + epilogue
    const int pw = warp - 2;
    const int q = warp & 3;          // TMEM lane quarter this warp may access
    const int half = pw >> 2;        // column half [64*half, 64*half + 64)
    const int r = 32 * q + lane;     // tile row owned by this thread
    const int ptid = threadIdx.x - 64;
    const uint32_t t_lane = static_cast<uint32_t>(32 * q) << 16;
    uint32_t acc_i = 0, accph = 0, sab = 0, saph = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      const Tile T = decode_tile(t, tab_tile, tab_row, tab_size, tab_crow, G);
      const int rp = sa_row_prev(T.row0, rb);
      const float* sbp = p.sb + (p.b_shared ? 0 : static_cast<int64_t>(T.g) * p.sb_sg) +
                         static_cast<int64_t>(T.n0 >> 7) * p.sb_snb;
      mbar_wait(&safull[sab], saph);
      const float* sa_row = reinterpret_cast<const float*>(sSA + sab * p.sa_buf_bytes +
                                                           static_cast<uint32_t>(rp + r) * rb);
      float acc[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) acc[i] = 0.0f;
      float sb_next = __ldg(sbp);
      for (int kb = 0; kb < kbc; ++kb) {
        const float sbv = sb_next;
        if (kb + 1 < kbc) sb_next = __ldg(sbp + static_cast<int64_t>(kb + 1) * p.sb_skb);
        const float s = __fmul_rn(sa_row[kb], sbv);
        mbar_wait(&tfull[acc_i], accph);
        tc_fence_after();
        uint32_t v0[32], v1[32];
        const uint32_t taddr = tmem_base + t_lane + acc_i * BN + half * 64;
        tmem_ld_32x32b_x32(taddr, v0);
        tmem_ld_32x32b_x32(taddr + 32, v1);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc_i]);
        if (++acc_i == kNumAcc) { acc_i = 0; accph ^= 1; }
        if constexpr (kExact) {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            acc[i] = __fadd_rn(acc[i], __fmul_rn(__uint_as_float(v0[i]), s));
            acc[32 + i] = __fadd_rn(acc[32 + i], __fmul_rn(__uint_as_float(v1[i]), s));
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            ffma2(acc[i], acc[i + 1], __uint_as_float(v0[i]), __uint_as_float(v0[i + 1]), s);
            ffma2(acc[32 + i], acc[33 + i], __uint_as_float(v1[i]), __uint_as_float(v1[i + 1]), s);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&saempty[sab]);
      if (++sab == 2) { sab = 0; saph ^= 1; }

      // ---- epilogue: bf16 -> smem staging -> TMA store (pool + dual phase)
      if (ptid == 0) bulk_wait_read0();  // previous tile's stores have read the staging
      named_bar_sync(1, 32 * kNumPromoWarps);
      const uint32_t row_addr = smem_u32(sC + half * kChunkBytesC) + static_cast<uint32_t>(r) * 128u;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t w0 = pack_bf16x2(acc[8 * j + 0], acc[8 * j + 1]);
        const uint32_t w1 = pack_bf16x2(acc[8 * j + 2], acc[8 * j + 3]);
        const uint32_t w2 = pack_bf16x2(acc[8 * j + 4], acc[8 * j + 5]);
        const uint32_t w3 = pack_bf16x2(acc[8 * j + 6], acc[8 * j + 7]);
        const uint32_t c16 = kSwizzleC ? static_cast<uint32_t>(j ^ (r & 7)) : static_cast<uint32_t>(j);
        st_shared_v4(row_addr + c16 * 16u, w0, w1, w2, w3);
      }
      fence_proxy_async_smem();
      named_bar_sync(1, 32 * kNumPromoWarps);
      if (ptid == 0) {
        const int lg = 31 - __clz(T.valid);  // pool index: d = 2^floor(log2 valid)
        const int d = 1 << lg;
        for (int h = 0; h < 2; ++h) {
          const int col = T.n0 + 64 * h;
          if (col >= p.N) break;
          const uint8_t* chunk = sC + h * kChunkBytesC;
          // phase a: smem rows [0, d) -> rows [crow0, crow0 + d)
          tma_store_2d(&p.tmap_c[lg], chunk, col, T.crow0);
          // phase b: smem rows [valid - d, valid) -> rows [crow0 + valid - d, crow0 + valid)
          // (for a full tile, or a power-of-two residual, both phases coincide:
          // a full tile issues one store, as engine.py:318-322 does)
          if (T.valid != BM)
            tma_store_2d(&p.tmap_c[lg], chunk + static_cast<uint32_t>(T.valid - d) * 128u, col,
                         T.crow0 + T.valid - d);
        }
        bulk_commit();
        if (p.tile_map) {
          int32_t* rec = p.tile_map + static_cast<int64_t>(t) * TAGG_TILE_MAP_FIELDS;
          rec[0] = T.g;
          rec[1] = T.mt;
          rec[2] = T.n0;
          rec[3] = T.row0;
          rec[4] = T.valid;
          rec[5] = d;
          rec[6] = T.crow0;
          rec[7] = T.valid - d;
          rec[8] = T.crow0 + T.valid - d;
        }
      }
    }
    if (ptid == 0) bulk_wait0();
  }

  // ------------------------------------------------------------ teardown
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

// ====================================================================== host
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

int num_sms_for_current_device() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (dev < 0 || dev >= 64) return -1;
  if (!cached[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    cached[dev] = n;
  }
  return cached[dev];
}

bool encode(CUtensorMap* m, CUtensorMapDataType dt, uint32_t rank, const void* base, const uint64_t* dims,
            const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle sw) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t d[5], s[4];
  cuuint32_t b[5], e[5];
  for (uint32_t i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
    if (i + 1 < rank) s[i] = strides_bytes[i];
  }
  CUresult r = fn(m, dt, rank, const_cast<void*>(base), d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

int gcd_int(int a, int b) {
  while (b) {
    const int t = a % b;
    a = b;
    b = t;
  }
  return a;
}

}  // namespace

// Smem layout for a given stage count; returns total bytes (incl. alignment slack).
static uint32_t smem_layout(Params& p, uint32_t stages, int G, int rb) {
  // row_prev < 16 / gcd(rb, 16): the residue class of row0*rb mod 16 has that period
  const int rp_max = 16 / gcd_int(rb, 16) - 1;
  const uint32_t sa_buf = align_up(static_cast<uint32_t>(((rp_max + BM) * rb + 15) & ~15), 128);
  p.stages = stages;
  p.sa_buf_bytes = sa_buf;
  p.off_a = 0;
  p.off_b = stages * kStageBytesA;
  p.off_c = p.off_b + stages * kStageBytesB;
  p.off_sa = p.off_c + kCStagingBytes;
  p.off_tab = p.off_sa + 2 * sa_buf;
  const uint32_t tab_bytes = align_up(4u * static_cast<uint32_t>(2 * (G + 1) + 2 * G), 16);
  p.off_bar = p.off_tab + tab_bytes;
  const uint32_t bar_bytes = (2 * stages + 2 * kNumAcc + 4) * 8 + 16;
  return p.off_bar + bar_bytes + 1024;
}

template <bool kExact, bool kSwizzleC>
static cudaError_t launch(const Params& p, uint32_t smem_bytes, int grid, cudaStream_t stream) {
  auto kern = tagg_gemm_kernel<kExact, kSwizzleC>;
  static uint32_t configured = 0;  // max dynamic smem already granted to this instance
  if (smem_bytes > configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e != cudaSuccess) return e;
    configured = 232448;
  }
  kern<<<grid, kThreads, smem_bytes, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace tagg

using namespace tagg;

extern "C" int64_t tagg_max_tiles(int64_t m_alloc, int G, int N) {
  if (m_alloc < 0 || G < 1 || N < 1) return 0;
  return ((m_alloc + BM - 1) / BM + G) * ((N + BN - 1) / BN);
}

extern "C" int tagg_grouped_gemm_fp8(const void* a, int64_t lda, const float* sa, int64_t m_alloc,
                                     const void* b, int b_layout, int b_experts, const float* sb,
                                     int64_t sb_stride_g, int64_t sb_stride_kb, int64_t sb_stride_nb,
                                     const int32_t* group_sizes, int G, int N, int K, void* c, int64_t ldc,
                                     int64_t c_rows, const int64_t* c_row_offsets, int32_t* tile_map,
                                     uint32_t flags, void* stream) {
  // ---- ProblemConfig rules (engine.py:77-92) and operand checks (engine.py:132-142)
  if (K < 16 || K % 16 != 0) return TAGG_ERR_CONFIG;
  if (N < 64 || N % 64 != 0) return TAGG_ERR_CONFIG;
  if (G < 1) return TAGG_ERR_CONFIG;
  if (b_layout != TAGG_B_KN && b_layout != TAGG_B_NK) return TAGG_ERR_CONFIG;
  if (b_experts != 1 && b_experts != G) return TAGG_ERR_SHAPE;
  if (m_alloc < 0 || c_rows < 0 || lda < K || ldc < N) return TAGG_ERR_SHAPE;
  if (!a || !sa || !b || !sb || !group_sizes || !c) return TAGG_ERR_SHAPE;
  // ---- global alignment rules (memory.py:27, GLOBAL_ALIGNMENT = 16)
  auto mis = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) != 0; };
  if (mis(a) || mis(sa) || mis(b) || mis(c) || (lda % 16) != 0 || ((ldc * 2) % 16) != 0)
    return TAGG_ERR_ALIGNMENT;
  if (m_alloc == 0 || c_rows == 0) return TAGG_OK;  // nothing can be stored
  if (m_alloc >= (int64_t(1) << 31) || c_rows >= (int64_t(1) << 31)) return TAGG_ERR_UNSUPPORTED;

  const int kb_count = (K + BK - 1) / BK;
  const int rb = 4 * kb_count;
  Params p;
  std::memset(&p, 0, sizeof(p));
  p.sa = sa;
  p.sb = sb;
  p.group_sizes = group_sizes;
  p.c_row_offsets = c_row_offsets;
  p.tile_map = tile_map;
  p.m_alloc = m_alloc;
  p.sb_sg = sb_stride_g;
  p.sb_skb = sb_stride_kb;
  p.sb_snb = sb_stride_nb;
  p.G = G;
  p.N = N;
  p.K = K;
  p.kb_count = kb_count;
  p.n_tiles = (N + BN - 1) / BN;
  p.sa_rb = rb;
  p.b_kmajor = (b_layout == TAGG_B_NK) ? 1 : 0;
  p.b_shared = (b_experts == 1) ? 1 : 0;

  uint32_t smem_bytes = 0;
  uint32_t stages = kMaxStages;
  for (; stages >= 2; --stages) {
    smem_bytes = smem_layout(p, stages, G, rb);
    if (smem_bytes <= 232448) break;
  }
  if (stages < 2) return TAGG_ERR_UNSUPPORTED;

  // ---- tensor maps: A, B, and the C store pool (8 heights)
  {
    const uint64_t dims[2] = {static_cast<uint64_t>(K), static_cast<uint64_t>(m_alloc)};
    const uint64_t str[1] = {static_cast<uint64_t>(lda)};
    const uint32_t box[2] = {BK, BM};
    if (!encode(&p.tmap_a, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, a, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return TAGG_ERR_CUDA;
  }
  {
    uint64_t dims[3], str[2];
    const uint32_t box[3] = {128, 128, 1};
    if (b_layout == TAGG_B_KN) {
      dims[0] = N; dims[1] = K; dims[2] = b_experts;
      str[0] = N; str[1] = static_cast<uint64_t>(K) * N;
    } else {
      dims[0] = K; dims[1] = N; dims[2] = b_experts;
      str[0] = K; str[1] = static_cast<uint64_t>(K) * N;
    }
    if (!encode(&p.tmap_b, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, b, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return TAGG_ERR_CUDA;
  }
  const bool swz = (flags & TAGG_FLAG_PLAIN_C_STAGING) == 0;
  for (int i = 0; i < kPoolSize; ++i) {
    const uint64_t dims[2] = {static_cast<uint64_t>(N), static_cast<uint64_t>(c_rows)};
    const uint64_t str[1] = {static_cast<uint64_t>(ldc) * 2};
    const uint32_t box[2] = {64, 1u << i};
    if (!encode(&p.tmap_c[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, c, dims, str, box,
                swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE))
      return TAGG_ERR_CUDA;
  }

  const int sms = num_sms_for_current_device();
  if (sms <= 0) return TAGG_ERR_CUDA;
  const int64_t max_tiles = tagg_max_tiles(m_alloc, G, N);
  const int grid = static_cast<int>(std::min<int64_t>(sms, max_tiles));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool exact = (flags & TAGG_FLAG_EXACT_PROMOTION) != 0;
  cudaError_t e;
  if (exact)
    e = swz ? launch<true, true>(p, smem_bytes, grid, st) : launch<true, false>(p, smem_bytes, grid, st);
  else
    e = swz ? launch<false, true>(p, smem_bytes, grid, st) : launch<false, false>(p, smem_bytes, grid, st);
  if (e != cudaSuccess) {
    std::fprintf(stderr, "tagg_grouped_gemm_fp8: launch failed: %s\n", cudaGetErrorString(e));
    return TAGG_ERR_CUDA;
  }
  return TAGG_OK;
}
