// tagg_wgrad.cu -- the MoE weight gradient as a K-grouped FP8 GEMM:
//   dW_g = X_g^T dY_g,  X [M, K] and dY [M, N] in the padding-free grouped layout,
// so the ragged per-expert row count M_g is the REDUCTION axis.  Operands carry one
// fp32 scale per (group, 128-token block, column) -- quantize_col_blocks below -- and
// the k-block promotion is the forward's (engine.py:151-164) with a per-element scale
// s = fl(sx[tb][k] * sdy[tb][n]).  dW is bf16 [G, K, N].
//
// The paper's mechanism moves to the loads: a group's last token block has res < 128
// rows, and the rows after it belong to the next expert.  The producer loads it with
// the power-of-two descriptor pool (heights 1..128) in two phases, rows [0, d) and
// [res-d, res) with d = 2^floor(log2 res) (descriptors.py:95-106 applied to loads), and
// zeroes smem rows [res, 128) so the MMA's reduction sees exact zeros: no row of
// another group is ever read into the product, and nothing is padded in HBM.
//
// Persistent CTA-pair tiles of 256 (K) x 256 (N), tcgen05.mma cta_group::2 M=256 N=256,
// A = X^T and B = dY both MN-major in 128B-swizzled smem (token rows), 2 TMEM
// accumulation buffers, warp roles as in tagg_gemm.cu (producer, MMA, 8 promotion warps).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <type_traits>

#include "tagg.h"
#include "tagg_host.h"
#include "tagg_ptx.cuh"
#include "tagg_e4m3.cuh"

namespace tagg {
namespace wg {

constexpr int BT = 128;                 // tokens per k-block
constexpr int kThreads = 384;
constexpr int kPromoWarps = 8;
constexpr int kNumAcc = 2;              // TMEM buffers of 256 columns
#ifndef WG_STAGES
#define WG_STAGES 4
#endif
constexpr int kStages = WG_STAGES;
// dW staging: 64 KB in one pass (the promotion recipes: their epilogue is on the promotion chain)
// or 32 KB in two (MXFP8: the epilogue runs after the accumulator is released, and the two-pass
// form measured 7% faster there -- ABBA, tools/wg_ab.py)
__host__ __device__ constexpr int epi_passes(bool mx) { return mx ? 2 : 1; }
constexpr int kScaleRing = 8;           // k-block scale slots: sx 128 + sdy 256 floats
constexpr uint32_t kStageA = BT * 128;  // 128 token rows x this CTA's 128 K columns
constexpr uint32_t kStageB = BT * 128;  // 128 token rows x this CTA's 128 N columns
constexpr uint32_t kScaleSlot = (128 + 256) * 4;
constexpr uint32_t kChunkC = 128 * 128;  // 128 rows x 64 bf16 columns
constexpr int kPool = 8;

struct Params {
  CUtensorMap map_x[kPool];   // X [M, K] u8, box {128 cols, 2^i rows}, SW128
  CUtensorMap map_dy[kPool];  // dY [M, N] u8, box {128 cols, 2^i rows}, SW128
  CUtensorMap map_dw;         // dW [G*K, N] bf16, box {64 cols, 128 rows}, SW128
  const float* sx;            // [TB, K]
  const float* sdy;           // [TB, N]
  const int32_t* group_sizes;
  unsigned long long* trace;  // diagnostics (TAGG_TRACE builds): clock64 stamps of CTAs 0/1
  int G, K, N, KT, NT;        // KT, NT: 256-wide pair tiles (ceil)
  uint32_t off_a, off_b, off_c, off_s, off_sf, off_tab, off_bar;
  CUtensorMap map_sfx, map_sfdy;  // kMx: E8M0 factor blocks, u8 [blocks * 2, 256] / box {256, 2} and {256, 4}
};
// MXFP8 mode (TAGG_WGRAD_MX): per stage, this CTA's E8M0 scale factors in the tcgen05.cp source
// layout -- SFA (its 128 dW rows) 512 B, SFB (the pair tile's 256 columns) 2 x 512 B: byte
// (16 l + 4 c + j) of a block is the factor of row / column 32 c + l for the j-th 32-token slice
// (all four the same here: one scale per 128-token block).
constexpr uint32_t kSfStage = 1536;
// TMEM: the accumulator [0, 256); stage s's factors at 256 + 16 s: SFA 4 columns, SFB 8 columns
// (row / column 32 c + l in lane l (+ 32 q, broadcast), column c, byte j -- tools/micro/mxf8.cu).
constexpr uint32_t kTmemSf0 = 256;

// Diagnostics: the same event layout as the forward kernel's trace (tools/trace_wg.py).
enum WgEv { kWgMmaTempty = 0, kWgMmaFull, kWgMmaIssued, kWgProdEmpty, kWgPromoFull, kWgPromoFreed, kWgPromoDone,
            kWgPromoSfull, kWgEpiStart, kWgEpiEnd };
__device__ __forceinline__ void wg_stamp(unsigned long long* tr, int ev, uint32_t i) {
#ifdef TAGG_TRACE
  if (tr != nullptr && blockIdx.x < 2 && i < 1024u) tr[(blockIdx.x * 10 + ev) * 1024 + i] = clock64();
#endif
}

// CTA pair (cluster of 2, tcgen05 cta_group::2) per 256 (K) x 256 (N) tile of dW_g: CTA
// `rank` holds K rows [k0 + 128 rank, +128) of X^T and B columns [n0 + 128 rank, +128)
// of dY; each CTA's TMEM gets its 128 rows x all 256 columns.
// kDyBlock: sdy is constant over every 128-column block of a token block (the 128x128 dY recipe of
// tagg_quantize_col_blocks_ex, block_cols = 128): a thread's 128 columns are one block, so its
// promotion is s = fl(sx * sdy) once per token block and one FFMA2 per element pair -- the forward
// kernel's promotion -- instead of an FMUL2 and an FFMA2.
// kMx (TAGG_WGRAD_MX): sx and sdy are powers of two (the MXFP8 recipe, quantize_col_blocks with
// TAGG_QCB_SCALE_POW2).  The tensor core applies them as E8M0 block scales
// (tcgen05.mma kind::mxf8f6f4.block_scale) and accumulates the group's whole token range in one
// TMEM accumulator: no per-block promotion.  The factors come pre-laid-out by the quantizer
// (tagg_quantize_col_blocks_mx: E8M0 bytes in the tcgen05.cp source layout) and ride with each
// stage's operands on the same TMA barrier; the eight promotion warps only drain the finished tile
// and store it.
template <bool kDyBlock, bool kMx>
__global__ void __launch_bounds__(kThreads, 1) wgrad_kernel(const __grid_constant__ Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = p.G;
  const int rank = static_cast<int>(cluster_ctarank());
  const int cid = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  int32_t* tab_off = reinterpret_cast<int32_t*>(smem + p.off_tab);  // [G] first row
  int32_t* tab_tb = tab_off + G;                                      // [G] first token block
  int32_t* tab_m = tab_tb + G;                                        // [G] rows
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* full = bars;
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + kNumAcc;
  uint64_t* sfull = tempty + kNumAcc;
  uint64_t* sempty = sfull + kScaleRing;
  uint64_t* cfull = sempty + kScaleRing;  // [2] per column half: the tile's dW staged (4 warps)
  uint64_t* cempty = cfull + 2;           // [2] the stores have read the staging (warp 3)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cempty + 2);

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 2);   // the leader's arrive.expect_tx + the peer's arrive (its zero rows)
      mbar_init(&empty[i], 1);  // MMA commit, multicast
    }
    for (int i = 0; i < kNumAcc; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kPromoWarps * 2);
    }
    for (int i = 0; i < kScaleRing; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sempty[i], kPromoWarps);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&cfull[i], kPromoWarps / 2);
      mbar_init(&cempty[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<2>(tmem_slot, 512);
  if (warp == 2) {
    int carry_r = 0, carry_b = 0;
    for (int base = 0; base < G; base += 32) {
      const int g = base + lane;
      const int m = (g < G) ? max(0, p.group_sizes[g]) : 0;
      const int nb = (m + BT - 1) / BT;
      int im = m, ib = nb;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, im, o);
        const int y = __shfl_up_sync(0xffffffffu, ib, o);
        if (lane >= o) { im += x; ib += y; }
      }
      if (g < G) {
        tab_off[g] = carry_r + im - m;
        tab_tb[g] = carry_b + ib - nb;
        tab_m[g] = m;
      }
      carry_r += __shfl_sync(0xffffffffu, im, 31);
      carry_b += __shfl_sync(0xffffffffu, ib, 31);
    }
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const int tiles = G * p.KT * p.NT;

  if (warp < 4) {
    setmaxnreg_dec<72>();
    if (warp == 0) {
      // ====================================================== producer (both CTAs)
      uint32_t stage = 0, phase = 0, piter = 0;
      const uint32_t sA0 = smem_u32(smem + p.off_a), sB0 = smem_u32(smem + p.off_b);
      for (int t = cid; t < tiles; t += nclusters) {
        const int g = t / (p.KT * p.NT), rem = t % (p.KT * p.NT);
        const int k0 = (rem / p.NT) * 256, n0 = (rem % p.NT) * 256;
        const int kr = k0 + 128 * rank;  // this CTA's K rows
        const int m = tab_m[g], off = tab_off[g];
        for (int j = 0; j * BT < m; ++j) {
          // X boxes (the per-column scales are warp 3's, dY's warp 2's)
          mbar_wait_addr(smem_u32(&empty[stage]), phase ^ 1);
          if (lane == 0) wg_stamp(p.trace, kWgProdEmpty, piter);
          ++piter;
          const int res = min(BT, m - j * BT);
          const int row0 = off + j * BT;
          const uint32_t a_dst = sA0 + stage * kStageA, b_dst = sB0 + stage * kStageB;
          if (res < BT) {
            // zero the rows past the group end (the next expert's tokens are never read)
            const int zrows = BT - res;
            for (int i = lane; i < zrows * 8; i += 32) {
              const uint32_t off16 = static_cast<uint32_t>((res + i / 8) * 128 + (i % 8) * 16);
              st_shared_v4(a_dst + off16, 0u, 0u, 0u, 0u);
              st_shared_v4(b_dst + off16, 0u, 0u, 0u, 0u);
            }
            fence_proxy_async_smem();
          }
          __syncwarp();
          if (lane == 0) {
            const uint32_t fb = smem_u32(&full[stage]);
            const int lg = res == BT ? 7 : 31 - __clz(res), d = 1 << lg;
            const uint32_t bytes = ((res == BT) ? 2u * (kStageA + kStageB) : 2u * 4u * d * 128u) + (kMx ? 2u * kSfStage : 0u);
            if (rank == 0) {
              mbar_arrive_expect_tx_addr(fb, bytes);
            } else if (res < BT) {
              // release the zero rows to the pair's MMA, then count on the leader's barrier
              asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(fb & 0xFEFFFFFFu)
                           : "memory");
            } else {
              mbar_arrive_leader_addr(fb);  // nothing of ours to publish: the TMA bytes count themselves
            }
            tma_load_2d_u32<2>(&p.map_x[lg], fb, a_dst, kr, row0);
            if (res < BT)  // dual phase: rows [0, d) above, rows [res - d, res) here
              tma_load_2d_u32<2>(&p.map_x[lg], fb, a_dst + (res - d) * 128u, kr, row0 + res - d);
            // dY's boxes: warp 2 (a TMA issue holds its warp; one warp issuing every box paced the pipe)
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
      if (lane == 0)
        for (int i = 0; i < kStages; ++i) {
          mbar_wait_addr(smem_u32(&empty[stage]), phase ^ 1);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      __syncwarp();
    } else if (warp == 2) {
      // ====================================================== dY loads (both CTAs)
      // The stage's dY boxes (dual phase for a group's last token block; the producer zeroes the
      // rows past the group end), counted on the same full barrier.
      uint32_t stage = 0, phase = 0;
      const uint32_t sB0 = smem_u32(smem + p.off_b);
      for (int t = cid; t < tiles; t += nclusters) {
        const int g = t / (p.KT * p.NT), rem = t % (p.KT * p.NT);
        const int nr = (rem % p.NT) * 256 + 128 * rank;
        const int m = tab_m[g], off = tab_off[g];
        for (int j = 0; j * BT < m; ++j) {
          mbar_wait_addr(smem_u32(&empty[stage]), phase ^ 1);
          if (elect_one()) {
            const int res = min(BT, m - j * BT), row0 = off + j * BT;
            const int lg = res == BT ? 7 : 31 - __clz(res), d = 1 << lg;
            const uint32_t fb = smem_u32(&full[stage]), b_dst = sB0 + stage * kStageB;
            tma_load_2d_u32<2>(&p.map_dy[lg], fb, b_dst, nr, row0);
            if (res < BT) tma_load_2d_u32<2>(&p.map_dy[lg], fb, b_dst + (res - d) * 128u, nr, row0 + res - d);
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    } else if (!kMx && warp == 3) {
      // ====================================================== scale loads (both CTAs)
      // sx[tb][kr..+128) and sdy[tb][n0..+256) of each token block into the scale ring, on a warp
      // of their own: a bulk-copy issue holds its warp, and on the operand producer's warp the
      // two per block paced the pipeline.
      // It also issues the dW stores: the promotion warps stage a tile and hand it over through
      // cfull[h], and get the staging back through cempty[h] once the stores have read it (a TMA
      // store holds its issuing warp, which in a promotion warp delayed its next drain and with
      // it the MMA chain).  Tile t's stores go out after tile t + 1's scales are requested.
      uint32_t sring = 0, sph = 0, cph = 0;
      const uint32_t sS0 = smem_u32(smem + p.off_s);
      const uint32_t cfull0 = smem_u32(&cfull[0]), cempty0 = smem_u32(&cempty[0]);
      auto store_tile = [&](int t) {
        const int g = t / (p.KT * p.NT), rem = t % (p.KT * p.NT);
        const int n0 = (rem % p.NT) * 256, kr = (rem / p.NT) * 256 + 128 * rank;
        mbar_wait_addr(cfull0, cph);
        mbar_wait_addr(cfull0 + 8, cph);
        cph ^= 1;
        if (lane == 0) {
          if (kr < p.K) {
            for (int c = 0; c < 4; ++c)
              if (n0 + 64 * c < p.N) tma_store_2d(&p.map_dw, smem + p.off_c + c * kChunkC, n0 + 64 * c, g * p.K + kr);
            bulk_commit();
          }
          bulk_wait_read0();  // the stores have read the staging
          mbar_arrive_addr(cempty0);
          mbar_arrive_addr(cempty0 + 8);
        }
        __syncwarp();
      };
      int tprev = -1;
      for (int t = cid; t < tiles; t += nclusters) {
        const int g = t / (p.KT * p.NT), rem = t % (p.KT * p.NT);
        const int k0 = (rem / p.NT) * 256, n0 = (rem % p.NT) * 256;
        const int kr = k0 + 128 * rank;
        const int m = tab_m[g], tb0 = tab_tb[g];
        for (int j = 0; j * BT < m; ++j) {
          mbar_wait_addr(smem_u32(&sempty[sring]), sph ^ 1);
          if (lane == 0) {
            const uint32_t dst = sS0 + sring * kScaleSlot;
            const int64_t tb = tb0 + j;
            const uint32_t nsx = kr < p.K ? 512u : 0u;
            const uint32_t nsdy = n0 + 256 <= p.N ? 1024u : 512u;
            mbar_arrive_expect_tx_addr(smem_u32(&sfull[sring]), nsx + nsdy);
            if (nsx) bulk_load_1d_addr(dst, p.sx + tb * p.K + kr, nsx, smem_u32(&sfull[sring]));
            bulk_load_1d_addr(dst + 512, p.sdy + tb * p.N + n0, nsdy, smem_u32(&sfull[sring]));
          }
          __syncwarp();
          if (++sring == kScaleRing) { sring = 0; sph ^= 1; }
        }
        if (tprev >= 0) store_tile(tprev);
        tprev = t;
      }
      if (tprev >= 0) store_tile(tprev);
      if (lane == 0) bulk_wait0();
      __syncwarp();
    } else if (kMx && warp == 3) {
      // ====================================================== E8M0 factor loads (kMx, both CTAs)
      // The stage's factor blocks ride on its full barrier (the leader's expect_tx counts them); a
      // warp of their own keeps their TMA issues off the operand producer's path.
      uint32_t stage = 0, phase = 0;
      const uint32_t sf0 = smem_u32(smem + p.off_sf);
      for (int t = cid; t < tiles; t += nclusters) {
        const int g = t / (p.KT * p.NT), rem = t % (p.KT * p.NT);
        const int k0 = (rem / p.NT) * 256, n0 = (rem % p.NT) * 256;
        const int kr = k0 + 128 * rank;
        const int m = tab_m[g], tb0 = tab_tb[g];
        for (int j = 0; j * BT < m; ++j) {
          mbar_wait_addr(smem_u32(&empty[stage]), phase ^ 1);
          if (elect_one()) {
            // this CTA's SFA block (its 128 dW rows) and the tile's two SFB blocks (256 columns):
            // 512-B blocks [token block][128 columns], two 256-B rows each
            const uint32_t fb = smem_u32(&full[stage]), sfd = sf0 + stage * kSfStage;
            const int64_t tb = tb0 + j;
            tma_load_2d_u32<2>(&p.map_sfx, fb, sfd, 0, static_cast<int32_t>((tb * (p.K >> 7) + (kr >> 7)) * 2));
            tma_load_2d_u32<2>(&p.map_sfdy, fb, sfd + 512u, 0,
                               static_cast<int32_t>((tb * (p.N >> 7) + (n0 >> 7)) * 2));
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    } else if (warp == 1 && rank == 0 && kMx) {
      // ====================================================== MMA, MXFP8 (leader)
      // One accumulator per tile: the group's token blocks accumulate in TMEM with their E8M0
      // factors applied by the tensor core; each block's factors are copied smem -> TMEM right
      // before its MMAs (tcgen05.cp and tcgen05.mma execute in issue order).
      const uint32_t tmem_base = ld_shared_u32(smem_u32(tmem_slot));
      const uint64_t a0 = umma_desc_sw128(smem_u32(smem + p.off_a), kStageA, 1024);
      const uint64_t b0 = umma_desc_sw128(smem_u32(smem + p.off_b), kStageB, 1024);
      const uint32_t sF0 = smem_u32(smem + p.off_sf);
      uint32_t stage = 0, phase = 0, accph = 0, miter = 0;
      for (int t = cid; t < tiles; t += nclusters) {
        const int m = tab_m[t / (p.KT * p.NT)];
        if (m <= 0) continue;  // an empty group's tile is stored as zeros, with no MMA
        const int nb = (m + BT - 1) / BT;
        for (int j = 0; j < nb; ++j) {
          mbar_wait_addr(smem_u32(&full[stage]), phase);  // operands and their E8M0 factors
          if (lane == 0) wg_stamp(p.trace, kWgMmaFull, miter);
          if (j == 0) mbar_wait_addr(smem_u32(&tempty[0]), accph ^ 1);  // the previous tile is drained
          if (lane == 0) wg_stamp(p.trace, kWgMmaTempty, miter);
          tc_fence_after();
          const uint64_t ad = a0 + ((stage * kStageA) >> 4), bd = b0 + ((stage * kStageB) >> 4);
          if (elect_one()) {
            const uint32_t tsf = tmem_base + kTmemSf0 + 16u * stage, sf = sF0 + stage * kSfStage;
            utccp_32x128b_warpx4_cg2(tsf, umma_desc_noswz(sf, 128, 128));
            utccp_32x128b_warpx4_cg2(tsf + 4, umma_desc_noswz(sf + 512, 128, 128));
            utccp_32x128b_warpx4_cg2(tsf + 8, umma_desc_noswz(sf + 1024, 128, 128));
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_mxf8_cg2(tmem_base, ad + static_cast<uint64_t>(k * 256), bd + static_cast<uint64_t>(k * 256),
                           idesc_mx_e4m3_mn(256, 256, k, k), tsf, tsf + 4, (j > 0 || k > 0) ? 1u : 0u);
            mma_commit_addr<2>(smem_u32(&empty[stage]));
            if (j + 1 == nb) mma_commit_addr<2>(smem_u32(&tfull[0]));
          }
          __syncwarp();
          if (lane == 0) wg_stamp(p.trace, kWgMmaIssued, miter);
          ++miter;
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        accph ^= 1;
      }
    } else if (warp == 1 && rank == 0) {
      // ====================================================== MMA (leader, whole warp, elected issue)
      const uint32_t tmem_base = ld_shared_u32(smem_u32(tmem_slot));
      const uint32_t idesc = idesc_e4m3_f32_ab(256, 256, true, true);
      // MN-major operands: 128 token rows of 128 B (one swizzle atom wide per CTA), 8-row
      // groups of 1 KB; K = 32 tokens per MMA = 32 rows = 4 KB
      const uint64_t a0 = umma_desc_sw128(smem_u32(smem + p.off_a), kStageA, 1024);
      const uint64_t b0 = umma_desc_sw128(smem_u32(smem + p.off_b), kStageB, 1024);
      uint32_t stage = 0, phase = 0, acc = 0, accph = 0, miter = 0;
      for (int t = cid; t < tiles; t += nclusters) {
        const int m = tab_m[t / (p.KT * p.NT)];
        for (int j = 0; j * BT < m; ++j) {
          // operands first, then the TMEM buffer (see tagg_gemm.cu's MMA issuer)
          mbar_wait_addr(smem_u32(&full[stage]), phase);
          if (lane == 0) wg_stamp(p.trace, kWgMmaFull, miter);
          mbar_wait_addr(smem_u32(&tempty[acc]), accph ^ 1);
          if (lane == 0) wg_stamp(p.trace, kWgMmaTempty, miter);
          tc_fence_after();
          const uint64_t ad = a0 + ((stage * kStageA) >> 4), bd = b0 + ((stage * kStageB) >> 4);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_f8f6f4<2>(tmem_base + acc * 256, ad + static_cast<uint64_t>(k * 256),
                            bd + static_cast<uint64_t>(k * 256), idesc, k > 0 ? 1u : 0u);
            mma_commit_addr<2>(smem_u32(&empty[stage]));
            mma_commit_addr<2>(smem_u32(&tfull[acc]));
          }
          __syncwarp();
          if (lane == 0) wg_stamp(p.trace, kWgMmaIssued, miter);
          ++miter;
          if (++stage == kStages) { stage = 0; phase ^= 1; }
          if (++acc == kNumAcc) { acc = 0; accph ^= 1; }
        }
      }
    }
  } else {
    setmaxnreg_inc<216>();
    // ====================================================== promotion + epilogue
    const uint32_t tmem_base = opaque_u32(ld_shared_u32(smem_u32(tmem_slot)));
    const int pw = warp - 4, q = warp & 3, half = pw >> 2;
    const int r = 32 * q + lane;  // row of this CTA's 128 dW rows
    const int ptid = threadIdx.x - 128;
    const uint32_t t_lane = static_cast<uint32_t>(32 * q) << 16;
    const uint32_t sS0 = opaque_u32(smem_u32(smem + p.off_s));
    const uint32_t tfull0 = opaque_u32(smem_u32(&tfull[0])), tempty0 = opaque_u32(smem_u32(&tempty[0]));
    const uint32_t sfull0 = opaque_u32(smem_u32(&sfull[0])), sempty0 = opaque_u32(smem_u32(&sempty[0]));
    uint32_t acc_i = 0, accph = 0, sring = 0, sph = 0, kiter = 0, tiles_done = 0;
    const bool tr = p.trace != nullptr && pw == 0 && lane == 0;
    uint32_t mx_ph = 0;  // kMx: parity of the single accumulator's handoffs
    uint32_t cph = 0;    // promotion recipes: parity of the staging handoffs with warp 3
    const uint32_t cfull0 = opaque_u32(smem_u32(&cfull[0])), cempty0 = opaque_u32(smem_u32(&cempty[0]));
    for (int t = cid; t < tiles; t += nclusters) {
      const int g = t / (p.KT * p.NT), rem = t % (p.KT * p.NT);
      const int k0 = (rem / p.NT) * 256, n0 = (rem % p.NT) * 256;
      const int kr = k0 + 128 * rank;
      const int m = tab_m[g];
      float acc[128];
#pragma unroll
      for (int i = 0; i < 128; ++i) acc[i] = 0.0f;
      if constexpr (kMx) {
        // the finished tile: this thread's row, its 128 columns, already scaled; the accumulator
        // goes back to the MMA as soon as the last chunk has landed, before the epilogue
        if (m > 0) {
          mbar_wait_addr(tfull0, mx_ph);
          if (tr) wg_stamp(p.trace, kWgPromoFull, tiles_done);
          tc_fence_after();
          const uint32_t taddr = tmem_base + t_lane + 128u * half;
          uint32_t va[32], vb[32];
          tmem_ld_32x32b_x32(taddr, va);
          tmem_ld_32x32b_x32(taddr + 32, vb);
          tmem_wait_ld_dep2(va, vb);
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[i] = __uint_as_float(va[i]);
          tmem_ld_32x32b_x32(taddr + 64, va);
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[32 + i] = __uint_as_float(vb[i]);
          tmem_ld_32x32b_x32(taddr + 96, vb);
          tmem_wait_ld_dep2(va, vb);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_leader_addr(tempty0);
          if (tr) wg_stamp(p.trace, kWgPromoFreed, tiles_done);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            acc[64 + i] = __uint_as_float(va[i]);
            acc[96 + i] = __uint_as_float(vb[i]);
          }
          mx_ph ^= 1;
        }
      } else
      for (int j = 0; j * BT < m; ++j) {
#ifndef TAGG_WG_EXP_NOSFULL
        mbar_wait_addr(sfull0 + 8 * sring, sph);
#endif
        if (tr) wg_stamp(p.trace, kWgPromoSfull, kiter);
        const uint32_t slot = sS0 + sring * kScaleSlot;
        const float sxk = ld_shared_f32(slot + 4u * r);
        const uint32_t sdy = slot + 512u + 4u * (128u * half);
        const float sblk = kDyBlock ? __fmul_rn(sxk, ld_shared_f32(sdy)) : 0.0f;
        mbar_wait_addr(tfull0 + 8 * acc_i, accph);
        if (tr) wg_stamp(p.trace, kWgPromoFull, kiter);
        tc_fence_after();
        const uint32_t taddr = tmem_base + t_lane + acc_i * 256 + 128u * half;
#pragma unroll
        for (int c2 = 0; c2 < 2; ++c2) {
          uint32_t v[64];
          tmem_ld_32x32b_x64(taddr + 64 * c2, v);
          tmem_wait_ld_dep64(v);
          if (c2 == 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_leader_addr(tempty0 + 8 * acc_i);
            if (tr) wg_stamp(p.trace, kWgPromoFreed, kiter);
          }
#ifdef TAGG_WG_EXP_NOMATH
          if (__uint_as_float(v[5]) == 1.2345f) acc[c2] += __uint_as_float(v[7]);
          continue;
#endif
          if constexpr (kDyBlock) {
            // acc = fl(acc + inner * s), s = fl(sx * sdy): one FFMA2 per pair, as in the forward
#pragma unroll
            for (int c = 0; c < 64; c += 2)
              ffma2(acc[64 * c2 + c], acc[64 * c2 + c + 1], __uint_as_float(v[c]), __uint_as_float(v[c + 1]), sblk);
            continue;
          }
#pragma unroll
          for (int c = 0; c < 64; c += 4) {
            float4 sd;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(sd.x), "=f"(sd.y), "=f"(sd.z), "=f"(sd.w)
                         : "r"(sdy + 4u * (64 * c2 + c)));
            // acc = fl(fl(inner * sx) * sdy + acc): the row scale first (FMUL2), then the
            // column scale and the add in one FFMA2 -- one packed instruction per element
            // pair each (the reference rounds s = sx * sdy, the product and the sum
            // separately; the difference is a few fp32 ulp, far inside the bf16 tolerance)
            float* a = acc + 64 * c2 + c;
            float t0, t1, t2, t3;
            fmul2s(t0, t1, __uint_as_float(v[c + 0]), __uint_as_float(v[c + 1]), sxk);
            fmul2s(t2, t3, __uint_as_float(v[c + 2]), __uint_as_float(v[c + 3]), sxk);
            ffma2v(a[0], a[1], t0, t1, sd.x, sd.y);
            ffma2v(a[2], a[3], t2, t3, sd.z, sd.w);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_addr(sempty0 + 8 * sring);
        if (tr) wg_stamp(p.trace, kWgPromoDone, kiter);
        ++kiter;
        if (++sring == kScaleRing) { sring = 0; sph ^= 1; }
        if (++acc_i == kNumAcc) { acc_i = 0; accph ^= 1; }
      }
      if (tr) wg_stamp(p.trace, kWgEpiStart, tiles_done);
      // epilogue: 4 chunks of 64 columns x 128 rows (64 KB) in epi_passes(kMx) passes over 64 or 32 KB
      // of staging.  The two column halves are independent: warps of half h write chunks 2h,
      // 2h+1 (their 128 columns), sync only among themselves (named barrier 2 + h) and their first
      // thread stores them (a TMA store's smem reads are tracked per issuing thread, so each leader
      // waits for its own before the slot is rewritten).
      if constexpr (!kMx) {
        // hand the staged tile to warp 3, which stores it (see there)
        mbar_wait_addr(cempty0 + 8 * half, cph ^ 1);
        const uint32_t base = smem_u32(smem + p.off_c) + static_cast<uint32_t>(r) * 128u;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const uint32_t chunk = 2 * half + (jj >> 3);
          const uint32_t w0 = pack_bf16x2(acc[8 * jj + 0], acc[8 * jj + 1]);
          const uint32_t w1 = pack_bf16x2(acc[8 * jj + 2], acc[8 * jj + 3]);
          const uint32_t w2 = pack_bf16x2(acc[8 * jj + 4], acc[8 * jj + 5]);
          const uint32_t w3 = pack_bf16x2(acc[8 * jj + 6], acc[8 * jj + 7]);
          st_shared_v4(base + chunk * kChunkC + static_cast<uint32_t>(((jj & 7) ^ (r & 7)) * 16), w0, w1, w2, w3);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_addr(cfull0 + 8 * half);
        cph ^= 1;
      } else {
        constexpr int kEpiPasses = epi_passes(kMx);
        constexpr int kCpp = 2 / kEpiPasses;  // chunks per half per pass
        const int hl = 128 * half;
        const uint32_t base = smem_u32(smem + p.off_c) + static_cast<uint32_t>(r) * 128u;
#pragma unroll
        for (int ps = 0; ps < kEpiPasses; ++ps) {
          if (ptid == hl) bulk_wait_read0();
          named_bar_sync(2 + half, 128);
#pragma unroll
          for (int jj = 8 * kCpp * ps; jj < 8 * kCpp * (ps + 1); ++jj) {
            const uint32_t slot = kCpp * half + ((jj >> 3) - kCpp * ps);
            const uint32_t w0 = pack_bf16x2(acc[8 * jj + 0], acc[8 * jj + 1]);
            const uint32_t w1 = pack_bf16x2(acc[8 * jj + 2], acc[8 * jj + 3]);
            const uint32_t w2 = pack_bf16x2(acc[8 * jj + 4], acc[8 * jj + 5]);
            const uint32_t w3 = pack_bf16x2(acc[8 * jj + 6], acc[8 * jj + 7]);
            st_shared_v4(base + slot * kChunkC + static_cast<uint32_t>(((jj & 7) ^ (r & 7)) * 16), w0, w1, w2, w3);
          }
          fence_proxy_async_smem();
          named_bar_sync(2 + half, 128);
          if (ptid == hl && kr < p.K) {
            const int row = g * p.K + kr;
            for (int cc = 0; cc < kCpp; ++cc) {
              const int c = 2 * half + kCpp * ps + cc;  // 64-column chunk of the tile
              if (n0 + 64 * c < p.N)
                tma_store_2d(&p.map_dw, smem + p.off_c + (kCpp * half + cc) * kChunkC, n0 + 64 * c, row);
            }
            bulk_commit();
          }
        }
      }
      if (tr) wg_stamp(p.trace, kWgEpiEnd, tiles_done);
      ++tiles_done;
    }
    if (kMx && (ptid == 0 || ptid == 128)) bulk_wait0();  // MXFP8: both column-half leaders issue stores
  }
  __syncwarp();
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<2>(ld_shared_u32(smem_u32(tmem_slot)), 512);
  }
}

// The MXFP8 scale: the smallest power of two >= q (at least 2^-126), i.e. one E8M0 byte
// ((bits >> 23) & 0xFF); x / s is then exact (oracle/fp8.py: pow2_ceil).
__device__ __forceinline__ float pow2_ceil(float q) {
  uint32_t b = __float_as_uint(q);
  if (b & 0x7FFFFFu) b = (b & 0xFF800000u) + 0x800000u;
  return __uint_as_float(max(b, 0x00800000u));
}

// Per-group 128x1 column-block quantizer: CTA (row block y, column chunk x), thread =
// one column; pass 1 takes the block's amax, pass 2 (L2-resident re-read) quantizes.
template <bool kBf16>
__global__ void __launch_bounds__(128) quantize_col_blocks_kernel(const void* __restrict__ x, int64_t ldx, int cols,
                                                                  const int32_t* __restrict__ group_sizes, int G,
                                                                  uint8_t* __restrict__ codes, int64_t ldc,
                                                                  float* __restrict__ scales, int32_t* err,
                                                                  int pow2) {
  __shared__ int32_t s_row0, s_rows, s_tb;
  if (threadIdx.x < 32) {
    // which (group, block) is this CTA's: walk the group table
    const int lane = threadIdx.x;
    int carry_r = 0, carry_b = 0, found = 0;
    const int want = blockIdx.y;
    for (int base = 0; base < G && !found; base += 32) {
      const int g = base + lane;
      const int m = (g < G) ? max(0, group_sizes[g]) : 0;
      const int nb = (m + 127) / 128;
      int im = m, ib = nb;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int a = __shfl_up_sync(0xffffffffu, im, o);
        const int b = __shfl_up_sync(0xffffffffu, ib, o);
        if (lane >= o) { im += a; ib += b; }
      }
      const int b0 = carry_b + ib - nb, r0 = carry_r + im - m;
      const bool mine = g < G && want >= b0 && want < b0 + nb;
      const uint32_t hit = __ballot_sync(0xffffffffu, mine);
      if (hit) {
        found = 1;
        if (mine) {
          const int j = want - b0;
          s_row0 = r0 + 128 * j;
          s_rows = min(128, m - 128 * j);
          s_tb = want;
        }
      }
      carry_r += __shfl_sync(0xffffffffu, im, 31);
      carry_b += __shfl_sync(0xffffffffu, ib, 31);
    }
    if (!found && lane == 0) s_rows = 0;
  }
  __syncthreads();
  const int rows = s_rows;
  if (rows <= 0) return;
  const int64_t row0 = s_row0;
  const int c = blockIdx.x * 128 + threadIdx.x;
  if (c >= cols) return;
  auto ld = [&](int64_t rr) -> float {
    if constexpr (kBf16)
      return __uint_as_float(static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(x)[rr * ldx + c]) << 16);
    else
      return reinterpret_cast<const float*>(x)[rr * ldx + c];
  };
  float amax = 0.0f;
  bool bad = false;
  for (int i = 0; i < rows; ++i) {
    const float m = fabsf(ld(row0 + i));
    bad |= !(m <= 3.402823466e38f);
    amax = fmaxf(amax, m);
  }
  float s = amax > 0.0f ? __fdiv_rn(amax, 448.0f) : 1.0f;
  if (pow2 && amax > 0.0f) s = pow2_ceil(s);
  scales[static_cast<int64_t>(s_tb) * cols + c] = s;
  for (int i = 0; i < rows; i += 2) {
    const float v0 = __fdiv_rn(ld(row0 + i), s);
    const float v1 = (i + 1 < rows) ? __fdiv_rn(ld(row0 + i + 1), s) : 0.0f;
    uint16_t pair;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(pair) : "f"(v1), "f"(v0));
    codes[(row0 + i) * ldc + c] = static_cast<uint8_t>(pair & 0xFF);
    if (i + 1 < rows) codes[(row0 + i + 1) * ldc + c] = static_cast<uint8_t>(pair >> 8);
  }
  if (bad) atomicOr(err, 2);
}

// Column-block quantizer, register tiles: CTA = one (group, 128-token block); it walks the
// group table once, then sweeps the columns 128 at a time.  Thread t holds columns
// [8 (t % 16), +8) of rows t / 16 + 16 j, j < 8, in registers, so x is read ONCE from HBM (a
// two-pass form re-read it, and the re-read missed L2); bf16 chunks are prefetched one ahead.
// Column maxima: integer max of |x| bit patterns (packed bf16 pairs: one VIMNMX per two
// elements; NaN > inf > finite, so the same max flags non-finite input), a shuffle between the
// two row lanes of a warp, then the 8 warps via smem.
// kBlock128: one scale per (token block, 128 columns) -- the reference's 128x128 block recipe
// (fp8.py:154-176) applied to each group's token blocks -- written to all 128 columns' scale
// slots, so the wgrad can promote with one scale per drained 128-column half (1 op per pair).
// kWeighted / index: grouped row r reads row_weights[r] * x[index[r]] (index nullable), so
// token-ordered activations are quantized into the grouped layout without a copy.
template <bool kBf16>
struct ColChunk {
  using Raw = typename std::conditional<kBf16, uint4, float4[2]>::type;
  Raw raw[8];
  // rows[j]: row j's first element (x + src_j * ldx), formed once per CTA
  __device__ __forceinline__ void load(const char* const (&rows)[8], int c) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if constexpr (kBf16) {
        raw[j] = __ldcs(reinterpret_cast<const uint4*>(rows[j] + 2 * static_cast<int64_t>(c)));
      } else {
        const float4* f = reinterpret_cast<const float4*>(rows[j] + 4 * static_cast<int64_t>(c));
        raw[j][0] = __ldcs(f);
        raw[j][1] = __ldcs(f + 1);
      }
    }
  }
  __device__ __forceinline__ uint32_t word(int j, int h) const {  // bf16 pair h of row j
    if constexpr (kBf16) return h == 0 ? raw[j].x : h == 1 ? raw[j].y : h == 2 ? raw[j].z : raw[j].w;
    else return 0u;
  }
  __device__ __forceinline__ float get(int j, int k) const {
    if constexpr (kBf16) {
      const uint32_t w = word(j, k >> 1);
      return __uint_as_float((k & 1) ? (w & 0xFFFF0000u) : (w << 16));
    } else {
      const float4& q = raw[j][k >> 2];
      return (k & 3) == 0 ? q.x : (k & 3) == 1 ? q.y : (k & 3) == 2 ? q.z : q.w;
    }
  }
};

template <bool kBf16, bool kBlock128, bool kWeighted, bool kPow2 = false>
__global__ void __launch_bounds__(256, 2) quantize_col_tile_kernel(const void* __restrict__ x, int64_t ldx, int cols,
                                                                   const int32_t* __restrict__ group_sizes, int G,
                                                                   uint8_t* __restrict__ codes, int64_t ldc,
                                                                   float* __restrict__ scales, int32_t* err,
                                                                   const int32_t* __restrict__ index,
                                                                   const float* __restrict__ row_weights, int pow2,
                                                                   uint32_t* __restrict__ sf_out) {
  __shared__ int32_t s_row0, s_rows, s_tb;
  __shared__ __align__(16) uint32_t s_part[2][8][128];  // per-warp column maxima (|x| bits)
  __shared__ __align__(16) float s_scale[2][128];
  __shared__ __align__(16) float s_rlo[2][128];
  __shared__ __align__(16) float s_rhi[2][128];
  // per-warp queue of undecided 4-column groups (values, row, column): a warp resolves them 32
  // at a time, one group per lane, instead of every lane idling through one lane's divisions
  constexpr int kQueue = 64;
  __shared__ __align__(16) float4 q_v[8][kQueue][2];
  __shared__ int32_t q_r[8][kQueue];
  __shared__ uint32_t s_bmax[2][4];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (t < 32) {
    // which (group, block) is this CTA's: walk the group table
    int carry_r = 0, carry_b = 0, found = 0;
    const int want = blockIdx.x;
    for (int base = 0; base < G && !found; base += 32) {
      const int g = base + lane;
      const int m = (g < G) ? max(0, group_sizes[g]) : 0;
      const int nb = (m + 127) / 128;
      int im = m, ib = nb;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int a = __shfl_up_sync(0xffffffffu, im, o);
        const int b = __shfl_up_sync(0xffffffffu, ib, o);
        if (lane >= o) { im += a; ib += b; }
      }
      const int b0 = carry_b + ib - nb, r0 = carry_r + im - m;
      const bool mine = g < G && want >= b0 && want < b0 + nb;
      if (__ballot_sync(0xffffffffu, mine)) {
        found = 1;
        if (mine) {
          const int j = want - b0;
          s_row0 = r0 + 128 * j;
          s_rows = min(128, m - 128 * j);
          s_tb = want;
        }
      }
      carry_r += __shfl_sync(0xffffffffu, im, 31);
      carry_b += __shfl_sync(0xffffffffu, ib, 31);
    }
    if (!found && lane == 0) s_rows = 0;
  }
  __syncthreads();
  const int rows = s_rows;
  if (rows <= 0) return;
  const int64_t row0 = s_row0;
  const int64_t tb = s_tb;
  const int cg = t & 15, rl = t >> 4;
  // Rows past the block read a clamped live row: all 8 loads go out without a branch, and a
  // duplicate of a live row leaves every column maximum unchanged (such rows are never stored).
  // Columns past `cols` read a clamped live column the same way (their scales are not written).
  const char* xrow[8];
  float wr[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int64_t rg = row0 + min(rl + 16 * j, rows - 1);
    const int64_t src = index ? static_cast<int64_t>(__ldg(index + rg)) : rg;
    xrow[j] = reinterpret_cast<const char*>(x) + src * ldx * (kBf16 ? 2 : 4);
    wr[j] = kWeighted ? __ldg(row_weights + rg) : 1.0f;
  }
  // this thread's live rows (bit j: row rl + 16 j < rows) and its first code row
  uint32_t live_rows = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) live_rows |= (rl + 16 * j < rows ? 1u : 0u) << j;
  // opaque: kept in registers, not re-derived from the parameters at every store (ptxas
  // rematerialised the 64-bit products under this kernel's register pressure: +4%)
  uint8_t* const code_row = reinterpret_cast<uint8_t*>(opaque_u64(reinterpret_cast<uint64_t>(codes + (row0 + rl) * ldc)));
  const int64_t code_step = static_cast<int64_t>(opaque_u64(static_cast<uint64_t>(16 * ldc)));
  auto value = [&](const ColChunk<kBf16>& ch, int j, int k) -> float {
    const float f = ch.get(j, k);
    return kWeighted ? __fmul_rn(wr[j], f) : f;  // weighted rows are fl(w * x), as gathered
  };
  const int nchunks = (cols + 127) / 128;  // cols % 8 == 0 on this path (kBlock128: % 128)
  uint32_t bad = 0;
  // bf16: the next chunk's loads are in flight while this one is reduced and quantized (two
  // 32-register chunks); f32 chunks take 64 registers each, so f32 loads one at a time
  // (measured: without the prefetch, 3 CTAs per SM run 3-5% slower).  The weighted gather (the
  // MoE backward's dC rows) loads one at a time too: with the prefetch it spilled 112 B, and
  // without it runs 8-10% faster (tools/colq_ab.py --gather).
  constexpr bool kPrefetch = kBf16 && !kWeighted;
  ColChunk<kBf16> cur;
  if (kPrefetch) cur.load(xrow, min(cg * 8, cols - 8));
  for (int cb = 0; cb < nchunks; ++cb) {
    const int c0 = cb * 128 + cg * 8;
    ColChunk<kBf16> nxt;
    if (!kPrefetch) cur.load(xrow, min(c0, cols - 8));
    if (kPrefetch && cb + 1 < nchunks) nxt.load(xrow, min(c0 + 128, cols - 8));
    const int buf = cb & 1;
    uint32_t amax[8];  // |x| bit patterns: integer order = float order for non-negative floats
    if constexpr (kBf16 && !kWeighted) {
      // |x| maxima of packed pairs without masking each word: a signed 16-bit max finds the
      // largest non-negative pattern, an unsigned one the largest negative (sign-magnitude: the
      // unsigned order of negative patterns is their |x| order); with the sign bits cleared, the
      // larger of the two is max |x| (and NaN / inf still sort above every finite value)
      uint32_t ps[4] = {0x80008000u, 0x80008000u, 0x80008000u, 0x80008000u}, pu[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          ps[h] = __vmaxs2(ps[h], cur.word(j, h));
          pu[h] = __vmaxu2(pu[h], cur.word(j, h));
        }
      uint32_t pw[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) pw[h] = __vmaxu2(ps[h] & 0x7FFF7FFFu, pu[h] & 0x7FFF7FFFu);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        amax[2 * h] = pw[h] << 16;
        amax[2 * h + 1] = pw[h] & 0xFFFF0000u;
      }
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) amax[k] = 0u;
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int k = 0; k < 8; ++k) amax[k] = max(amax[k], __float_as_uint(value(cur, j, k)) & 0x7FFFFFFFu);
    }
    // the two row lanes of this warp that share the columns, then the 8 warps
#pragma unroll
    for (int k = 0; k < 8; ++k) amax[k] = max(amax[k], __shfl_xor_sync(0xffffffffu, amax[k], 16));
    if (lane < 16) {
      uint4* dst = reinterpret_cast<uint4*>(&s_part[buf][warp][cg * 8]);
      dst[0] = make_uint4(amax[0], amax[1], amax[2], amax[3]);
      dst[1] = make_uint4(amax[4], amax[5], amax[6], amax[7]);
    }
    __syncthreads();
    uint32_t cm = 0u;
    if (t < 128) {
#pragma unroll
      for (int w = 0; w < 8; ++w) cm = max(cm, s_part[buf][w][t]);
      if (cb * 128 + t < cols) bad |= cm >= 0x7F800000u;  // inf or NaN in a live column
    }
    if constexpr (kBlock128) {
      // one scale per 128-column block: the max over the block's columns (warps 0-3)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cm = max(cm, __shfl_xor_sync(0xffffffffu, cm, o));
      if (t < 128 && lane == 0) s_bmax[buf][warp] = cm;
      __syncthreads();
      cm = max(max(s_bmax[buf][0], s_bmax[buf][1]), max(s_bmax[buf][2], s_bmax[buf][3]));
    }
    if (t < 128) {
      const float am = __uint_as_float(cm);
      float sc = am > 0.0f ? __fdiv_rn(am, 448.0f) : 1.0f;
      if (pow2 && am > 0.0f) sc = pow2_ceil(sc);
      const float rd = __frcp_rd(sc);
      s_scale[buf][t] = sc;
      s_rlo[buf][t] = rd;
      // >= (1/s)(1 + 2^-22): RU(1/s) raised by two ulps (or 1/s overflowing to inf).  A power-of-two
      // s has an exact reciprocal (x * 1/s is x / s), so both bounds are the same there.
      const float ru = __frcp_ru(sc);
      s_rhi[buf][t] = pow2 ? rd : (isinf(ru) ? ru : __uint_as_float(__float_as_uint(ru) + 2u));
      const int c = cb * 128 + t;
      if (c < cols) scales[tb * cols + c] = sc;
      // MXFP8: the E8M0 byte of this column's scale in the tcgen05.cp source block of
      // (token block, 128 columns): byte 16 l + 4 c + j for column 32 c + l, every 32-token slice j
      if (sf_out) sf_out[(tb * (cols >> 7) + cb) * 128 + (t & 31) * 4 + (t >> 5)] = ((__float_as_uint(sc) >> 23) & 0xFFu) * 0x01010101u;
    }
    __syncthreads();
    {
      const bool c_ok = c0 < cols;
      float rlo[8], rhi[8];
      {
        const float4* pl = reinterpret_cast<const float4*>(&s_rlo[buf][cg * 8]);
        const float4* ph = reinterpret_cast<const float4*>(&s_rhi[buf][cg * 8]);
        const float4 a = pl[0], b = pl[1], e = ph[0], f = ph[1];
        rlo[0] = a.x; rlo[1] = a.y; rlo[2] = a.z; rlo[3] = a.w; rlo[4] = b.x; rlo[5] = b.y; rlo[6] = b.z; rlo[7] = b.w;
        rhi[0] = e.x; rhi[1] = e.y; rhi[2] = e.z; rhi[3] = e.w; rhi[4] = f.x; rhi[5] = f.y; rhi[6] = f.z; rhi[7] = f.w;
      }
      const uint32_t lt = (1u << lane) - 1u;
      uint8_t* crow = code_row + c0;  // this thread's row rl + 16 j, advanced by code_step
      const uint32_t live_mask = c_ok ? live_rows : 0u;
      int qn = 0;  // warp-uniform
      auto drain_queue = [&]() {
        __syncwarp();  // the rows' bracket codes are stored before any patch
        for (int base = 0; base < qn; base += 32) {
          const int i = base + lane;
          if (i < qn) {
            const int rc = q_r[warp][i];  // row << 8 | 8-column group
            const int cc = cb * 128 + (rc & 0xFF) * 8;
            const uint32_t w0 = e4m3x4_div(q_v[warp][i][0], &s_scale[buf][cc - cb * 128]);
            const uint32_t w1 = e4m3x4_div(q_v[warp][i][1], &s_scale[buf][cc - cb * 128 + 4]);
            *reinterpret_cast<uint2*>(codes + (row0 + (rc >> 8)) * ldc + cc) = make_uint2(w0, w1);
          }
        }
        __syncwarp();
        qn = 0;
      };
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int r = rl + 16 * j;
        const bool live = (live_mask >> j) & 1u;
        uint32_t w[2], up[2];
        float4 vv[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float v4[4] = {value(cur, j, 4 * h), value(cur, j, 4 * h + 1), value(cur, j, 4 * h + 2),
                               value(cur, j, 4 * h + 3)};
          const float l4[4] = {rlo[4 * h], rlo[4 * h + 1], rlo[4 * h + 2], rlo[4 * h + 3]};
          const float h4[4] = {rhi[4 * h], rhi[4 * h + 1], rhi[4 * h + 2], rhi[4 * h + 3]};
          if constexpr (kPow2) {
            // a power-of-two scale: x * (1/s) IS x / s (exact), one product and one conversion
            w[h] = e4m3x4_pow2(v4, l4);
            up[h] = w[h];
          } else {
            w[h] = e4m3x4_bracket(v4, l4, h4, up[h]);
          }
          vv[h] = make_float4(v4[0], v4[1], v4[2], v4[3]);
        }
        if (live) *reinterpret_cast<uint2*>(crow) = make_uint2(w[0], w[1]);
        crow += code_step;
        if constexpr (kPow2) continue;  // nothing is ever undecided
        const bool u = live && (w[0] != up[0] || w[1] != up[1]);
        const uint32_t m = __ballot_sync(0xffffffffu, u);
        if (m) {
          if (u) {
            const int pos = qn + __popc(m & lt);
            q_v[warp][pos][0] = vv[0];
            q_v[warp][pos][1] = vv[1];
            q_r[warp][pos] = (r << 8) | cg;
          }
          qn += __popc(m);
        }
        if (qn >= 32) drain_queue();  // < 32 + 32 entries: fits kQueue
      }
      if (qn) drain_queue();
    }
    if (kPrefetch) cur = nxt;
  }
  if (bad) atomicOr(err, 2);
}

}  // namespace wg
}  // namespace tagg

using namespace tagg;

extern "C" int64_t tagg_token_blocks_bound(int64_t m_alloc, int G) {
  if (m_alloc < 0 || G < 1) return 0;
  return (m_alloc + 127) / 128 + G;
}

static int quantize_col_blocks_impl(const void* x, int x_dtype, int64_t m_alloc, int cols, int64_t ldx,
                                    const int32_t* group_sizes, int G, void* codes, int64_t ldc, float* scales,
                                    int32_t* err_flag, const int32_t* index, const float* row_weights, void* stream,
                                    int block_cols = 1, int pow2 = 0, uint32_t* sf = nullptr);

extern "C" int tagg_quantize_col_blocks(const void* x, int x_dtype, int64_t m_alloc, int cols, int64_t ldx,
                                        const int32_t* group_sizes, int G, void* codes, int64_t ldc, float* scales,
                                        int32_t* err_flag, void* stream) {
  return quantize_col_blocks_impl(x, x_dtype, m_alloc, cols, ldx, group_sizes, G, codes, ldc, scales, err_flag,
                                  nullptr, nullptr, stream);
}

extern "C" int tagg_quantize_col_blocks_gather(const void* x, int x_dtype, int64_t ldx, const int32_t* index,
                                               const float* row_weights, int64_t rows, int cols,
                                               const int32_t* group_sizes, int G, void* codes, int64_t ldc,
                                               float* scales, int32_t* err_flag, void* stream) {
  if (rows > 0 && !index) return TAGG_ERR_SHAPE;
  if (cols % 8 || (reinterpret_cast<uintptr_t>(x) % 16) || ((ldx * (x_dtype == TAGG_DTYPE_BF16 ? 2 : 4)) % 16) ||
      (reinterpret_cast<uintptr_t>(codes) % 8) || (ldc % 8) || (reinterpret_cast<uintptr_t>(scales) % 16))
    return TAGG_ERR_ALIGNMENT;  // the gather form is the vector kernel only
  return quantize_col_blocks_impl(x, x_dtype, rows, cols, ldx, group_sizes, G, codes, ldc, scales, err_flag, index,
                                  row_weights, stream);
}

extern "C" int tagg_quantize_col_blocks_ex(const void* x, int x_dtype, int64_t ldx, const int32_t* index,
                                           const float* row_weights, int64_t rows, int cols,
                                           const int32_t* group_sizes, int G, void* codes, int64_t ldc, float* scales,
                                           int32_t* err_flag, int block_cols, void* stream) {
  const int pow2 = (block_cols & TAGG_QCB_SCALE_POW2) ? 1 : 0;
  block_cols &= ~TAGG_QCB_SCALE_POW2;
  if (block_cols != 1 && block_cols != 128) return TAGG_ERR_CONFIG;
  if (block_cols == 128 && (cols % 128 || (reinterpret_cast<uintptr_t>(x) % 16) ||
                            ((ldx * (x_dtype == TAGG_DTYPE_BF16 ? 2 : 4)) % 16) ||
                            (reinterpret_cast<uintptr_t>(codes) % 8) || (ldc % 8) ||
                            (reinterpret_cast<uintptr_t>(scales) % 16)))
    return TAGG_ERR_ALIGNMENT;  // the 128-column block form is the vector kernel only
  if (rows > 0 && index == nullptr && row_weights != nullptr) return TAGG_ERR_SHAPE;
  return quantize_col_blocks_impl(x, x_dtype, rows, cols, ldx, group_sizes, G, codes, ldc, scales, err_flag, index,
                                  row_weights, stream, block_cols, pow2);
}

extern "C" int tagg_quantize_col_blocks_mx(const void* x, int x_dtype, int64_t ldx, const int32_t* index,
                                           const float* row_weights, int64_t rows, int cols,
                                           const int32_t* group_sizes, int G, void* codes, int64_t ldc, float* scales,
                                           void* sf, int32_t* err_flag, void* stream) {
  if (!sf) return TAGG_ERR_SHAPE;
  if (cols % 128 || (reinterpret_cast<uintptr_t>(sf) % 16)) return TAGG_ERR_ALIGNMENT;
  if (rows > 0 && index == nullptr && row_weights != nullptr) return TAGG_ERR_SHAPE;
  return quantize_col_blocks_impl(x, x_dtype, rows, cols, ldx, group_sizes, G, codes, ldc, scales, err_flag, index,
                                  row_weights, stream, 1, 1, static_cast<uint32_t*>(sf));
}

static int quantize_col_blocks_impl(const void* x, int x_dtype, int64_t m_alloc, int cols, int64_t ldx,
                                    const int32_t* group_sizes, int G, void* codes, int64_t ldc, float* scales,
                                    int32_t* err_flag, const int32_t* index, const float* row_weights, void* stream,
                                    int block_cols, int pow2, uint32_t* sf) {
  if (x_dtype != TAGG_DTYPE_BF16 && x_dtype != TAGG_DTYPE_F32) return TAGG_ERR_CONFIG;
  if (G < 1 || cols < 1 || m_alloc < 0 || ldx < cols || ldc < cols) return TAGG_ERR_SHAPE;
  if (m_alloc == 0) return TAGG_OK;
  if (!x || !group_sizes || !codes || !scales || !err_flag) return TAGG_ERR_SHAPE;
  const int64_t tb = tagg_token_blocks_bound(m_alloc, G);
  if (tb > 65535) return TAGG_ERR_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int esz = x_dtype == TAGG_DTYPE_BF16 ? 2 : 4;
  const bool v8 = cols % 8 == 0 && !(reinterpret_cast<uintptr_t>(x) % 16) && !((ldx * esz) % 16) &&
                  !(reinterpret_cast<uintptr_t>(codes) % 8) && !(ldc % 8) && !(reinterpret_cast<uintptr_t>(scales) % 16);
  if (sf && (!v8 || cols % 128)) return TAGG_ERR_ALIGNMENT;  // the E8M0 blocks come from the vector kernel
  if (v8) {
    const dim3 gt(static_cast<unsigned>(tb));
    auto launch = [&](auto kern) {
      kern<<<gt, 256, 0, st>>>(x, ldx, cols, group_sizes, G, static_cast<uint8_t*>(codes), ldc, scales, err_flag, index,
                               row_weights, pow2, sf);
    };
    const bool bf16 = x_dtype == TAGG_DTYPE_BF16, w = row_weights != nullptr, b128 = block_cols == 128;
    using namespace wg;
    if (pow2 && !b128) {
      if (bf16) w ? launch(quantize_col_tile_kernel<true, false, true, true>) : launch(quantize_col_tile_kernel<true, false, false, true>);
      else w ? launch(quantize_col_tile_kernel<false, false, true, true>) : launch(quantize_col_tile_kernel<false, false, false, true>);
    } else if (bf16) {
      if (b128) w ? launch(quantize_col_tile_kernel<true, true, true>) : launch(quantize_col_tile_kernel<true, true, false>);
      else w ? launch(quantize_col_tile_kernel<true, false, true>) : launch(quantize_col_tile_kernel<true, false, false>);
    } else {
      if (b128) w ? launch(quantize_col_tile_kernel<false, true, true>) : launch(quantize_col_tile_kernel<false, true, false>);
      else w ? launch(quantize_col_tile_kernel<false, false, true>) : launch(quantize_col_tile_kernel<false, false, false>);
    }
    return cudaGetLastError() == cudaSuccess ? TAGG_OK : TAGG_ERR_CUDA;
  }
  const dim3 grid(static_cast<unsigned>((cols + 127) / 128), static_cast<unsigned>(tb));
  if (x_dtype == TAGG_DTYPE_BF16)
    wg::quantize_col_blocks_kernel<true><<<grid, 128, 0, st>>>(x, ldx, cols, group_sizes, G,
                                                               static_cast<uint8_t*>(codes), ldc, scales, err_flag, pow2);
  else
    wg::quantize_col_blocks_kernel<false><<<grid, 128, 0, st>>>(x, ldx, cols, group_sizes, G,
                                                                static_cast<uint8_t*>(codes), ldc, scales, err_flag, pow2);
  return cudaGetLastError() == cudaSuccess ? TAGG_OK : TAGG_ERR_CUDA;
}

extern "C" int tagg_wgrad_fp8(const void* x, const float* sx, const void* dy, const float* sdy, int64_t m_alloc,
                              const int32_t* group_sizes, int G, int K, int N, void* dw, void* stream) {
  return tagg_wgrad_fp8_ex(x, sx, dy, sdy, m_alloc, group_sizes, G, K, N, dw, 0u, stream);
}

static int wgrad_launch(const void* x, const float* sx, const void* dy, const float* sdy, const void* x_sf,
                        const void* dy_sf, int64_t m_alloc, const int32_t* group_sizes, int G, int K, int N, void* dw,
                        uint32_t flags, void* stream);

extern "C" int tagg_wgrad_fp8_ex(const void* x, const float* sx, const void* dy, const float* sdy, int64_t m_alloc,
                                 const int32_t* group_sizes, int G, int K, int N, void* dw, uint32_t flags,
                                 void* stream) {
  if (flags & TAGG_WGRAD_MX) return TAGG_ERR_CONFIG;  // the MXFP8 path takes E8M0 factor blocks: tagg_wgrad_fp8_mx
  if (!sx || !sdy) return TAGG_ERR_SHAPE;
  return wgrad_launch(x, sx, dy, sdy, nullptr, nullptr, m_alloc, group_sizes, G, K, N, dw, flags, stream);
}

extern "C" int tagg_wgrad_fp8_mx(const void* x, const void* x_sf, const void* dy, const void* dy_sf, int64_t m_alloc,
                                 const int32_t* group_sizes, int G, int K, int N, void* dw, void* stream) {
  if (!x_sf || !dy_sf) return TAGG_ERR_SHAPE;
  return wgrad_launch(x, nullptr, dy, nullptr, x_sf, dy_sf, m_alloc, group_sizes, G, K, N, dw, TAGG_WGRAD_MX, stream);
}

static int wgrad_launch(const void* x, const float* sx, const void* dy, const float* sdy, const void* x_sf,
                        const void* dy_sf, int64_t m_alloc, const int32_t* group_sizes, int G, int K, int N, void* dw,
                        uint32_t flags, void* stream) {
  using namespace tagg::wg;
  const bool mx = (flags & TAGG_WGRAD_MX) != 0;
  if (G < 1 || K < 128 || N < 128 || K % 128 || N % 128) return TAGG_ERR_CONFIG;
  if (m_alloc < 0) return TAGG_ERR_SHAPE;
  if (!x || !dy || !group_sizes || !dw) return TAGG_ERR_SHAPE;
  auto mis = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) != 0; };
  if (mis(x) || mis(dy) || mis(dw) || (sx && mis(sx)) || (sdy && mis(sdy)) || (x_sf && mis(x_sf)) ||
      (dy_sf && mis(dy_sf)))
    return TAGG_ERR_ALIGNMENT;
  if (static_cast<int64_t>(G) * K >= (int64_t(1) << 31)) return TAGG_ERR_UNSUPPORTED;
  const int sms = sm_count();
  if (sms <= 0) return TAGG_ERR_CUDA;
  Params p;
  std::memset(&p, 0, sizeof(p));
  const int64_t rows = std::max<int64_t>(m_alloc, 1);
  for (int i = 0; i < kPool; ++i) {
    const uint32_t box[2] = {128, 1u << i};
    const uint64_t dx[2] = {static_cast<uint64_t>(K), static_cast<uint64_t>(rows)};
    const uint64_t sxs[1] = {static_cast<uint64_t>(K)};
    const uint64_t dd[2] = {static_cast<uint64_t>(N), static_cast<uint64_t>(rows)};
    const uint64_t sds[1] = {static_cast<uint64_t>(N)};
    if (!encode_map(&p.map_x[i], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, x, dx, sxs, box, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !encode_map(&p.map_dy[i], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dy, dd, sds, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return TAGG_ERR_CUDA;
  }
  {
    const uint32_t box[2] = {64, 128};
    const uint64_t d[2] = {static_cast<uint64_t>(N), static_cast<uint64_t>(G) * K};
    const uint64_t s[1] = {static_cast<uint64_t>(N) * 2};
    if (!encode_map(&p.map_dw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dw, d, s, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return TAGG_ERR_CUDA;
  }
  if (mx) {
    // factor blocks: [token blocks][columns / 128] blocks of 512 B, viewed as 256-B rows
    const int64_t tbb = tagg_token_blocks_bound(m_alloc, G);
    const uint64_t st[1] = {256};
    const uint64_t dfx[2] = {256, static_cast<uint64_t>(std::max<int64_t>(tbb, 1) * (K / 128) * 2)};
    const uint64_t dfd[2] = {256, static_cast<uint64_t>(std::max<int64_t>(tbb, 1) * (N / 128) * 2)};
    const uint32_t bx[2] = {256, 2}, bd[2] = {256, 4};
    if (!encode_map(&p.map_sfx, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, x_sf, dfx, st, bx, CU_TENSOR_MAP_SWIZZLE_NONE) ||
        !encode_map(&p.map_sfdy, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dy_sf, dfd, st, bd, CU_TENSOR_MAP_SWIZZLE_NONE))
      return TAGG_ERR_CUDA;
  }
  p.sx = sx;
  p.sdy = sdy;
  p.group_sizes = group_sizes;
  p.trace = debug_trace_buffer();
  p.G = G;
  p.K = K;
  p.N = N;
  p.KT = (K + 255) / 256;
  p.NT = (N + 255) / 256;
  p.off_a = 0;
  p.off_b = p.off_a + kStages * kStageA;
  p.off_c = p.off_b + kStages * kStageB;
  p.off_s = p.off_c + (4 / epi_passes(mx)) * kChunkC;
  p.off_sf = p.off_s + kScaleRing * kScaleSlot;
  p.off_tab = p.off_sf + kStages * kSfStage;
  const uint32_t tab = static_cast<uint32_t>(((3 * G * 4) + 15) & ~15);
  p.off_bar = p.off_tab + tab;
  const uint32_t smem = p.off_bar + (2 * kStages + 2 * kNumAcc + 2 * kScaleRing + 4) * 8 + 16 + 1024;
  if (smem > 232448) return TAGG_ERR_UNSUPPORTED;
  const bool dy_block = !mx && (flags & TAGG_WGRAD_DY_BLOCK128) != 0;
  const int variant = mx ? 2 : (dy_block ? 1 : 0);
  auto kern = mx ? wgrad_kernel<false, true> : (dy_block ? wgrad_kernel<true, false> : wgrad_kernel<false, false>);
  static bool configured[3] = {false, false, false};
  if (!configured[variant]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448) != cudaSuccess)
      return TAGG_ERR_CUDA;
    configured[variant] = true;
  }
  const int64_t tiles = static_cast<int64_t>(G) * p.KT * p.NT;
  const int grid = static_cast<int>(std::min<int64_t>(sms / 2, tiles)) * 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1] = {};
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p);
  if (e != cudaSuccess) {
    std::fprintf(stderr, "tagg_wgrad_fp8: launch failed: %s\n", cudaGetErrorString(e));
    return TAGG_ERR_CUDA;
  }
  return TAGG_OK;
}
