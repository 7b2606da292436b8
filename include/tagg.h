/*
 * tagg.h -- C ABI of the B200-native padding-free FP8 grouped GEMM
 * ("TMA-adaptive grouped GEMM", arxiv 2508.16584), libtagg.so.
 *
 * Plain pointers and sizes only: no torch types cross this boundary.  Every
 * device pointer argument is a CUDA device address; `stream` is a
 * cudaStream_t (NULL = legacy default stream).  All launches are
 * stream-ordered and never synchronise the host.  Functions are reentrant.
 *
 * Reference interfaces replaced (paths relative to
 * /root/reference/pkg/src/tma_sim/):
 *   tagg_grouped_gemm_fp8 -> engine.run_adaptive            engine.py:184-343
 *   tagg_padded_baseline  -> engine.run_padded_baseline     engine.py:346-402
 *     (implemented as tagg_pad_groups + tagg_grouped_gemm_fp8 + tagg_unpad_rows)
 *   tagg_plan_group_stores-> descriptors.plan_group_stores  descriptors.py:117-129
 *                            (+ plan_two_phase              descriptors.py:95-106)
 *   tagg_pool_heights     -> descriptors.pool_heights       descriptors.py:31-35
 *   tagg_pool_select      -> DescriptorPool.select          descriptors.py:48-54
 *   tagg_plan_prefetch    -> prefetch.plan_prefetch         prefetch.py:50-72
 *   tagg_validate_config  -> ProblemConfig.__post_init__    engine.py:77-92
 *   tagg_pad_rows         -> workload.pad_rows              workload.py:59-65
 * Error codes mirror the reference's exception hierarchy (errors.py:6-76).
 */
#ifndef TAGG_H
#define TAGG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py) ---- */
#define TAGG_OK 0
#define TAGG_ERR_CONFIG (-1)            /* ConfigError          errors.py:14 */
#define TAGG_ERR_INVALID_BLOCK_M (-2)   /* InvalidBlockM        errors.py:18 */
#define TAGG_ERR_INVALID_BLOCK_N (-3)   /* InvalidBlockN        errors.py:22 */
#define TAGG_ERR_SHAPE (-4)             /* ShapeMismatch        errors.py:71 */
#define TAGG_ERR_ALIGNMENT (-5)         /* AlignmentError       errors.py:30-40 */
#define TAGG_ERR_NO_ALIGNED_SOLUTION (-6) /* NoAlignedSolution  errors.py:64-68 */
#define TAGG_ERR_RES_OUT_OF_RANGE (-7)  /* ResOutOfRange        errors.py:60 */
#define TAGG_ERR_UNSUPPORTED (-8)       /* shape exceeds this build's on-chip budget: K <= 16384
                                           (128 k-blocks of S_B staging; the S_A window drops to one
                                           slot when two do not fit beside two pipeline stages),
                                           G up to ~8k (device group tables in smem), M < 2^31 */
#define TAGG_ERR_CUDA (-9)              /* CUDA runtime / driver failure */

/* ---- B operand storage ---- */
#define TAGG_B_KN 0 /* [G_b, K, N], N contiguous (reference layout, engine.py:137) */
#define TAGG_B_NK 1 /* [G_b, N, K], K contiguous (transposed weights, dgrad)      */

/* ---- flags ---- */
#define TAGG_FLAG_EXACT_PROMOTION 1u /* s=fl(sa*sb); acc=fl(acc+fl(inner*s)) with two roundings
                                        (engine.py:161-164) instead of one FFMA2 */
#define TAGG_FLAG_PLAIN_C_STAGING 2u /* unswizzled C staging + SWIZZLE_NONE store pool */
#define TAGG_FLAG_SINGLE_CTA 4u      /* 128x128 tiles on one CTA (tcgen05 cta_group::1) instead of the
                                        default CTA-pair tile (cta_group::2) */
#define TAGG_FLAG_TILE_N128 8u       /* CTA-pair tile 256x128 (more, smaller tiles: fewer idle SMs
                                        in the last wave of small problems) */
#define TAGG_FLAG_TILE_N256 16u      /* CTA-pair tile 256x256.  With none of SINGLE_CTA / TILE_N128 /
                                        TILE_N256 set, the launch picks 256x256 pair tiles, or 1-CTA
                                        128x128 tiles when m_alloc <= 128 G (HBM-bound skinny
                                        groups) */
#define TAGG_FLAG_SERIAL 32u         /* no programmatic dependent launch.  By default a grouped GEMM
                                        is launched with PDL: when the previous kernel in the stream
                                        is a grouped GEMM, this one's CTAs start on the SMs that grid
                                        releases, initialise their barriers and TMEM, and then wait
                                        (griddepcontrol.wait) for its completion and memory before
                                        they read any input.  Stream order is fully kept. */
#define TAGG_FLAG_PDL_OVERLAP 64u    /* the caller asserts that the kernel launched right before this
                                        one in the stream writes none of this launch's inputs (A, S_A,
                                        B, S_B, group sizes, c_row_offsets), e.g. a chain of independent
                                        grouped GEMMs over resident operands.  Then the main loop runs
                                        during the previous grid's tail and only the global stores
                                        (C, tile map, error flag) wait for its completion, which keeps
                                        write-after-write order on a shared C.  Ignored with SERIAL. */
/* Cap the persistent grid at n SMs (flags bits 16-27; 0 = every SM).  An overlapped
   expert-parallel exchange leaves the rest to the NCCL kernels that run beside the GEMM. */
#define TAGG_SM_LIMIT_SHIFT 16
#define TAGG_SM_LIMIT_MASK 0xFFFu
#define TAGG_SM_LIMIT(n) (((uint32_t)(n) & TAGG_SM_LIMIT_MASK) << TAGG_SM_LIMIT_SHIFT)

#define TAGG_TILE_MAP_FIELDS 9

/*
 * Padding-free grouped GEMM: for every group g with M_g rows (rows stacked
 * along M in A, group g starting at sum(M_0..M_{g-1})):
 *   C[c_row0(g) + i, n] = bf16( sum_kb  inner_kb(i, n) * fl(SA[row, kb] * SB_g[kb, n/128]) )
 * with inner_kb the exact-product FP8 dot product over the 128-wide k block
 * (tensor cores) and the k-block sum accumulated in fp32 registers in
 * ascending kb (engine.py:294-314).
 *
 *  a              [m_alloc, K] e4m3fn codes, row stride lda bytes (lda % 16 == 0)
 *  sa             [m_alloc, ceil(K/128)] fp32, K-major, dense (row stride 4*ceil(K/128) B)
 *  b              b_layout TAGG_B_KN: [b_experts, K, N]; TAGG_B_NK: [b_experts, N, K];
 *                 b_experts == 1 shares one B across all groups (reference API)
 *  sb             fp32 scales; element (g, kb, nb) at sb[g*sb_stride_g + kb*sb_stride_kb +
 *                 nb*sb_stride_nb] (strides in floats; sb_stride_g = 0 for a shared B)
 *  group_sizes    DEVICE int32 [G], M_g >= 0, sum <= m_alloc (not read by the host)
 *  c              [c_rows, N] bf16 bits, row stride ldc elements (ldc % 8 == 0)
 *  c_row_offsets  nullable DEVICE int64 [G]: output row of group g's first row;
 *                 NULL = contiguous (same rows as A)
 *  tile_map       nullable DEVICE int32 [tagg_max_tiles(), 9]: per tile
 *                 (g, m_tile, n0, a_row0, valid, d, phaseA_row, phaseB_smem_row, phaseB_row),
 *                 the exact store geometry the kernel used; unused rows untouched
 *  flags          TAGG_FLAG_*
 *
 * Only C rows [c_row0(g), c_row0(g) + M_g) of each group are written.  No row
 * beyond M_g is ever stored: residual tiles use the power-of-two TMA
 * descriptor pool with the dual-phase store (descriptors.py:95-106).
 */
int tagg_grouped_gemm_fp8(const void* a, int64_t lda, const float* sa, int64_t m_alloc,
                          const void* b, int b_layout, int b_experts, const float* sb,
                          int64_t sb_stride_g, int64_t sb_stride_kb, int64_t sb_stride_nb,
                          const int32_t* group_sizes, int G, int N, int K, void* c, int64_t ldc,
                          int64_t c_rows, const int64_t* c_row_offsets, int32_t* tile_map,
                          uint32_t flags, void* stream);

/*
 * The general entry point; tagg_grouped_gemm_fp8 is this with b_index = err_flag = NULL.
 *  b_index   nullable DEVICE int32 [G]: group g multiplies B expert b_index[g] (0 <= . < b_experts),
 *            so several groups may share one expert's weights -- e.g. the (source rank, expert)
 *            segments an expert-parallel all-to-all delivers, read in place without a regroup.
 *            NULL = group g uses expert g (b_experts == G) or the shared B (b_experts == 1).
 *  err_flag  nullable DEVICE int32, OR-ed, never cleared.  The group sizes live on the device, so
 *            the kernel validates them: bit 0 a negative M_g (ConfigError, engine.py:82-92); bit 1
 *            sum(M_g) > m_alloc, or more rows than C holds (c_rows without c_row_offsets; with
 *            them, a non-empty group's rows outside [0, c_rows)) (ShapeMismatch,
 *            engine.py:132-142); bit 2 a non-empty group's b_index outside [0, b_experts).  A
 *            launch that flags does no loads, stores or tile-map writes at all.
 */
int tagg_grouped_gemm_fp8_ex(const void* a, int64_t lda, const float* sa, int64_t m_alloc, const void* b,
                             int b_layout, int b_experts, const float* sb, int64_t sb_stride_g,
                             int64_t sb_stride_kb, int64_t sb_stride_nb, const int32_t* group_sizes, int G, int N,
                             int K, void* c, int64_t ldc, int64_t c_rows, const int64_t* c_row_offsets,
                             int32_t* tile_map, const int32_t* b_index, int32_t* err_flag, uint32_t flags,
                             void* stream);

/* Upper bound on the tile count, to size tile_map (no device data needed). */
int64_t tagg_max_tiles(int64_t m_alloc, int G, int N);

/* CTA clusters (pairs, or single CTAs with TAGG_FLAG_SINGLE_CTA) a launch with these
   sizes uses on the current device.  The 256x256 pair tile balances its last wave
   with it: when T mod clusters <= clusters / 2 for T scheduled tiles, those last tiles
   each run as two 128-row half tiles (oracle/plan.py: kernel_tile_map). */
int tagg_launch_clusters(int64_t m_alloc, int G, int N, uint32_t flags);

/*
 * Baseline K2 (engine.py:369-373): copy each group into a 128-row-aligned
 * slot, A pad rows = 0, S_A pad rows = 1.0.  a_pad / sa_pad need
 * tagg_padded_rows_bound(m_alloc, G) rows.  padded_sizes (DEVICE int32 [G])
 * receives ceil(M_g/128)*128.
 */
int tagg_pad_groups(const void* a, int64_t lda, const float* sa, const int32_t* group_sizes, int G,
                    int K, void* a_pad, float* sa_pad, int32_t* padded_sizes, int64_t m_pad_alloc,
                    void* stream);
/* Baseline K3 (engine.py:399-401): gather each group's valid rows from C_pad. */
int tagg_unpad_rows(const void* c_pad, const int32_t* group_sizes, int G, int N, void* c,
                    int64_t m_alloc, void* stream);
int64_t tagg_padded_rows_bound(int64_t m_alloc, int G);

/* ---- producer side: fused 1x128 quantize + dispatch permutation ---- */
#define TAGG_DTYPE_BF16 0
#define TAGG_DTYPE_F32 1

/*
 * Route plan: a stable counting sort of `rows` routed rows by expert.
 *   expert_ids   DEVICE int32 [rows], 0 <= id < num_experts (<= 1024)
 *   group_sizes  DEVICE int32 [num_experts]  <- rows per expert (the GEMM's M_g)
 *   dest_rows    DEVICE int32 [rows]         <- row of the padding-free grouped layout:
 *                experts in order, rows of one expert in ascending source order
 *   workspace    DEVICE int32 [tagg_route_workspace_ints(rows, num_experts)]
 * Out-of-range ids (e.g. -1 for a token the router dropped) get dest_rows = -1, are
 * counted in no group and are flagged (tagg_route_error); the quantize / dispatch,
 * combine and router-gradient kernels skip such routes.  Stream-ordered, no host sync.
 */
int64_t tagg_route_workspace_ints(int64_t rows, int num_experts);
int tagg_route_plan(const int32_t* expert_ids, int64_t rows, int num_experts, int32_t* group_sizes,
                    int32_t* dest_rows, int32_t* workspace, void* stream);
/* Synchronous read of the route plan's error flag (1 = an expert id out of range). */
int tagg_route_error(const int32_t* workspace, int64_t rows, int num_experts, int32_t* host_flag);

/*
 * Fused 1x128 quantization (fp8.py:132-151; encode fp8.py:54-80) and dispatch:
 * token t's row of x [tokens, K] (bf16 or f32, row stride ldx elements) is quantized
 * once per 128-column tile, s = fl(amax / 448) (1.0 for an all-zero tile),
 * code = e4m3(fl(x / s)) RNE saturating, and written to rows dest_rows[t*topk + k],
 * k < topk (<= 8), of a [*, lda] (codes) and sa [*, ceil(K/128)] (scales).
 * dest_rows may be NULL with topk == 1 (plain quantize_row_tiles).  Non-finite
 * inputs set bit 2 of *err_flag (DEVICE int32; the reference raises InvalidInput).
 */
int tagg_quantize_dispatch(const void* x, int x_dtype, int64_t ldx, int64_t tokens, int K, int topk,
                           const int32_t* dest_rows, void* a, int64_t lda, float* sa, int32_t* err_flag,
                           void* stream);
/*
 * The same 1x128 quantization over gathered, weighted rows, without materialising them: row r of
 * a / sa quantizes bf16(row_weights[r] * x[index[r]]) (fl(w*x) rounded to bf16 RNE, i.e. exactly
 * the rows tagg_gather_scale_rows writes; row_weights may be NULL for a plain gather).  The MoE
 * backward's dL/dc rows go straight from the token-ordered dy to the dgrad GEMM's A / S_A.
 */
int tagg_quantize_gather_rows(const void* x, int x_dtype, int64_t ldx, const int32_t* index, const float* row_weights,
                              int64_t rows, int K, void* a, int64_t lda, float* sa, int32_t* err_flag, void* stream);

/*
 * 128x128 block quantization (fp8.py:154-176), batched: matrix b of x (rows x cols,
 * row stride ldx, matrix stride x_batch_stride elements) -> codes (row stride ldc,
 * matrix stride codes_batch_stride bytes) and scales [batch][ceil(rows/128)][ceil(cols/128)].
 * One scale per block, s = fl(amax / 448) (1.0 for an all-zero block), codes as in
 * tagg_quantize_dispatch.  Per-expert weights [G, K, N] are batch = G, rows = K, cols = N.
 */
int tagg_quantize_blocks(const void* x, int x_dtype, int64_t batch, int64_t rows, int64_t cols, int64_t ldx,
                         int64_t x_batch_stride, void* codes, int64_t ldc, int64_t codes_batch_stride,
                         float* scales, int32_t* err_flag, void* stream);

/* ---- backward: weight gradient as a K-grouped GEMM ---- */
/*
 * Per-group 128x1 quantization for the weight gradient: for every group's 128-token
 * block and column c, s = fl(amax / 448) (1.0 when zero) over the block's rows (fewer
 * than 128 in a group's last block) and codes = e4m3(fl(x / s)).  codes [m_alloc, cols]
 * (row stride ldc), scales [tagg_token_blocks_bound(m_alloc, G), cols] of which the
 * first sum(ceil(M_g/128)) rows are written, group by group.  group_sizes on the device.
 */
int64_t tagg_token_blocks_bound(int64_t m_alloc, int G);
int tagg_quantize_col_blocks(const void* x, int x_dtype, int64_t m_alloc, int cols, int64_t ldx,
                             const int32_t* group_sizes, int G, void* codes, int64_t ldc, float* scales,
                             int32_t* err_flag, void* stream);
/* The same with a row gather: grouped row r is row_weights[r] * x[index[r], :] (row_weights
   nullable = 1), for rows grouped rows; x is token-ordered (e.g. activations or dL/dy), so no
   grouped copy is materialized.  Needs cols % 8 == 0 and 16-byte aligned x rows. */
int tagg_quantize_col_blocks_gather(const void* x, int x_dtype, int64_t ldx, const int32_t* index,
                                    const float* row_weights, int64_t rows, int cols, const int32_t* group_sizes,
                                    int G, void* codes, int64_t ldc, float* scales, int32_t* err_flag, void* stream);
/*
 * dW_g = X_g^T dY_g for every group (K % 128 == 0, N % 128 == 0): x [m_alloc, K] and
 * dy [m_alloc, N] e4m3 codes in the padding-free grouped layout (dense rows), sx [TB, K]
 * and sdy [TB, N] from tagg_quantize_col_blocks, dw bf16 [G, K, N].  The ragged M_g is the
 * reduction axis: a group's last token block is loaded with the power-of-two TMA
 * descriptor pool in two phases and the rows past the group end are zeroed in smem, so
 * no other group's token enters the sum.  An empty group gets dW = 0.
 */
int tagg_wgrad_fp8(const void* x, const float* sx, const void* dy, const float* sdy, int64_t m_alloc,
                   const int32_t* group_sizes, int G, int K, int N, void* dw, void* stream);
/* The same with flags.  TAGG_WGRAD_DY_BLOCK128: the caller asserts sdy is constant over every
   128-column block of each token block (dY quantized with tagg_quantize_col_blocks_ex, block_cols
   = 128, the reference's 128x128 block recipe fp8.py:154-176 per group token block).  The
   promotion then uses one scale per drained 128-column half: one FFMA2 per element pair instead of
   an FMUL2 and an FFMA2. */
#define TAGG_WGRAD_DY_BLOCK128 1u
#define TAGG_WGRAD_MX 2u /* internal: the tagg_wgrad_fp8_mx path (rejected by tagg_wgrad_fp8_ex) */
int tagg_wgrad_fp8_ex(const void* x, const float* sx, const void* dy, const float* sdy, int64_t m_alloc,
                      const int32_t* group_sizes, int G, int K, int N, void* dw, uint32_t flags, void* stream);
/* ---- MXFP8 weight gradient: power-of-two scales applied by the tensor core ----
 * tagg_quantize_col_blocks_mx: the column-block quantizer (row gather as in _gather / _ex, index
 * and row_weights nullable) with every scale rounded up to a power of two,
 * s = 2^ceil(log2(fl(amax / 448))) (1.0 when zero), so x / s is exact; besides the fp32 scales it
 * writes sf: per (token block, 128 columns) a 512-B block of E8M0 bytes in the tcgen05.cp source
 * layout (byte 16 l + 4 c + j = the exponent byte of column 32 c + l's scale, j = 0..3),
 * [tagg_token_blocks_bound(rows, G), cols / 128, 512] bytes.  cols % 128 == 0.
 * tagg_wgrad_fp8_mx: dW_g = X_g^T dY_g from such operands (x_sf / dy_sf the sf blocks): the tensor
 * core applies the factors as block scales (tcgen05.mma kind::mxf8f6f4.block_scale) and accumulates
 * each tile's whole token range in TMEM, with no per-block promotion -- the same real sum as
 * tagg_wgrad_fp8 over the same operands, rounded in fp32 by the tensor core instead of per block. */
int tagg_quantize_col_blocks_mx(const void* x, int x_dtype, int64_t ldx, const int32_t* index, const float* row_weights,
                                int64_t rows, int cols, const int32_t* group_sizes, int G, void* codes, int64_t ldc,
                                float* scales, void* sf, int32_t* err_flag, void* stream);
int tagg_wgrad_fp8_mx(const void* x, const void* x_sf, const void* dy, const void* dy_sf, int64_t m_alloc,
                      const int32_t* group_sizes, int G, int K, int N, void* dw, void* stream);
/* Column-block quantization with a row gather (index / row_weights nullable, as above) and a block
   width: block_cols = 1 is tagg_quantize_col_blocks(_gather); block_cols = 128 takes one amax per
   (token block, 128 columns) and writes it to all 128 columns' scale slots (cols % 128 == 0). */
/* OR'ed into block_cols: every scale is rounded up to a power of two, s = 2^ceil(log2(fl(amax / 448)))
   (1.0 when zero), so x / s is exact and s is one E8M0 byte -- the MXFP8 recipe that
   TAGG_WGRAD_MX consumes. */
#define TAGG_QCB_SCALE_POW2 0x10000
int tagg_quantize_col_blocks_ex(const void* x, int x_dtype, int64_t ldx, const int32_t* index,
                                const float* row_weights, int64_t rows, int cols, const int32_t* group_sizes, int G,
                                void* codes, int64_t ldc, float* scales, int32_t* err_flag, int block_cols,
                                void* stream);

/* ---- host planners (no GPU needed) ---- */
/* ProblemConfig validation (engine.py:77-92). */
int tagg_validate_config(int64_t n, int64_t k, const int64_t* group_sizes, int G, int64_t block_m,
                         int64_t block_n, int64_t block_k);
/* Per group 8 int64: group, rows, full_tiles, res, desc, a_smem, a_gmem, b_smem, b_gmem
   (res = 0 and the phase fields = -1 when the group divides evenly).  out: [G, 9]. */
int tagg_plan_group_stores(const int64_t* group_sizes, int G, int64_t block_rows, int64_t* out);
/* Pool heights 1..block_rows (powers of two); returns the count or an error. */
int tagg_pool_heights(int64_t block_rows, int64_t* out, int cap);
/* Largest pool height <= residual_rows; TAGG_ERR_RES_OUT_OF_RANGE outside [1, block_rows]. */
int64_t tagg_pool_select(int64_t residual_rows, int64_t block_rows);
/* out[4] = start_addr, row_prev, row_next, total_rows. */
int tagg_plan_prefetch(int64_t tile_start_addr, int64_t row_bytes, int64_t block_rows, int64_t* out);
int64_t tagg_pad_rows(const int64_t* group_sizes, int G, int64_t block_rows);

const char* tagg_error_string(int code);
/* Diagnostics only: subsequent tagg_grouped_gemm_fp8 launches stamp clock64()
   at 10 pipeline events for the first 1024 k-block iterations of CTAs 0 and 1
   into buf (DEVICE u64 [2][10][1024]); NULL (the default) disables it. */
void tagg_debug_trace(void* buf);
int tagg_version(void);

/* ---- MoE FFN steps around the GEMM (csrc/tagg_moe.cu) ---- */
/*
 * SwiGLU + 1x128 quantize of the gate|up GEMM output, in place in the padding-free layout:
 *   h            bf16 [m_alloc, >= 2I], row pitch ldh elements: gate = columns [0, I),
 *                up = columns [I, 2I)
 *   group_sizes  DEVICE int32 [G]: only rows [0, sum M_g) are read and written
 *   a / sa       the down GEMM's A: e4m3 codes [m_alloc, I] (pitch lda bytes) and fp32 scales
 *                [m_alloc, ceil(I/128)], from v = fl(silu(gate) * up) with the fp8.py:132-151 recipe
 *   err_flag     DEVICE int32, |= 2 on a non-finite v
 * ldh*2, I*2, lda and both bases must be multiples of 16 bytes.
 */
int tagg_swiglu_quantize(const void* h, int64_t ldh, const int32_t* group_sizes, int G, int64_t m_alloc, int I,
                         void* a, int64_t lda, float* sa, int32_t* err_flag, void* v_out, int64_t ldv,
                         void* stream);
/* (v_out: nullable bf16 [m_alloc, I] copy of v, pitch ldv, kept by a training forward for wgrad.) */

/* out[r, :] = bf16(row_weights[r] * src[index[r], :]) for r < rows (row_weights nullable = 1):
   token rows gathered into the grouped layout, e.g. the backward's dL/dc = w[t,k] * dy[t].
   bf16, H % 8 == 0, 16-byte aligned bases and pitches. */
int tagg_gather_scale_rows(const void* src, int64_t lds, const int32_t* index, const float* row_weights, int64_t rows,
                           int H, void* out, int64_t ldo, void* stream);
/* Router-weight gradient: out[t*topk + k] = <dy[t, :], c[dest_rows[t*topk + k], :]> in fp32. */
int tagg_router_grad(const void* dy, int64_t lddy, const void* c, int64_t ldc, const int32_t* dest_rows,
                     int64_t tokens, int topk, int H, float* out, void* stream);
/*
 * Backward of tagg_swiglu_quantize: from the saved gate|up rows h = [g | u] (bf16 [m_alloc, 2I])
 * and dh = dL/dv (bf16 [m_alloc, I], v = silu(g) * u):
 *   dg = dh * u * sig(g) * (1 + g * (1 - sig(g))),  du = dh * silu(g)
 * written as bf16 d[g | u] to dgu (nullable, [m_alloc, 2I]) and row-quantized 1x128 FP8 to a / sa
 * ([m_alloc, 2I] codes, [m_alloc, 2I/128] scales; dg and du tiles separately): the A operand of the
 * gate|up dgrad GEMM.  Rows [0, sum M_g) only; I % 128 == 0; 16-byte aligned bases and pitches.
 */
int tagg_swiglu_backward_quantize(const void* h, int64_t ldh, const void* dh, int64_t lddh,
                                  const int32_t* group_sizes, int G, int64_t m_alloc, int I, void* dgu,
                                  int64_t lddgu, void* a, int64_t lda, float* sa, int32_t* err_flag, void* stream);
/*
 * Top-k combine of the down GEMM output: out[t, :] = bf16( sum_{k < topk} fl(w[t,k] * c[dest[t*topk+k], :]) ),
 * accumulated in fp32 in k order with separate roundings (no FMA); routes with dest < 0 (dropped)
 * contribute nothing.  dest = the dispatch plan's dest_rows (tagg_route_plan); c bf16 [rows, N] (pitch ldc), out bf16 [tokens, N] (pitch ldo),
 * N % 8 == 0, topk <= 8, 16-byte aligned bases and pitches.
 */
int tagg_combine(const void* c, int64_t ldc, const int32_t* dest_rows, const float* weights, int64_t tokens, int topk,
                 int N, void* out, int64_t ldo, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TAGG_H */
