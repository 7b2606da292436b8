/*
 * tagg_oracle.c -- CPU ORACLE (test infrastructure, never the product path).
 *
 * A plain-C restatement of the reference's grouped FP8 GEMM semantics:
 *   /root/reference/pkg/src/tma_sim/engine.py
 *     run_padded_baseline            :346-402  (semantic anchor)
 *     run_adaptive tile math         :294-315  (identical per-element math)
 *     _sequential_block_inner        :151-158  inner = fl(inner + a*b), ascending k
 *     _accumulate_scaled             :161-164  s = fl(sa*sb); acc = fl(acc + fl(inner*s))
 *     _col_scale_vector              :167-169  column scale block = col // 128
 *     bf16_from_f32                  :46-50    RNE via (u + 0x7FFF + ((u>>16)&1)) >> 16
 *   /root/reference/pkg/src/tma_sim/fp8.py
 *     DECODE_TABLE                   :34-46    e4m3fn, bias 7, 0x7F/0xFF = NaN
 *   and the scalar triple-loop oracle in pkg/tests/test_engine.py:29-46.
 *
 * Per-expert B (absent from the reference, engine.py:137) is the loop of
 * single-group reference calls: the groups are independent, so expert g simply
 * uses its own B_g and S_B_g.  tests/golden/make_golden.py pins that
 * equivalence with the reference itself.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  Build: see oracle/Makefile.
 * It must be compiled with -ffp-contract=off: an FMA contraction would fuse the
 * reference's separately rounded multiply and add.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static float g_decode[256];
static int g_decode_ready = 0;

/* fp8.py:34-46 */
static void build_decode_table(void) {
  for (int c = 0; c < 256; ++c) {
    int sign = c >> 7, e = (c >> 3) & 0xF, m = c & 7;
    double v = (e == 0) ? ldexp(m / 8.0, -6) : ldexp(1.0 + m / 8.0, e - 7);
    if (sign) v = -v;
    if ((c & 0x7F) == 0x7F) v = NAN;
    g_decode[c] = (float)v;
  }
  g_decode_ready = 1;
}

float tagg_oracle_decode(uint8_t code) {
  if (!g_decode_ready) build_decode_table();
  return g_decode[code];
}

/* engine.py:46-50 */
uint16_t tagg_oracle_bf16_from_f32(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}

typedef struct {
  const uint8_t* a;      /* [M_total, K] row-major codes */
  const float* sa;       /* [M_total, kb] */
  const uint8_t* b;      /* expert base, layout per b_kmajor */
  int64_t b_expert_stride;
  int b_kmajor;          /* 0: [K, N] (reference layout), 1: [N, K] */
  const float* sb;       /* expert base */
  int64_t sb_expert_stride, sb_stride_kb, sb_stride_nb;
  const int64_t* group_sizes;
  int G, N, K;
  uint16_t* c;
  const int64_t* c_row_offsets; /* nullable: output row of each group's row 0 */
  int64_t ldc;
  int n0, n1;            /* computed column range [n0, n1) */
  /* work split */
  int64_t row_begin, row_end; /* global A-row range for this worker */
} job_t;

/* Computes rows [row_begin,row_end) of the stacked problem, columns [n0,n1). */
static void* worker(void* arg) {
  const job_t* j = (const job_t*)arg;
  const int K = j->K, N = j->N, kb_count = (K + 127) / 128;
  const int W = j->n1 - j->n0;
  float* bdec = (float*)malloc((size_t)128 * W * sizeof(float)); /* one k-block of B_g */
  float* inner = (float*)malloc((size_t)W * sizeof(float));
  float* acc = (float*)malloc((size_t)W * sizeof(float));
  float* scol = (float*)malloc((size_t)W * sizeof(float));
  int64_t off = 0;
  for (int g = 0; g < j->G; ++g) {
    const int64_t rows = j->group_sizes[g];
    const int64_t r_lo = off > j->row_begin ? off : j->row_begin;
    const int64_t r_hi = (off + rows) < j->row_end ? (off + rows) : j->row_end;
    if (r_lo < r_hi) {
      const uint8_t* bg = j->b + (int64_t)g * j->b_expert_stride;
      const float* sbg = j->sb + (int64_t)g * j->sb_expert_stride;
      const int64_t crow0 = j->c_row_offsets ? j->c_row_offsets[g] : off;
      /* rows in chunks so the decoded B k-block is reused across rows */
      for (int64_t r0 = r_lo; r0 < r_hi; r0 += 64) {
        const int64_t r1 = (r0 + 64 < r_hi) ? r0 + 64 : r_hi;
        float* accs = (float*)calloc((size_t)(r1 - r0) * W, sizeof(float));
        for (int kb = 0; kb < kb_count; ++kb) {
          const int kc = kb * 128, kw = (K - kc) < 128 ? (K - kc) : 128;
          for (int jj = 0; jj < kw; ++jj)
            for (int n = 0; n < W; ++n) {
              const int col = j->n0 + n;
              const uint8_t code = j->b_kmajor ? bg[(int64_t)col * K + kc + jj]
                                               : bg[(int64_t)(kc + jj) * N + col];
              bdec[(size_t)jj * W + n] = g_decode[code];
            }
          for (int n = 0; n < W; ++n)
            scol[n] = sbg[(int64_t)kb * j->sb_stride_kb + (int64_t)((j->n0 + n) / 128) * j->sb_stride_nb];
          for (int64_t r = r0; r < r1; ++r) {
            const uint8_t* arow = j->a + r * K + kc;
            /* _sequential_block_inner: ascending k chain of rounded f32 adds */
            for (int n = 0; n < W; ++n) inner[n] = 0.0f;
            for (int jj = 0; jj < kw; ++jj) {
              const float av = g_decode[arow[jj]];
              const float* brow = bdec + (size_t)jj * W;
              for (int n = 0; n < W; ++n) inner[n] = inner[n] + av * brow[n];
            }
            /* _accumulate_scaled */
            const float sa = j->sa[r * kb_count + kb];
            float* ac = accs + (size_t)(r - r0) * W;
            for (int n = 0; n < W; ++n) {
              const float s = sa * scol[n];
              const float t = inner[n] * s;
              ac[n] = ac[n] + t;
            }
          }
        }
        for (int64_t r = r0; r < r1; ++r) {
          uint16_t* crow = j->c + (crow0 + (r - off)) * j->ldc + j->n0;
          const float* ac = accs + (size_t)(r - r0) * W;
          for (int n = 0; n < W; ++n) crow[n] = tagg_oracle_bf16_from_f32(ac[n]);
        }
        free(accs);
      }
    }
    off += rows;
  }
  free(bdec);
  free(inner);
  free(acc);
  free(scol);
  return NULL;
}

/*
 * Grouped GEMM oracle.  Returns 0 on success, -1 on bad arguments.
 * Computes C rows of every group for columns [n0, n1) (pass 0, N for all).
 * nthreads <= 1 runs on the calling thread.
 */
int tagg_oracle_grouped_gemm(const uint8_t* a, const float* sa, const uint8_t* b,
                             int64_t b_expert_stride, int b_kmajor, const float* sb,
                             int64_t sb_expert_stride, int64_t sb_stride_kb,
                             int64_t sb_stride_nb, const int64_t* group_sizes, int G, int N,
                             int K, uint16_t* c, const int64_t* c_row_offsets, int64_t ldc,
                             int n0, int n1, int nthreads) {
  if (!g_decode_ready) build_decode_table();
  if (G < 1 || N < 1 || K < 1 || n0 < 0 || n1 > N || n0 >= n1) return -1;
  int64_t m_total = 0;
  for (int g = 0; g < G; ++g) {
    if (group_sizes[g] < 0) return -1;
    m_total += group_sizes[g];
  }
  if (m_total == 0) return 0;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if ((int64_t)nthreads > m_total) nthreads = (int)m_total;
  job_t base = {a, sa, b, b_expert_stride, b_kmajor, sb, sb_expert_stride, sb_stride_kb,
                sb_stride_nb, group_sizes, G, N, K, c, c_row_offsets, ldc, n0, n1, 0, 0};
  job_t jobs[256];
  pthread_t tids[256];
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = base;
    jobs[t].row_begin = m_total * t / nthreads;
    jobs[t].row_end = m_total * (t + 1) / nthreads;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&tids[t], NULL, worker, &jobs[t]);
  worker(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(tids[t], NULL);
  return 0;
}

/* Bytes/rows the padded baseline adds: workload.py:59-65. */
int64_t tagg_oracle_pad_rows(const int64_t* group_sizes, int G, int block_rows) {
  int64_t total = 0;
  for (int g = 0; g < G; ++g)
    total += ((group_sizes[g] + block_rows - 1) / block_rows) * block_rows - group_sizes[g];
  return total;
}

/*
 * Weight-gradient oracle (the reference has no backward,
 * SPEC.md:361, so this is the forward's arithmetic applied along the ragged axis):
 *   dW[g][k][n] = bf16( acc ),  acc over the group's 128-token blocks j ascending:
 *     inner_j = ascending-token chain of rounded f32 adds of exact products
 *               x[t][k] * dy[t][n], t in block j  (_sequential_block_inner, engine.py:151-158)
 *     s       = fl(sx[tb][k] * sdy[tb][n])              (_accumulate_scaled, engine.py:161-164)
 *     acc     = fl(acc + fl(inner_j * s))
 * x [M_total, K], dy [M_total, N] row-major codes; sx [TB, K], sdy [TB, N] with one row per
 * (group, 128-token block), blocks numbered group by group (tb0(g) = sum of
 * ceil(M_h/128) over h < g).  An empty group gives dW[g] = 0.  out: [G, K, N] bf16 bits.
 */
typedef struct {
  const uint8_t *x, *dy;
  const float *sx, *sdy;
  const int64_t* group_sizes;
  int G, K, N;
  uint16_t* out;
  int64_t job_begin, job_end; /* (g, k) pairs */
} wjob_t;

static void* wgrad_worker(void* arg) {
  const wjob_t* j = (const wjob_t*)arg;
  const int K = j->K, N = j->N;
  float* inner = (float*)malloc((size_t)N * sizeof(float));
  float* acc = (float*)malloc((size_t)N * sizeof(float));
  for (int64_t p = j->job_begin; p < j->job_end; ++p) {
    const int g = (int)(p / K), k = (int)(p % K);
    int64_t off = 0, tb0 = 0;
    for (int h = 0; h < g; ++h) {
      off += j->group_sizes[h];
      tb0 += (j->group_sizes[h] + 127) / 128;
    }
    const int64_t rows = j->group_sizes[g];
    for (int n = 0; n < N; ++n) acc[n] = 0.0f;
    for (int64_t b0 = 0; b0 < rows; b0 += 128) {
      const int64_t b1 = (b0 + 128 < rows) ? b0 + 128 : rows;
      for (int n = 0; n < N; ++n) inner[n] = 0.0f;
      for (int64_t t = off + b0; t < off + b1; ++t) {
        const float xv = g_decode[j->x[t * K + k]];
        const uint8_t* dyr = j->dy + t * N;
        for (int n = 0; n < N; ++n) inner[n] = inner[n] + xv * g_decode[dyr[n]];
      }
      const int64_t tb = tb0 + b0 / 128;
      const float sxk = j->sx[tb * K + k];
      const float* sdyr = j->sdy + tb * N;
      for (int n = 0; n < N; ++n) {
        const float s = sxk * sdyr[n];
        const float t = inner[n] * s;
        acc[n] = acc[n] + t;
      }
    }
    uint16_t* o = j->out + ((int64_t)g * K + k) * N;
    for (int n = 0; n < N; ++n) o[n] = tagg_oracle_bf16_from_f32(acc[n]);
  }
  free(inner);
  free(acc);
  return NULL;
}

int tagg_oracle_wgrad(const uint8_t* x, const float* sx, const uint8_t* dy, const float* sdy,
                      const int64_t* group_sizes, int G, int K, int N, uint16_t* out, int nthreads) {
  if (!g_decode_ready) build_decode_table();
  if (G < 1 || K < 1 || N < 1) return -1;
  for (int g = 0; g < G; ++g)
    if (group_sizes[g] < 0) return -1;
  const int64_t jobs_total = (int64_t)G * K;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if ((int64_t)nthreads > jobs_total) nthreads = (int)jobs_total;
  wjob_t jobs[256];
  pthread_t tids[256];
  for (int t = 0; t < nthreads; ++t) {
    wjob_t w = {x, dy, sx, sdy, group_sizes, G, K, N, out, jobs_total * t / nthreads,
                jobs_total * (t + 1) / nthreads};
    jobs[t] = w;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&tids[t], NULL, wgrad_worker, &jobs[t]);
  wgrad_worker(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(tids[t], NULL);
  return 0;
}
