// tagg_plan.cpp -- host-side planners of the padding-free grouped GEMM.
//
// These functions are the C-ABI counterparts of the reference's planning layer
// (paths relative to /root/reference/pkg/src/tma_sim/).  The kernel applies
// the same geometry on the device.  tests/test_capi.py checks these
// functions, and the kernel's tile map, bit for bit against oracle/plan.py
// and the reference pins.
#include <cstdint>

#include "tagg.h"

namespace {
int64_t floor_pow2(int64_t n) {  // descriptors.py:27-28
  int64_t p = 1;
  while ((p << 1) <= n) p <<= 1;
  return p;
}
bool is_pow2(int64_t x) { return x >= 1 && (x & (x - 1)) == 0; }
}  // namespace

// ProblemConfig.__post_init__ (engine.py:77-92)
extern "C" int tagg_validate_config(int64_t n, int64_t k, const int64_t* group_sizes, int G, int64_t block_m,
                                    int64_t block_n, int64_t block_k) {
  if (k < 16 || k % 16 != 0) return TAGG_ERR_CONFIG;
  if (n < 64 || n % 64 != 0) return TAGG_ERR_CONFIG;
  if (!is_pow2(block_m)) return TAGG_ERR_INVALID_BLOCK_M;
  if (block_n < 64 || block_n % 64 != 0) return TAGG_ERR_INVALID_BLOCK_N;
  if (block_k != 128) return TAGG_ERR_CONFIG;
  if (G < 1) return TAGG_ERR_CONFIG;
  for (int g = 0; g < G; ++g)
    if (group_sizes[g] < 0) return TAGG_ERR_CONFIG;
  return TAGG_OK;
}

// pool_heights (descriptors.py:31-35)
extern "C" int tagg_pool_heights(int64_t block_rows, int64_t* out, int cap) {
  if (!is_pow2(block_rows)) return TAGG_ERR_INVALID_BLOCK_M;
  int n = 0;
  for (int64_t h = 1; h <= block_rows; h <<= 1) {
    if (n < cap && out) out[n] = h;
    ++n;
  }
  return n;
}

// DescriptorPool.select (descriptors.py:48-54)
extern "C" int64_t tagg_pool_select(int64_t residual_rows, int64_t block_rows) {
  if (residual_rows < 1 || residual_rows > block_rows) return TAGG_ERR_RES_OUT_OF_RANGE;
  return floor_pow2(residual_rows);
}

// plan_group_stores + plan_two_phase (descriptors.py:95-129).
// out[g*9 ..]: group, rows, full_tiles, res, desc, a_smem, a_gmem, b_smem, b_gmem
extern "C" int tagg_plan_group_stores(const int64_t* group_sizes, int G, int64_t block_rows, int64_t* out) {
  if (!is_pow2(block_rows)) return TAGG_ERR_INVALID_BLOCK_M;
  for (int g = 0; g < G; ++g) {
    const int64_t rows = group_sizes[g];
    if (rows < 0) return TAGG_ERR_CONFIG;
    int64_t* o = out + static_cast<int64_t>(g) * 9;
    const int64_t res = rows % block_rows;
    o[0] = g;
    o[1] = rows;
    o[2] = rows / block_rows;
    o[3] = res;
    if (res == 0) {
      o[4] = o[5] = o[6] = o[7] = o[8] = -1;
    } else {
      const int64_t d = floor_pow2(res);
      o[4] = d;
      o[5] = 0;
      o[6] = rows - res;
      o[7] = res - d;
      o[8] = rows - d;
    }
  }
  return TAGG_OK;
}

// plan_prefetch (prefetch.py:50-72), GUARD_ROWS = 16 (prefetch.py:19)
extern "C" int tagg_plan_prefetch(int64_t tile_start_addr, int64_t row_bytes, int64_t block_rows, int64_t* out) {
  if (row_bytes <= 0) return TAGG_ERR_CONFIG;
  for (int64_t r = 0; r < 16; ++r) {
    const int64_t start = tile_start_addr - r * row_bytes;
    if (((start % 16) + 16) % 16 == 0) {
      out[0] = start;
      out[1] = r;
      out[2] = block_rows + 16 - r;
      out[3] = block_rows + 16;
      return TAGG_OK;
    }
  }
  return TAGG_ERR_NO_ALIGNED_SOLUTION;
}

// pad_rows (workload.py:59-65)
extern "C" int64_t tagg_pad_rows(const int64_t* group_sizes, int G, int64_t block_rows) {
  int64_t total = 0;
  for (int g = 0; g < G; ++g) total += (group_sizes[g] + block_rows - 1) / block_rows * block_rows - group_sizes[g];
  return total;
}

extern "C" const char* tagg_error_string(int code) {
  switch (code) {
    case TAGG_OK: return "ok";
    case TAGG_ERR_CONFIG: return "ConfigError";
    case TAGG_ERR_INVALID_BLOCK_M: return "InvalidBlockM";
    case TAGG_ERR_INVALID_BLOCK_N: return "InvalidBlockN";
    case TAGG_ERR_SHAPE: return "ShapeMismatch";
    case TAGG_ERR_ALIGNMENT: return "AlignmentError";
    case TAGG_ERR_NO_ALIGNED_SOLUTION: return "NoAlignedSolution";
    case TAGG_ERR_RES_OUT_OF_RANGE: return "ResOutOfRange";
    case TAGG_ERR_UNSUPPORTED: return "Unsupported";
    case TAGG_ERR_CUDA: return "CudaError";
    default: return "unknown";
  }
}

extern "C" int tagg_version(void) { return 100; }
