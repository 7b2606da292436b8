// tagg_host.h -- host helpers shared by the kernels' launchers (defined in tagg_gemm.cu).
#pragma once

#include <cuda.h>

#include <cstdint>

namespace tagg {
// cuTensorMapEncodeTiled through the runtime's driver entry point, cached by description.
bool encode_map(CUtensorMap* m, CUtensorMapDataType dt, uint32_t rank, const void* base, const uint64_t* dims,
                const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle sw);
// SM count of the current device (cached); -1 on error.
int sm_count();
// Diagnostics trace buffer set by tagg_debug_trace (nullptr when off).
unsigned long long* debug_trace_buffer();
}  // namespace tagg
