"""B200-native padding-free FP8 grouped GEMM (arxiv 2508.16584).

The hot path is one hand-written sm_100a kernel (csrc/tagg_gemm.cu) behind the
C ABI in include/tagg.h.  This package is the host-side mirror of the
reference's Python entry points (tma_sim.engine / descriptors / prefetch /
workload), with the same names, argument meanings and exceptions.
"""

from .engine import (  # noqa: F401
    AdaptiveRun,
    BitwiseReport,
    GroupedOperands,
    PaddedWorkspace,
    ProblemConfig,
    bf16_from_f32,
    f32_from_bf16,
    grouped_gemm_fp8,
    max_tiles,
    pad_groups,
    padded_grouped_gemm_fp8,
    run_adaptive,
    run_padded_baseline,
    unpad_rows,
    verify_bitwise,
)
from .errors import (  # noqa: F401
    AlignmentError,
    ConfigError,
    CudaError,
    InvalidBlockM,
    InvalidBlockN,
    InvalidInput,
    NoAlignedSolution,
    ResOutOfRange,
    ShapeMismatch,
    SimError,
    Unsupported,
)
from .quant import (  # noqa: F401
    DispatchedActivations,
    gather_rows,
    quantize_blocks,
    quantize_dispatch,
    quantize_gather_rows,
    quantize_row_tiles,
    route_plan,
)
from .wgrad import quantize_col_blocks, quantize_col_blocks_mx, wgrad_fp8, wgrad_fp8_mx  # noqa: F401
from . import tensorio  # noqa: F401
from . import moe  # noqa: F401
from .hostpipe import HostBatch, run_host_batches  # noqa: F401
from .tensorio import load_tensor, read_fixture, read_tensor, save_tensor, write_fixture, write_tensor  # noqa: F401
from .planning import (  # noqa: F401
    account,
    build_pool,
    format_plan,
    generate_group_sizes,
    pad_rows,
    plan_group_stores,
    plan_prefetch,
    plan_two_phase,
    pool_heights,
    scale_row_bytes,
    window_rows,
)

from . import ops  # noqa: F401,E402  (registers torch.ops.tagg.*)

__version__ = "0.1.0"
