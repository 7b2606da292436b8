"""ctypes binding of libtagg.so (include/tagg.h), the product's C ABI.

The library is built in-tree (``make -C paper_2508_16584_b200/csrc``, or
``__graft_entry__.build()``).  There is no fallback: if the shared object is
missing, every GPU entry point raises instead of computing on the CPU.
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libtagg.so"

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_u32 = ctypes.c_uint32
c_vp = ctypes.c_void_p

# symbol -> (restype, argtypes), exactly the declarations of include/tagg.h
SIGNATURES = {
    "tagg_grouped_gemm_fp8": (c_int, [c_vp, c_i64, c_vp, c_i64, c_vp, c_int, c_int, c_vp, c_i64, c_i64,
                                      c_i64, c_vp, c_int, c_int, c_int, c_vp, c_i64, c_i64, c_vp, c_vp,
                                      c_u32, c_vp]),
    "tagg_grouped_gemm_fp8_ex": (c_int, [c_vp, c_i64, c_vp, c_i64, c_vp, c_int, c_int, c_vp, c_i64, c_i64,
                                         c_i64, c_vp, c_int, c_int, c_int, c_vp, c_i64, c_i64, c_vp, c_vp,
                                         c_vp, c_vp, c_u32, c_vp]),
    "tagg_max_tiles": (c_i64, [c_i64, c_int, c_int]),
    "tagg_launch_clusters": (c_int, [c_i64, c_int, c_int, c_u32]),
    "tagg_pad_groups": (c_int, [c_vp, c_i64, c_vp, c_vp, c_int, c_int, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "tagg_unpad_rows": (c_int, [c_vp, c_vp, c_int, c_int, c_vp, c_i64, c_vp]),
    "tagg_padded_rows_bound": (c_i64, [c_i64, c_int]),
    "tagg_route_workspace_ints": (c_i64, [c_i64, c_int]),
    "tagg_token_blocks_bound": (c_i64, [c_i64, c_int]),
    "tagg_quantize_col_blocks": (c_int, [c_vp, c_int, c_i64, c_int, c_i64, c_vp, c_int, c_vp, c_i64, c_vp, c_vp,
                                         c_vp]),
    "tagg_quantize_col_blocks_gather": (c_int, [c_vp, c_int, c_i64, c_vp, c_vp, c_i64, c_int, c_vp, c_int, c_vp,
                                                c_i64, c_vp, c_vp, c_vp]),
    "tagg_wgrad_fp8": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_int, c_int, c_int, c_vp, c_vp]),
    "tagg_wgrad_fp8_ex": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_int, c_int, c_int, c_vp, c_u32, c_vp]),
    "tagg_wgrad_fp8_mx": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_int, c_int, c_int, c_vp, c_vp]),
    "tagg_quantize_col_blocks_mx": (c_int, [c_vp, c_int, c_i64, c_vp, c_vp, c_i64, c_int, c_vp, c_int, c_vp, c_i64,
                                            c_vp, c_vp, c_vp, c_vp]),
    "tagg_quantize_col_blocks_ex": (c_int, [c_vp, c_int, c_i64, c_vp, c_vp, c_i64, c_int, c_vp, c_int, c_vp, c_i64,
                                            c_vp, c_vp, c_int, c_vp]),
    "tagg_quantize_blocks": (c_int, [c_vp, c_int, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_i64, c_vp, c_vp,
                                     c_vp]),
    "tagg_swiglu_quantize": (c_int, [c_vp, c_i64, c_vp, c_int, c_i64, c_int, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64,
                                     c_vp]),
    "tagg_gather_scale_rows": (c_int, [c_vp, c_i64, c_vp, c_vp, c_i64, c_int, c_vp, c_i64, c_vp]),
    "tagg_router_grad": (c_int, [c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_int, c_int, c_vp, c_vp]),
    "tagg_combine": (c_int, [c_vp, c_i64, c_vp, c_vp, c_i64, c_int, c_int, c_vp, c_i64, c_vp]),
    "tagg_swiglu_backward_quantize": (c_int, [c_vp, c_i64, c_vp, c_i64, c_vp, c_int, c_i64, c_int, c_vp, c_i64, c_vp,
                                              c_i64, c_vp, c_vp, c_vp]),
    "tagg_route_plan": (c_int, [c_vp, c_i64, c_int, c_vp, c_vp, c_vp, c_vp]),
    "tagg_route_error": (c_int, [c_vp, c_i64, c_int, c_vp]),
    "tagg_quantize_gather_rows": (c_int, [c_vp, c_int, c_i64, c_vp, c_vp, c_i64, c_int, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "tagg_quantize_dispatch": (c_int, [c_vp, c_int, c_i64, c_i64, c_int, c_int, c_vp, c_vp, c_i64, c_vp, c_vp,
                                       c_vp]),
    "tagg_validate_config": (c_int, [c_i64, c_i64, c_vp, c_int, c_i64, c_i64, c_i64]),
    "tagg_plan_group_stores": (c_int, [c_vp, c_int, c_i64, c_vp]),
    "tagg_pool_heights": (c_int, [c_i64, c_vp, c_int]),
    "tagg_pool_select": (c_i64, [c_i64, c_i64]),
    "tagg_plan_prefetch": (c_int, [c_i64, c_i64, c_i64, c_vp]),
    "tagg_pad_rows": (c_i64, [c_vp, c_int, c_i64]),
    "tagg_error_string": (ctypes.c_char_p, [c_int]),
    "tagg_version": (c_int, []),
    "tagg_debug_trace": (None, [c_vp]),
}

_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(PKG / "csrc")], check=True)
    return LIB_PATH


def lib():
    """The loaded libtagg.so; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(the product has no CPU fallback)")
        L = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
