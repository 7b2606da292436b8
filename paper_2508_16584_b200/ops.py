"""torch.ops.tagg.* -- the grouped GEMM and the producer kernels as PyTorch operators
(SURVEY.md §8b, item 2).

Registered with torch.library for the CUDA device type only: there is no CPU kernel,
so a CPU tensor raises instead of silently falling back.  Each op has a fake
(meta) implementation, so the ops trace under torch.compile / FakeTensor and can
sit inside captured graphs.  The CUDA implementations call libtagg.so through
the C ABI, stream-ordered on the current stream, with no host sync.
"""

from __future__ import annotations

import torch

from . import engine, moe, quant

_LIB = "tagg"


@torch.library.custom_op(f"{_LIB}::grouped_gemm_fp8", mutates_args=(), device_types="cuda")
def grouped_gemm_fp8(a: torch.Tensor, a_scales: torch.Tensor, b: torch.Tensor, b_scales: torch.Tensor,
                     group_sizes: torch.Tensor, b_layout: str = "kn", exact_promotion: bool = False) -> torch.Tensor:
    """Padding-free FP8 grouped GEMM -> bf16 [m_alloc, N] (rows past sum(M_g) are unspecified)."""
    return engine.grouped_gemm_fp8(a, a_scales, b, b_scales, group_sizes, b_layout=b_layout,
                                   exact_promotion=exact_promotion)


@grouped_gemm_fp8.register_fake
def _(a, a_scales, b, b_scales, group_sizes, b_layout="kn", exact_promotion=False):
    n = b.shape[-1] if b_layout == "kn" else b.shape[-2]
    return a.new_empty((a.shape[0], n), dtype=torch.bfloat16)


@torch.library.custom_op(f"{_LIB}::quantize_row_tiles", mutates_args=(), device_types="cuda")
def quantize_row_tiles(x: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """fp8.py:132-151: (codes uint8 [rows, K], scales f32 [rows, ceil(K/128)])."""
    codes, scales = quant.quantize_row_tiles(x)
    return codes.contiguous(), scales


@quantize_row_tiles.register_fake
def _(x):
    k = x.shape[1]
    return x.new_empty((x.shape[0], k), dtype=torch.uint8), x.new_empty((x.shape[0], -(-k // 128)),
                                                                        dtype=torch.float32)


@torch.library.custom_op(f"{_LIB}::quantize_dispatch", mutates_args=(), device_types="cuda")
def quantize_dispatch(x: torch.Tensor, expert_ids: torch.Tensor,
                      num_experts: int) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor]:
    """Fused 1x128 quantize + dispatch: (a_codes, a_scales, group_sizes, dest_rows)."""
    d = quant.quantize_dispatch(x, expert_ids, num_experts)
    return d.a_codes.contiguous(), d.a_scales, d.group_sizes, d.dest_rows


@quantize_dispatch.register_fake
def _(x, expert_ids, num_experts):
    t, k = x.shape
    rows = expert_ids.numel()
    return (x.new_empty((rows, k), dtype=torch.uint8), x.new_empty((rows, -(-k // 128)), dtype=torch.float32),
            x.new_empty((num_experts,), dtype=torch.int32), x.new_empty((rows,), dtype=torch.int32))


@torch.library.custom_op(f"{_LIB}::wgrad_fp8", mutates_args=(), device_types="cuda")
def wgrad_fp8(x_codes: torch.Tensor, x_scales: torch.Tensor, dy_codes: torch.Tensor, dy_scales: torch.Tensor,
              group_sizes: torch.Tensor) -> torch.Tensor:
    """dW [G, K, N] bf16 = X_g^T dY_g (the K-grouped weight gradient)."""
    from . import wgrad

    return wgrad.wgrad_fp8(x_codes, x_scales, dy_codes, dy_scales, group_sizes)


@wgrad_fp8.register_fake
def _(x_codes, x_scales, dy_codes, dy_scales, group_sizes):
    return x_codes.new_empty((group_sizes.shape[0], x_codes.shape[1], dy_codes.shape[1]), dtype=torch.bfloat16)


@torch.library.custom_op(f"{_LIB}::swiglu_quantize", mutates_args=(), device_types="cuda")
def swiglu_quantize(h: torch.Tensor, group_sizes: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """gate|up bf16 rows -> the down GEMM's (codes, scales), padding-free (moe.py)."""
    a, sa = moe.swiglu_quantize(h, group_sizes)
    return a.contiguous(), sa


@swiglu_quantize.register_fake
def _(h, group_sizes):
    i = h.shape[1] // 2
    return h.new_empty((h.shape[0], i), dtype=torch.uint8), h.new_empty((h.shape[0], -(-i // 128)),
                                                                       dtype=torch.float32)


@torch.library.custom_op(f"{_LIB}::combine", mutates_args=(), device_types="cuda")
def combine(c: torch.Tensor, dest_rows: torch.Tensor, weights: torch.Tensor) -> torch.Tensor:
    """Top-k weighted combine of grouped rows back to tokens (moe.py)."""
    return moe.combine(c, dest_rows, weights)


@combine.register_fake
def _(c, dest_rows, weights):
    return c.new_empty((weights.shape[0], c.shape[1]), dtype=torch.bfloat16)
