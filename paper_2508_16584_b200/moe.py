"""The MoE FFN around the padding-free grouped GEMM (widening beyond SURVEY.md §8f).

    x --quantize_dispatch--> A1 (grouped rows) --GEMM gate|up--> H --swiglu_quantize--> A2
      --GEMM down--> C --combine (top-k weights)--> y

Every intermediate stays in the padding-free grouped layout: no pad rows and no
permutation between the two GEMMs.  The two new steps (csrc/tagg_moe.cu, K7 / K8) are
HBM-bound; the GEMMs are K1.  No CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import quant
from ._lib import lib
from .engine import grouped_gemm_fp8
from .errors import InvalidInput, ShapeMismatch, raise_for_status


def _stream():
    return torch.cuda.current_stream().cuda_stream


def swiglu_quantize(h: torch.Tensor, group_sizes: torch.Tensor, *, check: bool = False):
    """bf16 [M, 2I] gate|up rows -> (codes uint8 [M, I], scales f32 [M, ceil(I/128)]).

    v = fl(silu(gate) * up) is quantized with the fp8.py:132-151 recipe.  Only the first
    sum(group_sizes) rows are written (sizes stay on the device).
    """
    if not h.is_cuda or not group_sizes.is_cuda:
        raise InvalidInput("swiglu_quantize expects CUDA tensors (no CPU path)")
    if h.dtype not in (torch.bfloat16, torch.int16, torch.uint16) or h.dim() != 2 or h.stride(1) != 1:
        raise ShapeMismatch("h must be a row-major bf16 [M, 2I] tensor")
    if h.shape[1] % 2:
        raise ShapeMismatch("h must have an even number of columns (gate | up)")
    m, i2 = h.shape
    i = i2 // 2
    lda = -(-i // 16) * 16
    a = torch.empty((m, lda), dtype=torch.uint8, device=h.device)
    sa = torch.empty((m, -(-i // 128)), dtype=torch.float32, device=h.device)
    err = torch.zeros(1, dtype=torch.int32, device=h.device)
    gs = group_sizes.to(torch.int32).contiguous()
    rc = lib().tagg_swiglu_quantize(h.data_ptr(), h.stride(0), gs.data_ptr(), gs.numel(), m, i, a.data_ptr(), lda,
                                    sa.data_ptr(), err.data_ptr(), _stream())
    raise_for_status(rc, "tagg_swiglu_quantize")
    if check and int(err.item()):
        raise InvalidInput("silu(gate) * up is not finite")
    return a[:, :i], sa


def combine(c: torch.Tensor, dest_rows: torch.Tensor, weights: torch.Tensor) -> torch.Tensor:
    """y[t] = bf16(sum_k fl(w[t,k] * c[dest_rows[t*topk+k]])), fp32 in k order (no FMA).

    c: bf16 [rows, N] grouped GEMM output; dest_rows: int32 [T*topk] from the dispatch plan;
    weights: f32 [T, topk] router weights.
    """
    if not c.is_cuda:
        raise InvalidInput("combine expects CUDA tensors (no CPU path)")
    if weights.dim() != 2:
        raise ShapeMismatch("weights must be [tokens, topk]")
    t, topk = weights.shape
    if dest_rows.numel() != t * topk:
        raise ShapeMismatch(f"dest_rows has {dest_rows.numel()} entries, expected {t * topk}")
    n = c.shape[1]
    w = weights.to(torch.float32).contiguous()
    d = dest_rows.to(torch.int32).contiguous()
    out = torch.empty((t, n), dtype=torch.bfloat16, device=c.device)
    rc = lib().tagg_combine(c.data_ptr(), c.stride(0), d.data_ptr(), w.data_ptr(), t, topk, n, out.data_ptr(),
                            out.stride(0), _stream())
    raise_for_status(rc, "tagg_combine")
    return out


@dataclass
class ExpertWeights:
    """FP8 expert weights, K-major per the reference layout [G, K, N] (b_layout "kn")."""

    w_gate_up: torch.Tensor   # uint8 [E, H, 2I]
    s_gate_up: torch.Tensor   # f32 [E, H/128, 2I/128]
    w_down: torch.Tensor      # uint8 [E, I, H]
    s_down: torch.Tensor      # f32 [E, I/128, H/128]


def moe_ffn(x: torch.Tensor, expert_ids: torch.Tensor, weights: torch.Tensor, w: ExpertWeights) -> torch.Tensor:
    """Top-k MoE FFN forward on one GPU: five launches' worth of steps, all padding-free."""
    e = w.w_gate_up.shape[0]
    d = quant.quantize_dispatch(x, expert_ids, e)
    h = grouped_gemm_fp8(d.a_codes, d.a_scales, w.w_gate_up, w.s_gate_up, d.group_sizes)
    a2, s2 = swiglu_quantize(h, d.group_sizes)
    c = grouped_gemm_fp8(a2, s2, w.w_down, w.s_down, d.group_sizes)
    return combine(c, d.dest_rows, weights)
