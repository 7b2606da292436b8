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


def swiglu_quantize(h: torch.Tensor, group_sizes: torch.Tensor, *, check: bool = False, keep_v: bool = False):
    """bf16 [M, 2I] gate|up rows -> (codes uint8 [M, I], scales f32 [M, ceil(I/128)]).

    v = fl(silu(gate) * up) is quantized with the fp8.py:132-151 recipe.  Only the first
    sum(group_sizes) rows are written (sizes stay on the device).  keep_v=True also returns v
    in bf16 [M, I] (a training forward keeps it for the backward's wgrad).
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
    v = torch.empty((m, i), dtype=torch.bfloat16, device=h.device) if keep_v else None
    rc = lib().tagg_swiglu_quantize(h.data_ptr(), h.stride(0), gs.data_ptr(), gs.numel(), m, i, a.data_ptr(), lda,
                                    sa.data_ptr(), err.data_ptr(), None if v is None else v.data_ptr(),
                                    0 if v is None else v.stride(0), _stream())
    raise_for_status(rc, "tagg_swiglu_quantize")
    if check and int(err.item()):
        raise InvalidInput("silu(gate) * up is not finite")
    return (a[:, :i], sa, v) if keep_v else (a[:, :i], sa)


def gather_scale_rows(src: torch.Tensor, index: torch.Tensor, row_weights: torch.Tensor | None = None):
    """out[r] = bf16(row_weights[r] * src[index[r]]): token rows into the grouped layout (K10)."""
    if not src.is_cuda or src.dtype != torch.bfloat16 or src.stride(1) != 1:
        raise ShapeMismatch("src must be a row-major bf16 CUDA tensor")
    idx = index.to(torch.int32).contiguous()
    w = None if row_weights is None else row_weights.to(torch.float32).contiguous()
    out = torch.empty((idx.numel(), src.shape[1]), dtype=torch.bfloat16, device=src.device)
    rc = lib().tagg_gather_scale_rows(src.data_ptr(), src.stride(0), idx.data_ptr(), None if w is None else w.data_ptr(),
                                      idx.numel(), src.shape[1], out.data_ptr(), out.stride(0), _stream())
    raise_for_status(rc, "tagg_gather_scale_rows")
    return out


def router_grad(dy: torch.Tensor, c: torch.Tensor, dest_rows: torch.Tensor, topk: int) -> torch.Tensor:
    """g[t, k] = <dy[t], c[dest_rows[t*topk + k]]> in fp32 (K11)."""
    t = dy.shape[0]
    d = dest_rows.to(torch.int32).contiguous()
    out = torch.empty((t, topk), dtype=torch.float32, device=dy.device)
    rc = lib().tagg_router_grad(dy.data_ptr(), dy.stride(0), c.data_ptr(), c.stride(0), d.data_ptr(), t, topk,
                                dy.shape[1], out.data_ptr(), _stream())
    raise_for_status(rc, "tagg_router_grad")
    return out


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


def swiglu_backward_quantize(h: torch.Tensor, dh: torch.Tensor, group_sizes: torch.Tensor, *, want_bf16: bool = True,
                             check: bool = False):
    """Backward of swiglu_quantize (K9): (d[g|u] bf16 [M, 2I] or None, codes [M, 2I], scales [M, 2I/128]).

    dg = dh * u * sig(g) * (1 + g * (1 - sig(g))), du = dh * silu(g) from the saved gate|up rows h
    and dh = dL/d(silu(g) * u); the codes are the gate|up dgrad GEMM's A operand.
    """
    for t, what in ((h, "h"), (dh, "dh"), (group_sizes, "group_sizes")):
        if not t.is_cuda:
            raise InvalidInput(f"{what} must be a CUDA tensor (no CPU path)")
    m, i2 = h.shape
    i = i2 // 2
    if i % 128 or tuple(dh.shape) != (m, i) or h.stride(1) != 1 or dh.stride(1) != 1:
        raise ShapeMismatch(f"h {tuple(h.shape)} / dh {tuple(dh.shape)}: need [M, 2I] / [M, I], I % 128 == 0")
    dgu = torch.empty((m, 2 * i), dtype=torch.bfloat16, device=h.device) if want_bf16 else None
    a = torch.empty((m, 2 * i), dtype=torch.uint8, device=h.device)
    sa = torch.empty((m, 2 * i // 128), dtype=torch.float32, device=h.device)
    err = torch.zeros(1, dtype=torch.int32, device=h.device)
    gs = group_sizes.to(torch.int32).contiguous()
    rc = lib().tagg_swiglu_backward_quantize(h.data_ptr(), h.stride(0), dh.data_ptr(), dh.stride(0), gs.data_ptr(),
                                             gs.numel(), m, i, None if dgu is None else dgu.data_ptr(),
                                             0 if dgu is None else dgu.stride(0), a.data_ptr(), a.stride(0),
                                             sa.data_ptr(), err.data_ptr(), _stream())
    raise_for_status(rc, "tagg_swiglu_backward_quantize")
    if check and int(err.item()):
        raise InvalidInput("swiglu backward is not finite")
    return dgu, a, sa


@dataclass
class ExpertWeights:
    """FP8 expert weights, K-major per the reference layout [G, K, N] (b_layout "kn")."""

    w_gate_up: torch.Tensor   # uint8 [E, H, 2I]
    s_gate_up: torch.Tensor   # f32 [E, H/128, 2I/128]
    w_down: torch.Tensor      # uint8 [E, I, H]
    s_down: torch.Tensor      # f32 [E, I/128, H/128]


@dataclass
class MoeContext:
    """What the backward needs from the forward (all device tensors, grouped rows)."""

    x: torch.Tensor
    weights: torch.Tensor
    dispatch: quant.DispatchedActivations
    h: torch.Tensor        # gate|up GEMM output, bf16 [R, 2I]
    v: torch.Tensor        # silu(gate) * up, bf16 [R, I]
    c: torch.Tensor        # down GEMM output, bf16 [R, H]


@dataclass
class MoeGrads:
    dx: torch.Tensor          # bf16 [T, H]
    dw_gate_up: torch.Tensor  # bf16 [E, H, 2I]
    dw_down: torch.Tensor     # bf16 [E, I, H]
    dweights: torch.Tensor    # f32 [T, topk]


def moe_ffn(x: torch.Tensor, expert_ids: torch.Tensor, weights: torch.Tensor, w: ExpertWeights, *,
            save: bool = False):
    """Top-k MoE FFN forward on one GPU: five launches' worth of steps, all padding-free.
    save=True also returns the MoeContext for moe_ffn_backward."""
    e = w.w_gate_up.shape[0]
    d = quant.quantize_dispatch(x, expert_ids, e)
    h = grouped_gemm_fp8(d.a_codes, d.a_scales, w.w_gate_up, w.s_gate_up, d.group_sizes)
    if save:
        a2, s2, v = swiglu_quantize(h, d.group_sizes, keep_v=True)
    else:
        a2, s2 = swiglu_quantize(h, d.group_sizes)
    c = grouped_gemm_fp8(a2, s2, w.w_down, w.s_down, d.group_sizes)
    y = combine(c, d.dest_rows, weights)
    return (y, MoeContext(x, weights, d, h, v, c)) if save else y


def _mark(marks, name):
    """Optional step timing: append (name, recorded CUDA event)."""
    if marks is not None:
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        marks.append((name, ev))


WGRAD_RECIPES = ("per_column", "dy_block128", "mxfp8")


def moe_ffn_backward(dy: torch.Tensor, ctx: MoeContext, w: ExpertWeights, *, marks: list | None = None,
                     wgrad_recipe: str = "per_column") -> MoeGrads:
    """Backward of moe_ffn, padding-free end to end.

    * dgrad: the two GEMMs again with the same FP8 weights read K-major (b_layout "nk");
    * SwiGLU backward + quantize (K9);
    * wgrad: the K-grouped GEMM (K6) over column-quantized activations and gradients, in one of
      three recipes (``wgrad_recipe``): "per_column" fp32 scales per (token block, column) on
      both sides (the default), "dy_block128" the gradient side with one scale per (token block,
      128 columns) (one FFMA2 per pair in the promotion), or "mxfp8" power-of-two scales applied
      by the tensor core (no per-block promotion);
    * dx: the top-k combine (K8) with unit weights; d(router weights): row dot products.
    Row gathers (K10) and the router-weight dot products (K11) are kernels too; only index
    arithmetic on [R] int vectors is torch.
    """
    from .wgrad import quantize_col_blocks, quantize_col_blocks_mx, wgrad_fp8, wgrad_fp8_mx

    if wgrad_recipe not in WGRAD_RECIPES:
        raise InvalidInput(f"wgrad_recipe must be one of {WGRAD_RECIPES}")

    def wgrad(xs, xi, xw, ys, yi, yw, name):
        """dW = X^T dY per group; X / dY rows optionally gathered (index) and weighted."""
        if wgrad_recipe == "mxfp8":
            xq, _, xf = quantize_col_blocks_mx(xs, gs, index=xi, row_weights=xw)
            yq, _, yf = quantize_col_blocks_mx(ys, gs, index=yi, row_weights=yw)
            _mark(marks, name + "_quantize")
            return wgrad_fp8_mx(xq, xf, yq, yf, gs)
        xq, xsc = quantize_col_blocks(xs, gs, index=xi, row_weights=xw)
        block = wgrad_recipe == "dy_block128"
        yq, ysc = quantize_col_blocks(ys, gs, index=yi, row_weights=yw, block_cols=128 if block else 1)
        _mark(marks, name + "_quantize")
        return wgrad_fp8(xq, xsc, yq, ysc, gs, dy_block128=block)

    _mark(marks, "start")
    d = ctx.dispatch
    gs = d.group_sizes
    t, topk = ctx.weights.shape
    dest = d.dest_rows.to(torch.int64)
    order = torch.empty_like(dest)
    order[dest] = torch.arange(dest.numel(), device=dest.device)   # grouped row -> (token, k)
    src = order // topk
    w_rows = ctx.weights.reshape(-1).index_select(0, order).to(torch.float32)
    # dL/dc for the grouped rows: w[t,k] * dy[t] (K10's values), 1x128-quantized in the same pass
    dc_codes, dc_scales = quant.quantize_gather_rows(dy, src, w_rows)  # K10's rows, quantized in place
    _mark(marks, "dc_gather_quantize")
    dh2 = grouped_gemm_fp8(dc_codes, dc_scales, w.w_down, w.s_down, gs, b_layout="nk")
    _mark(marks, "dgrad_down")
    dgu, dgu_codes, dgu_scales = swiglu_backward_quantize(ctx.h, dh2, gs)
    _mark(marks, "swiglu_backward")
    dxd = grouped_gemm_fp8(dgu_codes, dgu_scales, w.w_gate_up, w.s_gate_up, gs, b_layout="nk")
    _mark(marks, "dgrad_gate_up")
    dx = combine(dxd, d.dest_rows, torch.ones((t, topk), dtype=torch.float32, device=dy.device))
    _mark(marks, "dx_combine")
    # wgrad: dW_down = H2^T dC, dW_gu = X^T dGU, per group
    # (dC rows are w[t,k] dy[t] and X rows x[t], both gathered in place by the quantizer)
    dw_down = wgrad(ctx.v, None, None, dy, src, w_rows, "wgrad_down")
    _mark(marks, "wgrad_down")
    dw_gate_up = wgrad(ctx.x, src, None, dgu, None, None, "wgrad_gate_up")
    _mark(marks, "wgrad_gate_up")
    # d(router weight)[t, k] = <dy[t], c[dest(t, k)]>
    dweights = router_grad(dy, ctx.c, d.dest_rows, topk)
    _mark(marks, "router_grads")
    return MoeGrads(dx, dw_gate_up, dw_down, dweights)
