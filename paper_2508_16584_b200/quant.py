"""Producer side of the padding-free grouped GEMM.

A device restatement of the reference's 1x128 quantizer (quantize_row_tiles,
fp8.py:132-151, with encode fp8.py:54-80), fused with the MoE dispatch
permutation: each token row is quantized once and its codes and scales are
written straight into every expert-contiguous row it is routed to.  That is the
padding-free grouped layout (no pad rows) grouped_gemm_fp8 consumes, together
with the device group sizes.

Kernels: csrc/tagg_quant.cu through the C ABI (include/tagg.h).  No CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from ._lib import lib
from .errors import InvalidInput, raise_for_status

_DTYPES = {torch.bfloat16: 0, torch.float32: 1}


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _check_cuda(t: torch.Tensor, what: str) -> None:
    if not t.is_cuda:
        raise InvalidInput(f"{what} must be a CUDA tensor (the product has no CPU path)")


def route_plan(expert_ids: torch.Tensor, num_experts: int, *, check: bool = False):
    """Stable counting sort of routed rows by expert.

    expert_ids: int [R] (CUDA).  Returns (group_sizes int32 [E], dest_rows int32 [R]):
    dest_rows[r] is row r's position in the expert-contiguous layout, experts in
    order and rows of one expert in ascending r.  check=True syncs and raises
    InvalidInput for an id outside [0, num_experts).
    """
    _check_cuda(expert_ids, "expert_ids")
    ids = expert_ids.reshape(-1).to(torch.int32).contiguous()
    rows = ids.numel()
    dev = ids.device
    gs = torch.empty(num_experts, dtype=torch.int32, device=dev)
    dest = torch.empty(rows, dtype=torch.int32, device=dev)
    ws = torch.empty(max(1, lib().tagg_route_workspace_ints(rows, num_experts)), dtype=torch.int32, device=dev)
    rc = lib().tagg_route_plan(ids.data_ptr() if rows else None, rows, num_experts, gs.data_ptr(),
                               dest.data_ptr() if rows else None, ws.data_ptr(), _stream())
    raise_for_status(rc, "tagg_route_plan")
    if check:
        torch.cuda.synchronize(dev)
        flag = torch.zeros(1, dtype=torch.int32).numpy()
        raise_for_status(lib().tagg_route_error(ws.data_ptr(), rows, num_experts, flag.ctypes.data), "route_error")
        if flag[0]:
            raise InvalidInput(f"expert id outside [0, {num_experts})")
    return gs, dest


def _quantize(x: torch.Tensor, topk: int, dest, out_rows: int, check: bool):
    _check_cuda(x, "x")
    if x.dim() != 2:
        raise InvalidInput("expected a 2-D matrix")
    if x.dtype not in _DTYPES:
        x = x.to(torch.float32)
    if x.stride(1) != 1:
        x = x.contiguous()
    t, k = x.shape
    if k < 1:
        raise InvalidInput("matrix must have at least one column")
    kb = -(-k // 128)
    lda = -(-k // 16) * 16  # 16-byte rows: the GEMM's TMA needs lda % 16 == 0
    a = torch.empty((out_rows, lda), dtype=torch.uint8, device=x.device)
    sa = torch.empty((out_rows, kb), dtype=torch.float32, device=x.device)
    err = torch.zeros(1, dtype=torch.int32, device=x.device)
    if t:
        rc = lib().tagg_quantize_dispatch(x.data_ptr(), _DTYPES[x.dtype], x.stride(0), t, k, topk,
                                          None if dest is None else dest.data_ptr(), a.data_ptr(), lda,
                                          sa.data_ptr(), err.data_ptr(), _stream())
        raise_for_status(rc, "tagg_quantize_dispatch")
    if check and int(err.item()):
        raise InvalidInput("matrix entries must be finite")
    return a[:, :k], sa


def quantize_row_tiles(x: torch.Tensor, *, check: bool = False):
    """fp8.py:132-151 on the GPU: (codes uint8 [rows, K], scales f32 [rows, ceil(K/128)]).

    Bit-identical to the reference for finite input (bf16 input is quantized as its
    exact f32 value).  check=True syncs and raises InvalidInput on non-finite entries.
    """
    return _quantize(x, 1, None, x.shape[0], check)


def quantize_gather_rows(x: torch.Tensor, index: torch.Tensor, row_weights: torch.Tensor | None = None, *,
                         check: bool = False):
    """quantize_row_tiles(bf16(row_weights[r] * x[index[r]])) without materialising the gathered rows
    (tagg_quantize_gather_rows): the codes and scales are bit-identical to gathering with
    moe.gather_scale_rows (K10) and then quantizing.  x: [T, K] bf16 / f32; index: int [R]."""
    _check_cuda(x, "x")
    if x.dim() != 2 or x.dtype not in _DTYPES or x.stride(1) != 1:
        raise ShapeMismatch("x must be a row-major bf16 / f32 matrix")
    idx = index.to(torch.int32).contiguous()
    w = None if row_weights is None else row_weights.to(torch.float32).contiguous()
    r, k = idx.numel(), x.shape[1]
    if k < 1:
        raise InvalidInput("matrix must have at least one column")
    kb = -(-k // 128)
    lda = -(-k // 16) * 16
    a = torch.empty((r, lda), dtype=torch.uint8, device=x.device)
    sa = torch.empty((r, kb), dtype=torch.float32, device=x.device)
    err = torch.zeros(1, dtype=torch.int32, device=x.device)
    if r:
        rc = lib().tagg_quantize_gather_rows(x.data_ptr(), _DTYPES[x.dtype], x.stride(0), idx.data_ptr(),
                                             None if w is None else w.data_ptr(), r, k, a.data_ptr(), lda,
                                             sa.data_ptr(), err.data_ptr(), _stream())
        raise_for_status(rc, "tagg_quantize_gather_rows")
    if check and int(err.item()):
        raise InvalidInput("matrix entries must be finite")
    return a[:, :k], sa


def quantize_blocks(w: torch.Tensor, *, check: bool = False):
    """fp8.py:154-176 on the GPU, batched over leading dims: one scale per 128x128 block.

    w: [..., rows, cols] bf16/f32 (e.g. per-expert weights [G, K, N]).  Returns
    (codes uint8 of w's shape, scales f32 [..., ceil(rows/128), ceil(cols/128)]),
    bit-identical to the reference for finite input.
    """
    _check_cuda(w, "w")
    if w.dim() < 2:
        raise InvalidInput("expected a matrix or a batch of matrices")
    if w.dtype not in _DTYPES:
        w = w.to(torch.float32)
    lead = w.shape[:-2]
    rows, cols = w.shape[-2:]
    w3 = w.reshape(-1, rows, cols)
    if w3.stride(-1) != 1:
        w3 = w3.contiguous()
    batch = w3.shape[0]
    rb, cb = -(-rows // 128), -(-cols // 128)
    codes = torch.empty((batch, rows, cols), dtype=torch.uint8, device=w.device)
    scales = torch.empty((batch, rb, cb), dtype=torch.float32, device=w.device)
    err = torch.zeros(1, dtype=torch.int32, device=w.device)
    if batch and rows and cols:
        rc = lib().tagg_quantize_blocks(w3.data_ptr(), _DTYPES[w3.dtype], batch, rows, cols, w3.stride(1),
                                        w3.stride(0), codes.data_ptr(), cols, rows * cols, scales.data_ptr(),
                                        err.data_ptr(), _stream())
        raise_for_status(rc, "tagg_quantize_blocks")
    if check and int(err.item()):
        raise InvalidInput("matrix entries must be finite")
    return codes.view(*lead, rows, cols), scales.view(*lead, rb, cb)


@dataclass
class DispatchedActivations:
    """Quantized activations in the padding-free grouped layout."""

    a_codes: torch.Tensor      # uint8 [T*topk, K], expert-contiguous
    a_scales: torch.Tensor     # f32 [T*topk, ceil(K/128)]
    group_sizes: torch.Tensor  # int32 [E] on the device (the GEMM's M_g)
    dest_rows: torch.Tensor    # int32 [T*topk]: grouped row of (token t, slot k) at t*topk + k
    topk: int


def quantize_dispatch(x: torch.Tensor, expert_ids: torch.Tensor, num_experts: int, *,
                      check: bool = False) -> DispatchedActivations:
    """Quantize token rows once and scatter them to their experts' rows.

    x: [T, K] bf16/f32 activations; expert_ids: int [T, topk] routing (topk <= 8).
    Grouped row dest_rows[t*topk + k] holds token t's codes and scales for expert
    expert_ids[t, k]; rows of one expert keep ascending (t, k) order.
    """
    _check_cuda(expert_ids, "expert_ids")
    if expert_ids.dim() == 1:
        expert_ids = expert_ids[:, None]
    t, topk = expert_ids.shape
    if x.shape[0] != t:
        raise InvalidInput(f"x has {x.shape[0]} rows, expert_ids {t}")
    if not 1 <= topk <= 8:
        raise InvalidInput("topk must be in [1, 8]")
    gs, dest = route_plan(expert_ids, num_experts, check=check)
    a, sa = _quantize(x, topk, dest, t * topk, check)
    return DispatchedActivations(a_codes=a, a_scales=sa, group_sizes=gs, dest_rows=dest, topk=topk)


def gather_rows(c: torch.Tensor, dest_rows: torch.Tensor, topk: int) -> torch.Tensor:
    """Inverse permutation for the combine: [T, topk, N] rows of the grouped output."""
    return c.index_select(0, dest_rows.to(torch.int64)).view(-1, topk, c.shape[1])
