"""Backward: the MoE weight gradient as a K-grouped FP8 GEMM.

dW_g = X_g^T dY_g over each expert's ragged rows, from operands quantized per
(group, 128-token block, column) -- the forward's 1x128 recipe (fp8.py:132-151) turned
to run down the token axis, which is the reduction axis here.  Kernels:
csrc/tagg_wgrad.cu through the C ABI.  dgrad needs no new kernel: it is the forward
grouped GEMM with K-major B (grouped_gemm_fp8(..., b_layout="nk")).
"""

from __future__ import annotations

import torch

from ._lib import lib
from .errors import InvalidInput, ShapeMismatch, raise_for_status
from .quant import _DTYPES, _check_cuda, _stream


TAGG_QCB_SCALE_POW2 = 0x10000  # include/tagg.h
TAGG_WGRAD_DY_BLOCK128 = 1


def quantize_col_blocks(x: torch.Tensor, group_sizes: torch.Tensor, *, check: bool = False,
                        index: torch.Tensor | None = None, row_weights: torch.Tensor | None = None,
                        block_cols: int = 1, scale_pow2: bool = False):
    """(codes uint8 [M, C], scales f32 [TB_bound, C]) for x [M, C] in the grouped layout.

    Scale row tb holds the tb-th (group, 128-token block) in group order; only the first
    sum(ceil(M_g/128)) rows are defined (group sizes stay on the device: no host sync).
    With ``index`` (int [M]), grouped row r is ``row_weights[r] * x[index[r]]`` (weights
    optional): token-ordered rows are quantized into the grouped layout without a copy.
    ``block_cols=128``: one scale per (token block, 128 columns) -- the 128x128 block recipe
    of fp8.py:154-176 per group token block -- repeated in its 128 columns' slots; a dY
    quantized this way lets ``wgrad_fp8(..., dy_block128=True)`` promote with one op per pair.
    ``scale_pow2``: every scale is rounded up to a power of two (the MXFP8 recipe: x / s is exact
    and s is one E8M0 byte); quantize_col_blocks_mx also returns the E8M0 factor blocks that
    wgrad_fp8_mx takes.
    """
    if block_cols not in (1, 128):
        raise InvalidInput("block_cols must be 1 or 128")
    if block_cols == 128 or scale_pow2:
        return _quantize_col_blocks_ex(x, group_sizes, index, row_weights, check,
                                       block_cols | (TAGG_QCB_SCALE_POW2 if scale_pow2 else 0))
    if index is not None:
        return _quantize_col_blocks_gather(x, group_sizes, index, row_weights, check)
    _check_cuda(x, "x")
    if x.dim() != 2:
        raise InvalidInput("expected a 2-D matrix")
    if x.dtype not in _DTYPES:
        x = x.to(torch.float32)
    if x.stride(1) != 1:
        x = x.contiguous()
    if group_sizes.dtype != torch.int32 or not group_sizes.is_cuda:
        raise ShapeMismatch("group_sizes must be an int32 CUDA tensor")
    m, c = x.shape
    g = group_sizes.numel()
    tb = lib().tagg_token_blocks_bound(m, g)
    codes = torch.empty((m, c), dtype=torch.uint8, device=x.device)
    scales = torch.empty((max(tb, 1), c), dtype=torch.float32, device=x.device)
    err = torch.zeros(1, dtype=torch.int32, device=x.device)
    rc = lib().tagg_quantize_col_blocks(x.data_ptr(), _DTYPES[x.dtype], m, c, x.stride(0), group_sizes.data_ptr(),
                                        g, codes.data_ptr(), c, scales.data_ptr(), err.data_ptr(), _stream())
    raise_for_status(rc, "tagg_quantize_col_blocks")
    if check and int(err.item()):
        raise InvalidInput("matrix entries must be finite")
    return codes, scales


def _quantize_col_blocks_gather(x, group_sizes, index, row_weights, check):
    _check_cuda(x, "x")
    if x.dim() != 2 or x.dtype not in _DTYPES or x.stride(1) != 1:
        raise ShapeMismatch("x must be a row-major bf16 / f32 matrix")
    if group_sizes.dtype != torch.int32 or not group_sizes.is_cuda:
        raise ShapeMismatch("group_sizes must be an int32 CUDA tensor")
    idx = index.to(torch.int32).contiguous()
    w = None if row_weights is None else row_weights.to(torch.float32).contiguous()
    m, c = idx.numel(), x.shape[1]
    g = group_sizes.numel()
    tb = lib().tagg_token_blocks_bound(m, g)
    codes = torch.empty((m, c), dtype=torch.uint8, device=x.device)
    scales = torch.empty((max(tb, 1), c), dtype=torch.float32, device=x.device)
    err = torch.zeros(1, dtype=torch.int32, device=x.device)
    rc = lib().tagg_quantize_col_blocks_gather(x.data_ptr(), _DTYPES[x.dtype], x.stride(0), idx.data_ptr(),
                                               None if w is None else w.data_ptr(), m, c, group_sizes.data_ptr(), g,
                                               codes.data_ptr(), c, scales.data_ptr(), err.data_ptr(), _stream())
    raise_for_status(rc, "tagg_quantize_col_blocks_gather")
    if check and int(err.item()):
        raise InvalidInput("matrix entries must be finite")
    return codes, scales


def _quantize_col_blocks_ex(x, group_sizes, index, row_weights, check, block_cols):
    _check_cuda(x, "x")
    if x.dim() != 2 or x.dtype not in _DTYPES or x.stride(1) != 1:
        raise ShapeMismatch("x must be a row-major bf16 / f32 matrix")
    if group_sizes.dtype != torch.int32 or not group_sizes.is_cuda:
        raise ShapeMismatch("group_sizes must be an int32 CUDA tensor")
    idx = None if index is None else index.to(torch.int32).contiguous()
    w = None if row_weights is None else row_weights.to(torch.float32).contiguous()
    m, c = (x.shape[0] if idx is None else idx.numel()), x.shape[1]
    g = group_sizes.numel()
    tb = lib().tagg_token_blocks_bound(m, g)
    codes = torch.empty((m, c), dtype=torch.uint8, device=x.device)
    scales = torch.empty((max(tb, 1), c), dtype=torch.float32, device=x.device)
    err = torch.zeros(1, dtype=torch.int32, device=x.device)
    rc = lib().tagg_quantize_col_blocks_ex(x.data_ptr(), _DTYPES[x.dtype], x.stride(0),
                                           None if idx is None else idx.data_ptr(), None if w is None else w.data_ptr(),
                                           m, c, group_sizes.data_ptr(), g, codes.data_ptr(), c, scales.data_ptr(),
                                           err.data_ptr(), block_cols, _stream())
    raise_for_status(rc, "tagg_quantize_col_blocks_ex")
    if check and int(err.item()):
        raise InvalidInput("matrix entries must be finite")
    return codes, scales


def wgrad_fp8(x_codes, x_scales, dy_codes, dy_scales, group_sizes, out=None, *, dy_block128=False) -> torch.Tensor:
    """dW [G, K, N] bf16 = X_g^T dY_g per group (K, N multiples of 128).  ``dy_block128``: dY's
    scales are constant per 128 columns (quantize_col_blocks(..., block_cols=128)); the promotion
    then takes one FFMA2 per element pair (TAGG_WGRAD_DY_BLOCK128).  The MXFP8 recipe has its
    own entry point, wgrad_fp8_mx."""
    for t, what in ((x_codes, "x_codes"), (dy_codes, "dy_codes")):
        _check_cuda(t, what)
    if x_codes.dtype == torch.float8_e4m3fn:
        x_codes = x_codes.view(torch.uint8)
    if dy_codes.dtype == torch.float8_e4m3fn:
        dy_codes = dy_codes.view(torch.uint8)
    m, k = x_codes.shape
    n = dy_codes.shape[1]
    if dy_codes.shape[0] != m:
        raise ShapeMismatch("X and dY need the same rows")
    for t in (x_codes, dy_codes, x_scales, dy_scales):
        if not t.is_contiguous():
            raise ShapeMismatch("operands must be contiguous")
    if x_scales.shape[1] != k or dy_scales.shape[1] != n:
        raise ShapeMismatch("scales must be [TB, K] and [TB, N]")
    if group_sizes.dtype != torch.int32 or not group_sizes.is_cuda:
        raise ShapeMismatch("group_sizes must be an int32 CUDA tensor")
    g = group_sizes.numel()
    tb = lib().tagg_token_blocks_bound(m, g)
    if x_scales.dtype != torch.float32 or dy_scales.dtype != torch.float32:
        raise ShapeMismatch("scales must be float32")
    if x_scales.shape[0] < tb or dy_scales.shape[0] < tb:
        raise ShapeMismatch(f"scales need >= {tb} token-block rows (tagg_token_blocks_bound)")
    if out is None:
        out = torch.empty((g, k, n), dtype=torch.bfloat16, device=x_codes.device)
    if (out.dtype not in (torch.bfloat16, torch.int16, torch.uint16) or tuple(out.shape) != (g, k, n)
            or not out.is_contiguous() or out.device != x_codes.device):
        raise ShapeMismatch(f"out must be a contiguous bf16 [{g}, {k}, {n}] tensor on the operands' device")
    rc = lib().tagg_wgrad_fp8_ex(x_codes.data_ptr(), x_scales.data_ptr(), dy_codes.data_ptr(), dy_scales.data_ptr(),
                                 m, group_sizes.data_ptr(), g, k, n, out.data_ptr(),
                                 TAGG_WGRAD_DY_BLOCK128 if dy_block128 else 0, _stream())
    raise_for_status(rc, "tagg_wgrad_fp8")
    return out


def quantize_col_blocks_mx(x: torch.Tensor, group_sizes: torch.Tensor, *, check: bool = False,
                           index: torch.Tensor | None = None, row_weights: torch.Tensor | None = None):
    """The MXFP8 recipe of quantize_col_blocks (cols % 128 == 0): power-of-two scales
    s = pow2_ceil(fl(amax / 448)) per (group token block, column), exact quotients, and the scales'
    E8M0 exponent bytes laid out for the tensor core (tagg_quantize_col_blocks_mx).  Returns
    (codes uint8 [M, C], scales f32 [TB_bound, C], sf uint8 [TB_bound, C / 128, 512])."""
    _check_cuda(x, "x")
    if x.dim() != 2 or x.dtype not in _DTYPES or x.stride(1) != 1:
        raise ShapeMismatch("x must be a row-major bf16 / f32 matrix")
    if group_sizes.dtype != torch.int32 or not group_sizes.is_cuda:
        raise ShapeMismatch("group_sizes must be an int32 CUDA tensor")
    if x.shape[1] % 128:
        raise ShapeMismatch("the MXFP8 quantizer needs a multiple of 128 columns")
    idx = None if index is None else index.to(torch.int32).contiguous()
    w = None if row_weights is None else row_weights.to(torch.float32).contiguous()
    m, c = (x.shape[0] if idx is None else idx.numel()), x.shape[1]
    g = group_sizes.numel()
    tb = max(lib().tagg_token_blocks_bound(m, g), 1)
    codes = torch.empty((m, c), dtype=torch.uint8, device=x.device)
    scales = torch.empty((tb, c), dtype=torch.float32, device=x.device)
    sf = torch.empty((tb, c // 128, 512), dtype=torch.uint8, device=x.device)
    err = torch.zeros(1, dtype=torch.int32, device=x.device)
    rc = lib().tagg_quantize_col_blocks_mx(x.data_ptr(), _DTYPES[x.dtype], x.stride(0),
                                           None if idx is None else idx.data_ptr(), None if w is None else w.data_ptr(),
                                           m, c, group_sizes.data_ptr(), g, codes.data_ptr(), c, scales.data_ptr(),
                                           sf.data_ptr(), err.data_ptr(), _stream())
    raise_for_status(rc, "tagg_quantize_col_blocks_mx")
    if check and int(err.item()):
        raise InvalidInput("matrix entries must be finite")
    return codes, scales, sf


def wgrad_fp8_mx(x_codes, x_sf, dy_codes, dy_sf, group_sizes, out=None) -> torch.Tensor:
    """dW [G, K, N] bf16 = X_g^T dY_g from MXFP8 operands (quantize_col_blocks_mx): the tensor
    core applies the E8M0 factors as block scales (tcgen05.mma kind::mxf8f6f4.block_scale) and
    accumulates each tile's whole token range in TMEM -- no per-block promotion
    (tagg_wgrad_fp8_mx)."""
    for t, what in ((x_codes, "x_codes"), (dy_codes, "dy_codes"), (x_sf, "x_sf"), (dy_sf, "dy_sf")):
        _check_cuda(t, what)
    if x_codes.dtype == torch.float8_e4m3fn:
        x_codes = x_codes.view(torch.uint8)
    if dy_codes.dtype == torch.float8_e4m3fn:
        dy_codes = dy_codes.view(torch.uint8)
    m, k = x_codes.shape
    n = dy_codes.shape[1]
    if dy_codes.shape[0] != m:
        raise ShapeMismatch("X and dY need the same rows")
    for t in (x_codes, dy_codes, x_sf, dy_sf):
        if not t.is_contiguous():
            raise ShapeMismatch("operands must be contiguous")
    if group_sizes.dtype != torch.int32 or not group_sizes.is_cuda:
        raise ShapeMismatch("group_sizes must be an int32 CUDA tensor")
    g = group_sizes.numel()
    tb = lib().tagg_token_blocks_bound(m, g)
    if (x_sf.dtype != torch.uint8 or dy_sf.dtype != torch.uint8 or tuple(x_sf.shape[1:]) != (k // 128, 512)
            or tuple(dy_sf.shape[1:]) != (n // 128, 512) or x_sf.shape[0] < tb or dy_sf.shape[0] < tb):
        raise ShapeMismatch(f"factor blocks must be uint8 [>= {tb}, columns / 128, 512] (quantize_col_blocks_mx)")
    if out is None:
        out = torch.empty((g, k, n), dtype=torch.bfloat16, device=x_codes.device)
    if (out.dtype not in (torch.bfloat16, torch.int16, torch.uint16) or tuple(out.shape) != (g, k, n)
            or not out.is_contiguous() or out.device != x_codes.device):
        raise ShapeMismatch(f"out must be a contiguous bf16 [{g}, {k}, {n}] tensor on the operands' device")
    rc = lib().tagg_wgrad_fp8_mx(x_codes.data_ptr(), x_sf.data_ptr(), dy_codes.data_ptr(), dy_sf.data_ptr(), m,
                                 group_sizes.data_ptr(), g, k, n, out.data_ptr(), _stream())
    raise_for_status(rc, "tagg_wgrad_fp8_mx")
    return out
