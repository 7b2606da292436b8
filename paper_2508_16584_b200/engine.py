"""Drop-in grouped-GEMM entry points (reference engine.py), running on B200.

Reference interface mirrored (paths relative to /root/reference/pkg/src/tma_sim/):

* ``ProblemConfig``        engine.py:58-120   (the same fields, validation and errors)
* ``GroupedOperands``      engine.py:123-148  (adds per-expert B [G,K,N] or [G,N,K])
* ``run_adaptive``         engine.py:184-343  -> one launch of the sm_100a kernel
* ``run_padded_baseline``  engine.py:346-402  -> pad kernel + the same GEMM + unpad kernel
* ``verify_bitwise``       engine.py:415-423
* ``bf16_from_f32`` / ``f32_from_bf16`` engine.py:46-55

The device-level API is ``grouped_gemm_fp8``.  It takes torch CUDA tensors,
DEVICE group sizes and a stream.  It has no host sync.  Everything funnels into
the C ABI of libtagg.so (include/tagg.h).  There is no CPU fallback: without a
CUDA device or the built library, the calls raise.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import planning
from ._lib import lib
from .errors import ConfigError, InvalidBlockM, InvalidBlockN, ShapeMismatch, raise_for_status

K_BLOCK = 128
FLAG_EXACT_PROMOTION = 1
FLAG_PLAIN_C_STAGING = 2
FLAG_SINGLE_CTA = 4
FLAG_TILE_N128 = 8
FLAG_TILE_N256 = 16
FLAG_SERIAL = 32  # no programmatic dependent launch (include/tagg.h TAGG_FLAG_SERIAL)
FLAG_PDL_OVERLAP = 64  # inputs not written by the previous kernel: overlap its tail (TAGG_FLAG_PDL_OVERLAP)
ERR_NEGATIVE_SIZE = 1  # device error flag bits (tagg_grouped_gemm_fp8_checked)
ERR_ROWS_OUT_OF_RANGE = 2
ERR_B_INDEX = 4
SM_LIMIT_SHIFT = 16  # TAGG_SM_LIMIT(n): cap the persistent grid at n SMs (include/tagg.h)
TILES = {None: 0, "auto": 0, "1cta": FLAG_SINGLE_CTA, "pair_n128": FLAG_TILE_N128, "pair_n256": FLAG_TILE_N256}
TILE_MAP_FIELDS = 9


def bf16_from_f32(x: np.ndarray) -> np.ndarray:
    """engine.py:46-50: float32 -> bfloat16 bits, ties to even."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    rounded = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
    return rounded.astype(np.uint16)


def f32_from_bf16(bits: np.ndarray) -> np.ndarray:
    """engine.py:53-55"""
    u = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return u.view(np.float32)


def num_blocks(n: int) -> int:
    return -(-int(n) // K_BLOCK)


@dataclass(frozen=True)
class ProblemConfig:
    """engine.py:58-120.  The same constraints, raising the same exception types."""

    n: int
    k: int
    group_sizes: tuple
    block_m: int = 128
    block_n: int = 128
    block_k: int = K_BLOCK

    def __post_init__(self):
        if self.k < 16 or self.k % 16 != 0:
            raise ConfigError(f"k must be a positive multiple of 16, got {self.k}")
        if self.n < 64 or self.n % 64 != 0:
            raise ConfigError(f"n must be a positive multiple of 64, got {self.n}")
        if self.block_m < 1 or self.block_m & (self.block_m - 1):
            raise InvalidBlockM(f"block_m must be a power of two, got {self.block_m}")
        if self.block_n < 64 or self.block_n % 64 != 0:
            raise InvalidBlockN(f"block_n must be a positive multiple of 64, got {self.block_n}")
        if self.block_k != K_BLOCK:
            raise ConfigError(f"block_k is fixed at {K_BLOCK} (scale granularity)")
        if len(self.group_sizes) == 0:
            raise ConfigError("need at least one group")
        if any(int(g) < 0 for g in self.group_sizes):
            raise ConfigError("group sizes must be non-negative")
        object.__setattr__(self, "group_sizes", tuple(int(g) for g in self.group_sizes))

    @property
    def groups(self) -> int:
        return len(self.group_sizes)

    @property
    def m_total(self) -> int:
        return sum(self.group_sizes)

    @property
    def k_blocks(self) -> int:
        return num_blocks(self.k)

    @property
    def n_scale_blocks(self) -> int:
        return num_blocks(self.n)

    def row_offsets(self) -> list[int]:
        off, out = 0, []
        for g in self.group_sizes:
            out.append(off)
            off += g
        return out

    def n_tiles(self) -> list[tuple[int, int]]:
        return [(c, min(self.block_n, self.n - c)) for c in range(0, self.n, self.block_n)]


def _codes(x):
    """Fp8Tensor-like, numpy uint8, or torch uint8 / float8_e4m3fn -> array-like."""
    return getattr(x, "codes", x)


@dataclass(frozen=True)
class GroupedOperands:
    """engine.py:123-148, generalised: B may be shared [K,N] (the reference) or
    per expert, [G,K,N] (b_layout "kn") or [G,N,K] (b_layout "nk", K-major,
    the dgrad layout), with S_B [kb,nb] / [G,kb,nb] / [G,nb,kb]."""

    a_codes: object
    a_scales: object
    b_codes: object
    b_scales: object
    b_layout: str = "kn"

    def validate(self, config: ProblemConfig) -> None:
        a = _codes(self.a_codes)
        b = _codes(self.b_codes)
        m, k, n, kb, nb, G = (config.m_total, config.k, config.n, config.k_blocks,
                              config.n_scale_blocks, config.groups)
        if tuple(a.shape) != (m, k):
            raise ShapeMismatch(f"A codes {tuple(a.shape)} != {(m, k)}")
        if tuple(self.a_scales.shape) != (m, kb):
            raise ShapeMismatch(f"A scales {tuple(self.a_scales.shape)}")
        if self.b_layout == "kn":
            ok_b = tuple(b.shape) in ((k, n), (G, k, n))
            ok_s = tuple(self.b_scales.shape) in ((kb, nb), (G, kb, nb))
        elif self.b_layout == "nk":
            ok_b = tuple(b.shape) == (G, n, k)
            ok_s = tuple(self.b_scales.shape) == (G, nb, kb)
        else:
            raise ConfigError(f"b_layout must be 'kn' or 'nk', got {self.b_layout!r}")
        if not ok_b:
            raise ShapeMismatch(f"B codes {tuple(b.shape)} do not match (k={k}, n={n}, G={G})")
        if not ok_s:
            raise ShapeMismatch(f"B scales {tuple(self.b_scales.shape)}")
        for s in (self.a_scales, self.b_scales):
            dt = s.dtype
            if dt not in (np.float32, torch.float32):
                raise ShapeMismatch("scales must be float32")

    @classmethod
    def from_dense(cls, a, b, *, device="cuda") -> "GroupedOperands":
        """engine.py:144-148: quantize dense A (1x128 tiles, fp8.py:132-151) and B (128x128
        blocks, fp8.py:154-176; [K,N] shared or [G,K,N] per expert) -- on the GPU
        (csrc/tagg_quant.cu, bit-identical to the reference), returning numpy codes and
        scales as the reference does.  Non-finite entries raise InvalidInput (fp8.py:54-80)."""
        from .quant import quantize_blocks, quantize_row_tiles

        at = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
        bt = b if isinstance(b, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(b, dtype=np.float32))
        ac, asc = quantize_row_tiles(at.to(device), check=True)
        bc, bsc = quantize_blocks(bt.to(device), check=True)
        return cls(ac.cpu().numpy(), asc.cpu().numpy(), bc.cpu().numpy(), bsc.cpu().numpy())


def _to_dev_u8(x, device):
    x = _codes(x)
    if isinstance(x, torch.Tensor):
        t = x
        if t.dtype == torch.float8_e4m3fn:
            t = t.view(torch.uint8)
    else:
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint8))
    return t.to(device, non_blocking=True).contiguous()


def _to_dev_f32(x, device):
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    return t.to(device=device, dtype=torch.float32, non_blocking=True).contiguous()


def _ptr(t):
    return None if t is None else t.data_ptr()


def grouped_gemm_fp8(a, a_scales, b, b_scales, group_sizes, *, b_layout="kn", out=None, c_row_offsets=None,
                     tile_map=None, exact_promotion=False, plain_staging=False, single_cta=False, tile=None,
                     stream=None, max_sms=None, pdl=True, pdl_overlap=False, err_flag=None, check=False,
                     b_index=None):
    """Padding-free FP8 grouped GEMM on device tensors (no host sync).

    a [m_alloc,K] uint8 / float8_e4m3fn; a_scales [m_alloc,ceil(K/128)] f32;
    b [K,N] or [G,K,N] (b_layout "kn") or [G,N,K] ("nk"); b_scales [kb,nb] /
    [G,kb,nb] / [G,nb,kb]; group_sizes int32 CUDA tensor [G] (sum <= m_alloc).
    Returns ``out`` (bf16 [c_rows, N]).  Only rows of valid group rows are
    written; with ``c_row_offsets`` (int64 CUDA [G]) group g's rows start at
    c_row_offsets[g].  ``tile`` picks the tile shape: "pair_n256" (CTA pair,
    256x256), "pair_n128" (CTA pair, 256x128), "1cta" (128x128) or None/"auto" (pair 256x256,
    or 1-CTA tiles when m_alloc <= 128 G: skinny, HBM-bound groups).

    ``b_index`` (int32 CUDA [G], optional): group g multiplies expert b_index[g] of B, so
    several groups may share one expert (an all-to-all's (source, expert) segments).

    Group sizes never reach the host, so the kernel validates them: a negative M_g or
    more rows than A / ``out`` hold makes the launch write nothing and OR-s a bit into
    ``err_flag`` (an int32 CUDA tensor [1]; ERR_NEGATIVE_SIZE / ERR_ROWS_OUT_OF_RANGE).
    ``check=True`` allocates the flag, synchronizes and raises ConfigError /
    ShapeMismatch like the reference (engine.py:77-92, 132-142).

    ``pdl`` (default on): programmatic dependent launch; the grid starts during the
    previous kernel's tail but reads its inputs only after that kernel completed.
    ``pdl_overlap=True`` asserts the previous kernel in the stream writes none of this
    call's inputs (e.g. a chain of independent GEMMs over resident operands): the main
    loop then overlaps it too, and only the stores wait (include/tagg.h).
    """
    if not (isinstance(a, torch.Tensor) and a.is_cuda):
        raise ValueError("grouped_gemm_fp8 expects CUDA tensors (no CPU fallback)")
    if a.dtype == torch.float8_e4m3fn:
        a = a.view(torch.uint8)
    if b.dtype == torch.float8_e4m3fn:
        b = b.view(torch.uint8)
    if a.dtype != torch.uint8 or b.dtype != torch.uint8:
        raise ShapeMismatch("A and B must be e4m3 codes (uint8 or float8_e4m3fn)")
    if a_scales.dtype != torch.float32 or b_scales.dtype != torch.float32:
        raise ShapeMismatch("scales must be float32")
    if group_sizes.dtype != torch.int32 or not group_sizes.is_cuda:
        raise ShapeMismatch("group_sizes must be an int32 CUDA tensor")
    m_alloc, K = a.shape
    G = group_sizes.numel()
    kb = num_blocks(K)
    if a.stride(1) != 1 or not a_scales.is_contiguous() or tuple(a_scales.shape) != (m_alloc, kb):
        raise ShapeMismatch(f"A scales must be a dense [m_alloc, {kb}] tensor")
    if b_layout == "kn":
        N = b.shape[-1]
        b_experts = 1 if b.dim() == 2 else b.shape[0]
        if tuple(b.shape[-2:]) != (K, N):
            raise ShapeMismatch(f"B {tuple(b.shape)} vs K={K}")
        nb = num_blocks(N)
        if tuple(b_scales.shape[-2:]) != (kb, nb):
            raise ShapeMismatch(f"B scales {tuple(b_scales.shape)}")
        sb_g = 0 if b_scales.dim() == 2 else b_scales.stride(0)
        sb_kb, sb_nb = b_scales.stride(-2), b_scales.stride(-1)
        layout = 0
    elif b_layout == "nk":
        N = b.shape[-2]
        b_experts = b.shape[0]
        if b.dim() != 3 or b.shape[2] != K:
            raise ShapeMismatch(f"B {tuple(b.shape)} vs K={K}")
        nb = num_blocks(N)
        if tuple(b_scales.shape) != (b_experts, nb, kb):
            raise ShapeMismatch(f"B scales {tuple(b_scales.shape)}")
        sb_g, sb_nb, sb_kb = b_scales.stride(0), b_scales.stride(1), b_scales.stride(2)
        layout = 1
    else:
        raise ConfigError(f"b_layout must be 'kn' or 'nk', got {b_layout!r}")
    if not b.is_contiguous():
        raise ShapeMismatch("B must be contiguous")
    if b_index is not None:
        if b_index.dtype != torch.int32 or not b_index.is_cuda or b_index.numel() != G:
            raise ShapeMismatch(f"b_index must be an int32 CUDA tensor of {G} entries")
        b_index = b_index.contiguous()
    elif b_experts not in (1, G):
        raise ShapeMismatch(f"B holds {b_experts} experts for {G} groups (give b_index)")
    if out is None:
        out = torch.empty((m_alloc, N), dtype=torch.bfloat16, device=a.device)
    if out.dtype not in (torch.bfloat16, torch.uint16, torch.int16) or out.stride(1) != 1 or out.dim() != 2:
        raise ShapeMismatch("out must be a row-major bf16 [c_rows, N] tensor")
    if out.shape[1] != N:
        raise ShapeMismatch(f"out has {out.shape[1]} columns, the problem has N={N}")
    if out.device != a.device:
        raise ShapeMismatch("out must be on the same device as A")
    if c_row_offsets is not None and (c_row_offsets.dtype != torch.int64 or not c_row_offsets.is_cuda):
        raise ShapeMismatch("c_row_offsets must be an int64 CUDA tensor")
    flags = ((FLAG_EXACT_PROMOTION if exact_promotion else 0) | (FLAG_PLAIN_C_STAGING if plain_staging else 0)
             | (FLAG_SINGLE_CTA if single_cta else 0) | TILES[tile] | (0 if pdl else FLAG_SERIAL)
             | (FLAG_PDL_OVERLAP if pdl_overlap else 0))
    if max_sms:
        if not 0 < int(max_sms) < 4096:
            raise ConfigError(f"max_sms must be in [1, 4095], got {max_sms}")
        flags |= int(max_sms) << SM_LIMIT_SHIFT
    st = stream if stream is not None else torch.cuda.current_stream(a.device)
    if check and err_flag is None:
        err_flag = torch.zeros(1, dtype=torch.int32, device=a.device)
    if err_flag is not None and (err_flag.dtype != torch.int32 or not err_flag.is_cuda):
        raise ShapeMismatch("err_flag must be an int32 CUDA tensor")
    rc = lib().tagg_grouped_gemm_fp8_ex(
        _ptr(a), a.stride(0), _ptr(a_scales), m_alloc, _ptr(b), layout, b_experts, _ptr(b_scales),
        sb_g, sb_kb, sb_nb, _ptr(group_sizes), G, N, K, _ptr(out), out.stride(0), out.shape[0],
        _ptr(c_row_offsets), _ptr(tile_map), _ptr(b_index), _ptr(err_flag), flags, st.cuda_stream)
    raise_for_status(rc, "tagg_grouped_gemm_fp8")
    if check:
        raise_for_device_flag(int(err_flag.item()), "tagg_grouped_gemm_fp8")
    return out


def raise_for_device_flag(bits: int, what: str) -> None:
    """The kernel's device-side validation of the group sizes (tagg_grouped_gemm_fp8_checked)."""
    if bits & ERR_NEGATIVE_SIZE:
        raise ConfigError(f"{what}: group sizes must be non-negative")
    if bits & ERR_ROWS_OUT_OF_RANGE:
        raise ShapeMismatch(f"{what}: sum of group sizes exceeds the rows of A / out")
    if bits & ERR_B_INDEX:
        raise ShapeMismatch(f"{what}: b_index names an expert outside B")


def max_tiles(m_alloc: int, groups: int, n: int) -> int:
    return int(lib().tagg_max_tiles(int(m_alloc), int(groups), int(n)))


class PaddedWorkspace:
    """Buffers of the pad + padded-GEMM baseline, allocated once (sizes need no host sync)."""

    def __init__(self, m_alloc: int, groups: int, k: int, n: int, device):
        rows = int(lib().tagg_padded_rows_bound(int(m_alloc), int(groups)))
        self.rows = rows
        self.a_pad = torch.empty((rows, k), dtype=torch.uint8, device=device)
        self.sa_pad = torch.empty((rows, num_blocks(k)), dtype=torch.float32, device=device)
        self.c_pad = torch.empty((rows, n), dtype=torch.bfloat16, device=device)
        self.padded_sizes = torch.empty((groups,), dtype=torch.int32, device=device)

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.a_pad, self.sa_pad, self.c_pad, self.padded_sizes))


def pad_groups(a, a_scales, group_sizes, ws: PaddedWorkspace, stream=None):
    """Baseline K2 (engine.py:369-373) on device."""
    if a.dtype == torch.float8_e4m3fn:
        a = a.view(torch.uint8)
    st = stream if stream is not None else torch.cuda.current_stream(a.device)
    rc = lib().tagg_pad_groups(_ptr(a), a.stride(0), _ptr(a_scales), _ptr(group_sizes), group_sizes.numel(),
                               a.shape[1], _ptr(ws.a_pad), _ptr(ws.sa_pad), _ptr(ws.padded_sizes), ws.rows,
                               st.cuda_stream)
    raise_for_status(rc, "tagg_pad_groups")


def unpad_rows(c_pad, group_sizes, out, stream=None):
    """Baseline K3 (engine.py:399-401) on device."""
    st = stream if stream is not None else torch.cuda.current_stream(out.device)
    rc = lib().tagg_unpad_rows(_ptr(c_pad), _ptr(group_sizes), group_sizes.numel(), out.shape[1], _ptr(out),
                               out.shape[0], st.cuda_stream)
    raise_for_status(rc, "tagg_unpad_rows")


def padded_grouped_gemm_fp8(a, a_scales, b, b_scales, group_sizes, ws: PaddedWorkspace, *, b_layout="kn",
                            out=None, unpad=True, stream=None, **kw):
    """The pad-to-128 + padded grouped GEMM baseline on the same GPU.

    K2 pads every group to a multiple of 128 rows (A rows 0, S_A rows 1.0).
    The same kernel then runs on the 128-aligned groups, so every store is a
    full-height store.  K3 optionally gathers the valid rows.  This is
    engine.py:346-402's data path.
    """
    kw.pop("pdl_overlap", None)  # the pad kernel right before writes this GEMM's inputs
    pad_groups(a, a_scales, group_sizes, ws, stream)
    grouped_gemm_fp8(ws.a_pad, ws.sa_pad, b, b_scales, ws.padded_sizes, b_layout=b_layout, out=ws.c_pad,
                     stream=stream, **kw)
    if not unpad:
        return ws.c_pad
    if out is None:
        out = torch.empty((a.shape[0], ws.c_pad.shape[1]), dtype=torch.bfloat16, device=a.device)
    unpad_rows(ws.c_pad, group_sizes, out, stream)
    return out


@dataclass
class AdaptiveRun:
    """engine.py:172-177.  ``engine`` (the simulated transfer log) is replaced by
    ``tile_map``, the store geometry the kernel actually used, one row per tile:
    (group, m_tile, n0, a_row0, valid, desc_rows, phaseA_row, phaseB_smem_row, phaseB_row)."""

    c_bits: np.ndarray
    plans: list
    pools: dict = field(default_factory=dict)
    tile_map: np.ndarray | None = None
    c: torch.Tensor | None = None


def _device_operands(config: ProblemConfig, operands: GroupedOperands, device):
    operands.validate(config)
    a = _to_dev_u8(operands.a_codes, device)
    sa = _to_dev_f32(operands.a_scales, device)
    b = _to_dev_u8(operands.b_codes, device)
    sb = _to_dev_f32(operands.b_scales, device)
    gs = torch.tensor(config.group_sizes, dtype=torch.int32, device=device)
    return a, sa, b, sb, gs


def run_adaptive(config: ProblemConfig, operands: GroupedOperands, *, poison: int = 0xA5,
                 device="cuda", exact_promotion=False, plain_staging=False, single_cta=False,
                 tile=None) -> AdaptiveRun:
    """engine.py:184-343 on the GPU: one launch of the padding-free kernel.

    C is pre-filled with the ``poison`` byte pattern before the launch, so any
    row the store plan failed to cover would show up in ``c_bits``.  This is
    the role the reference's arena poison plays.
    """
    a, sa, b, sb, gs = _device_operands(config, operands, device)
    m, n = config.m_total, config.n
    pv = (int(poison) & 0xFF) * 0x0101
    c = torch.full((m, n), pv - 65536 if pv >= 32768 else pv, dtype=torch.int16, device=device)
    tmap = None
    if m:
        tmap = torch.full((max_tiles(m, config.groups, n), TILE_MAP_FIELDS), -1, dtype=torch.int32, device=device)
        grouped_gemm_fp8(a, sa, b, sb, gs, b_layout=operands.b_layout, out=c, tile_map=tmap,
                         exact_promotion=exact_promotion, plain_staging=plain_staging, single_cta=single_cta,
                         tile=tile)
    c_bits = c.cpu().numpy().view(np.uint16) if m else np.zeros((0, n), dtype=np.uint16)
    tm = None
    if tmap is not None:
        tm = tmap.cpu().numpy()
        tm = tm[tm[:, 0] >= 0]
    plans = planning.plan_group_stores(config.group_sizes, config.block_m)
    pools = {w: planning.build_pool(config.block_m) for _, w in config.n_tiles()}
    return AdaptiveRun(c_bits=c_bits, plans=plans, pools=pools, tile_map=tm, c=c.view(torch.bfloat16))


def run_padded_baseline(config: ProblemConfig, operands: GroupedOperands, *, device="cuda",
                        exact_promotion=False) -> np.ndarray:
    """engine.py:346-402 on the GPU: pad kernel + the same GEMM + unpad kernel."""
    a, sa, b, sb, gs = _device_operands(config, operands, device)
    m, n = config.m_total, config.n
    if m == 0:
        return np.zeros((0, n), dtype=np.uint16)
    ws = PaddedWorkspace(m, config.groups, config.k, n, device)
    out = padded_grouped_gemm_fp8(a, sa, b, sb, gs, ws, b_layout=operands.b_layout,
                                  exact_promotion=exact_promotion)
    return out.view(torch.int16).cpu().numpy().view(np.uint16).copy()


@dataclass(frozen=True)
class BitwiseReport:
    """engine.py:405-412"""

    equal: bool
    mismatches: int
    first: tuple | None

    def __bool__(self) -> bool:
        return self.equal


def verify_bitwise(got_bits: np.ndarray, want_bits: np.ndarray) -> BitwiseReport:
    """engine.py:415-423"""
    if got_bits.shape != want_bits.shape:
        raise ShapeMismatch(f"{got_bits.shape} vs {want_bits.shape}")
    diff = got_bits != want_bits
    count = int(diff.sum())
    if count == 0:
        return BitwiseReport(True, 0, None)
    first = np.argwhere(diff)[0]
    return BitwiseReport(False, count, (int(first[0]), int(first[1])))
