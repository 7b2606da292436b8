"""CPU ORACLE for FP8 numerics and the input recipe (test infrastructure).

A numpy restatement of the reference's e4m3 codec and quantizers
(/root/reference/pkg/src/tma_sim/fp8.py).  Tests use it to build operands
with the reference's recipe (cli.py:112-121) at sizes the reference never
shipped as fixtures.  The product path never imports it.
"""

from __future__ import annotations

import numpy as np

E4M3_MAX = 448.0          # fp8.py:29
NAN_CODES = (0x7F, 0xFF)  # fp8.py:30
SCALE_BLOCK = 128         # fp8.py:31


def _build_decode_table() -> np.ndarray:
    """fp8.py:34-46"""
    codes = np.arange(256)
    sign = np.where(codes >> 7, -1.0, 1.0)
    e = (codes >> 3) & 0xF
    m = (codes & 0x7).astype(np.float64)
    vals = sign * np.where(e == 0, np.ldexp(m / 8.0, -6), np.ldexp(1.0 + m / 8.0, e - 7))
    vals[list(NAN_CODES)] = np.nan
    return vals.astype(np.float32)


DECODE_TABLE = _build_decode_table()


def encode(values) -> np.ndarray:
    """fp8.py:54-80: RNE, saturating at +-448, never emits NaN."""
    x = np.asarray(values, dtype=np.float32)
    if not np.all(np.isfinite(x)):
        raise ValueError("cannot encode non-finite values")
    sign = np.signbit(x)
    mag = np.minimum(np.abs(x.astype(np.float64)), E4M3_MAX)
    _, e2 = np.frexp(mag)
    e = np.maximum(e2 - 1, -6)
    q = np.rint(mag * np.exp2(3.0 - e)).astype(np.int64)
    carry = q >= 16
    e = e + carry
    q = np.where(carry, 8, q)
    exp_field = np.where(q >= 8, e + 7, 0)
    mant = np.where(q >= 8, q - 8, q)
    return ((sign.astype(np.int64) << 7) | (exp_field << 3) | mant).astype(np.uint8)


def quantize_row_tiles(x):
    """fp8.py:132-151: one f32 scale per 1x128 row tile -> (codes, scales[rows, kb])."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    rows, cols = x.shape
    tiles = -(-cols // SCALE_BLOCK)
    codes = np.empty((rows, cols), dtype=np.uint8)
    scales = np.empty((rows, tiles), dtype=np.float32)
    for t in range(tiles):
        sl = slice(t * SCALE_BLOCK, min((t + 1) * SCALE_BLOCK, cols))
        amax = np.abs(x[:, sl]).max(axis=1) if rows else np.zeros(0, np.float32)
        s = np.where(amax > 0, amax / np.float32(E4M3_MAX), np.float32(1.0)).astype(np.float32)
        scales[:, t] = s
        codes[:, sl] = encode(x[:, sl] / s[:, None])
    return codes, scales


def quantize_blocks(x):
    """fp8.py:154-176: one f32 scale per 128x128 block -> (codes, scales[rb, cb])."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    rows, cols = x.shape
    rb, cb = -(-rows // SCALE_BLOCK), -(-cols // SCALE_BLOCK)
    codes = np.empty((rows, cols), dtype=np.uint8)
    scales = np.empty((rb, cb), dtype=np.float32)
    for i in range(rb):
        rsl = slice(i * SCALE_BLOCK, min((i + 1) * SCALE_BLOCK, rows))
        for j in range(cb):
            csl = slice(j * SCALE_BLOCK, min((j + 1) * SCALE_BLOCK, cols))
            block = x[rsl, csl]
            amax = np.abs(block).max()
            s = np.float32(amax / np.float32(E4M3_MAX)) if amax > 0 else np.float32(1.0)
            scales[i, j] = s
            codes[rsl, csl] = encode(block / s)
    return codes, scales


def random_operands(m: int, n: int, k: int, seed: int):
    """cli.py:112-121 input recipe -> (a_codes, a_scales, b_codes[K,N], b_scales[kb,nb])."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence((seed, 0xA11CE))))
    a = rng.standard_normal((m, k), dtype=np.float32)
    a *= np.exp2(rng.integers(-4, 5, size=(m, 1)).astype(np.float32))
    b = rng.standard_normal((k, n), dtype=np.float32)
    b *= np.exp2(rng.integers(-2, 3, size=(1, n)).astype(np.float32))
    ac, asc = quantize_row_tiles(a)
    bc, bsc = quantize_blocks(b)
    return ac, asc, bc, bsc


def bf16_bits_to_f32(bits) -> np.ndarray:
    """engine.py:53-55"""
    u = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return u.view(np.float32)


def pow2_ceil(s):
    """The smallest power of two >= s (fp32, s > 0; at least 2^-126): the UE8M0-representable
    scale of the MXFP8 weight-gradient recipe (quantize_col_blocks(..., scale_pow2=True))."""
    b = np.asarray(s, dtype=np.float32).view(np.uint32).copy()
    up = (b & 0x7FFFFF) != 0
    b = np.where(up, (b & 0xFF800000) + 0x800000, b).astype(np.uint32)
    b = np.maximum(b, np.uint32(0x00800000))
    return b.view(np.float32)


def quantize_col_blocks(x, group_sizes, block_cols: int = 1, scale_pow2: bool = False):
    """Per-group 128x1 quantization for the weight gradient (the ragged token axis is the
    reduction axis): for each group and each of its 128-token blocks, one scale per
    column, s = fl(amax / 448) (1.0 when zero), codes = encode(fl(x / s)) -- the
    fp8.py:132-151 recipe applied down the columns of each block.  Returns
    (codes [M, C], scales [TB, C]) with TB = sum(ceil(M_g / 128)) rows, group by group.
    block_cols = 128: one scale per (token block, 128 columns), the 128x128 block recipe of
    fp8.py:154-176 (quantize_blocks) applied per group token block, repeated in each of the
    block's 128 column slots.
    scale_pow2: s = pow2_ceil(fl(amax / 448)) (1.0 when zero), a power of two, so x / s is exact
    and s is one E8M0 byte -- the MXFP8 recipe the block-scaled weight gradient takes.
    """
    x = np.ascontiguousarray(x, dtype=np.float32)
    rows, cols = x.shape
    codes = np.empty((rows, cols), dtype=np.uint8)
    blocks = []
    off = 0
    for m in group_sizes:
        m = int(m)
        for b0 in range(0, m, SCALE_BLOCK):
            sl = slice(off + b0, off + min(b0 + SCALE_BLOCK, m))
            amax = np.abs(x[sl]).max(axis=0)
            if block_cols == 128:
                amax = np.repeat(amax.reshape(-1, 128).max(axis=1), 128)
            s = np.where(amax > 0, amax / np.float32(E4M3_MAX), np.float32(1.0)).astype(np.float32)
            if scale_pow2:
                s = np.where(amax > 0, pow2_ceil(s), np.float32(1.0)).astype(np.float32)
            blocks.append(s)
            codes[sl] = encode(x[sl] / s[None, :])
        off += m
    scales = np.stack(blocks) if blocks else np.zeros((0, cols), np.float32)
    return codes, scales
