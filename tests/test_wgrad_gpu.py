"""Weight gradient as a K-grouped FP8 GEMM (csrc/tagg_wgrad.cu) against the oracle.

The ragged per-expert row count is the reduction axis: every residue M_g mod 128
(dual-phase pool loads + zeroed tail rows), empty groups, and the per-(group, token
block, column) quantizer (bit-exact vs oracle/fp8.quantize_col_blocks).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2508_16584_b200 as tg
from helpers import assert_parity
from oracle import fp8 as ofp8
from oracle import oracle as orc

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def _data(sizes, k, n, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    m = sum(sizes)
    x = rng.standard_normal((m, k)).astype(np.float32) * np.exp2(rng.integers(-3, 4, size=(m, 1))).astype(np.float32)
    dy = rng.standard_normal((m, n)).astype(np.float32) * np.exp2(rng.integers(-3, 4, size=(m, 1))).astype(np.float32)
    return x, dy


@pytest.mark.parametrize("sizes", [(200,), (1, 0, 129, 255, 384), tuple(128 * (g % 3) + (g * 37) % 128 + 1 for g in range(8))])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_quantize_col_blocks_is_bit_exact(sizes, dtype):
    x, _ = _data(sizes, 384, 128, 1)
    xt = torch.from_numpy(x).to(DEV).to(dtype)
    gs = torch.tensor(sizes, dtype=torch.int32, device=DEV)
    codes, scales = tg.quantize_col_blocks(xt, gs, check=True)
    torch.cuda.synchronize()
    want_c, want_s = ofp8.quantize_col_blocks(xt.float().cpu().numpy(), sizes)
    np.testing.assert_array_equal(codes.cpu().numpy(), want_c)
    tb = want_s.shape[0]
    np.testing.assert_array_equal(scales[:tb].cpu().numpy().view(np.uint32), want_s.view(np.uint32))


def _midpoint_inputs(seed):
    """Rows fl(M * s_j) for every e4m3 rounding midpoint M (and 1-3 fp32 ulp either side), with
    a planted column maximum A_j in the first row of each 128-row block, so s_j = fl(A_j / 448)
    and the quotient x / s_j lands on (or next to) a midpoint."""
    rng = np.random.Generator(np.random.PCG64(seed))
    vals = np.unique(np.abs(ofp8.DECODE_TABLE[np.isfinite(ofp8.DECODE_TABLE)]).astype(np.float64))
    mids = ((vals[:-1] + vals[1:]) / 2).astype(np.float32)
    ms = [mids]
    for d in (1, 2, 3):
        up, dn = mids.copy(), mids.copy()
        for _ in range(d):
            up = np.nextafter(up, np.float32(np.inf))
            dn = np.nextafter(dn, np.float32(0))
        ms += [up, dn]
    m_all = np.concatenate(ms)
    m_all = m_all[rng.permutation(m_all.size)]
    cols = 256
    amax = np.exp2(rng.uniform(-12, 12, size=cols)).astype(np.float32)
    s = (amax / np.float32(448.0)).astype(np.float32)
    rows = []
    for b0 in range(0, m_all.size, 127):
        blk = m_all[b0:b0 + 127]
        sign = np.where(rng.random((blk.size, cols)) < 0.5, np.float32(-1), np.float32(1))
        rows.append(amax[None, :])
        rows.append((blk[:, None] * s[None, :] * sign).astype(np.float32))
    return np.concatenate(rows).astype(np.float32)


@pytest.mark.parametrize("block_cols", [1, 128])
def test_quantize_col_blocks_quotients_at_e4m3_midpoints(block_cols):
    """The kernel decides each code from q = x * RN(1/s) and hands the quotients that sit near
    an e4m3 rounding midpoint (or in the e4m3 subnormal range) to the IEEE division: inputs whose
    x / s land on every midpoint and 1-3 ulp around it, bit-exact against the oracle's fp32
    division (fp8.py:54-80)."""
    x = _midpoint_inputs(5)
    m = x.shape[0]
    sizes = (128 * (m // 256), m - 128 * (m // 256))
    gs = torch.tensor(sizes, dtype=torch.int32, device=DEV)
    codes, scales = tg.quantize_col_blocks(torch.from_numpy(x).to(DEV), gs, check=True, block_cols=block_cols)
    torch.cuda.synchronize()
    want_c, want_s = ofp8.quantize_col_blocks(x, sizes, block_cols=block_cols)
    np.testing.assert_array_equal(codes.cpu().numpy(), want_c)
    np.testing.assert_array_equal(scales[:want_s.shape[0]].cpu().numpy().view(np.uint32), want_s.view(np.uint32))


@pytest.mark.parametrize("sizes,k,n", [
    ((128,), 128, 128),
    ((300, 0, 1, 77, 256), 256, 384),
    (tuple(range(1, 128, 9)), 128, 256),       # every residue class, ragged reduction
    ((1000, 513), 384, 256),
])
def test_wgrad_matches_oracle(sizes, k, n):
    x, dy = _data(sizes, k, n, sum(sizes))
    gs = torch.tensor(sizes, dtype=torch.int32, device=DEV)
    xc, xs = tg.quantize_col_blocks(torch.from_numpy(x).to(DEV), gs)
    dc, ds = tg.quantize_col_blocks(torch.from_numpy(dy).to(DEV), gs)
    dw = tg.wgrad_fp8(xc, xs, dc, ds, gs)
    torch.cuda.synchronize()
    tb = sum(-(-s // 128) for s in sizes)
    want = orc.wgrad(xc.cpu().numpy(), xs[:tb].cpu().numpy(), dc.cpu().numpy(), ds[:tb].cpu().numpy(), sizes,
                     threads=8)
    got = dw.view(torch.int16).cpu().numpy().view(np.uint16)
    for g, m in enumerate(sizes):
        if m == 0:
            assert np.all(got[g] == 0), "an empty group's gradient is zero"
        else:
            assert_parity(got[g], want[g], label=f"group {g} (M_g={m})")


@pytest.mark.parametrize("sizes,k,n", [
    ((300, 0, 1, 77, 256), 256, 384),
    (tuple(range(1, 128, 9)), 128, 256),
    ((1000, 513), 384, 256),
])
def test_wgrad_dy_block128_matches_oracle(sizes, k, n):
    """TAGG_WGRAD_DY_BLOCK128: dY quantized with one scale per (token block, 128 columns) (the
    128x128 block recipe, fp8.py:154-176, per group token block); the kernel promotes with
    s = fl(sx * sdy) once per block and one FFMA2 per pair.  Same oracle, same tolerance."""
    x, dy = _data(sizes, k, n, 3 * sum(sizes))
    gs = torch.tensor(sizes, dtype=torch.int32, device=DEV)
    xc, xs = tg.quantize_col_blocks(torch.from_numpy(x).to(DEV), gs)
    dc, ds = tg.quantize_col_blocks(torch.from_numpy(dy).to(DEV), gs, block_cols=128)
    dw = tg.wgrad_fp8(xc, xs, dc, ds, gs, dy_block128=True)
    torch.cuda.synchronize()
    tb = sum(-(-s // 128) for s in sizes)
    dsn = ds[:tb].cpu().numpy()
    assert np.all(dsn.reshape(tb, n // 128, 128) == dsn.reshape(tb, n // 128, 128)[:, :, :1])
    want = orc.wgrad(xc.cpu().numpy(), xs[:tb].cpu().numpy(), dc.cpu().numpy(), dsn, sizes, threads=8)
    got = dw.view(torch.int16).cpu().numpy().view(np.uint16)
    for g, m in enumerate(sizes):
        if m == 0:
            assert np.all(got[g] == 0), "an empty group's gradient is zero"
        else:
            assert_parity(got[g], want[g], label=f"group {g} (M_g={m})")


def test_wgrad_never_reads_the_next_group():
    """Poison the rows after a short group: its gradient must not change."""
    sizes = (70, 300)
    k, n = 128, 128
    x, dy = _data(sizes, k, n, 5)
    gs = torch.tensor(sizes, dtype=torch.int32, device=DEV)
    xc, xs = tg.quantize_col_blocks(torch.from_numpy(x).to(DEV), gs)
    dc, ds = tg.quantize_col_blocks(torch.from_numpy(dy).to(DEV), gs)
    base = tg.wgrad_fp8(xc, xs, dc, ds, gs)[0].clone()
    xc2, dc2 = xc.clone(), dc.clone()
    xc2[70:198] = 0x7E  # large codes in the rows a full 128-row box would have read
    dc2[70:198] = 0x7E
    again = tg.wgrad_fp8(xc2, xs, dc2, ds, gs)[0]
    torch.cuda.synchronize()
    assert torch.equal(base.view(torch.int16), again.view(torch.int16))


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_col_block_gather_equals_quantizing_the_gathered_copy(dtype):
    """quantize_col_blocks(x, index=, row_weights=) is bit-identical to quantizing the gathered,
    scaled copy fl(w[r] * x[index[r]])."""
    torch.manual_seed(4)
    t, c = 150, 256
    sizes = (130, 0, 77, 1)
    x = (torch.randn((t, c), device=DEV) * 3).to(dtype)
    idx = torch.randint(0, t, (sum(sizes),), device=DEV, dtype=torch.int32)
    w = torch.rand(sum(sizes), device=DEV)
    gs = torch.tensor(sizes, dtype=torch.int32, device=DEV)
    got_c, got_s = tg.quantize_col_blocks(x, gs, index=idx, row_weights=w)
    copy = (x.float().index_select(0, idx.long()) * w[:, None])
    want_c, want_s = tg.quantize_col_blocks(copy, gs)
    tb = sum(-(-s // 128) for s in sizes)
    assert torch.equal(got_c, want_c)
    assert torch.equal(got_s[:tb], want_s[:tb])
    plain_c, plain_s = tg.quantize_col_blocks(x, gs, index=idx)
    want_pc, want_ps = tg.quantize_col_blocks(x.index_select(0, idx.long()).contiguous(), gs)
    assert torch.equal(plain_c, want_pc) and torch.equal(plain_s[:tb], want_ps[:tb])


_SPECIAL_BITS = {  # bit patterns: (bf16 as int16, f32 as int32)
    "+inf": (0x7F80, 0x7F800000), "-inf": (-0x0080, -0x00800000),
    "+nan": (0x7FC0, 0x7FC00000), "-nan": (-0x0040, -0x00400000),
}


@pytest.mark.parametrize("special", sorted(_SPECIAL_BITS))
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("path", ["per_column", "block128", "gather", "mxfp8"])
def test_quantize_col_blocks_flags_non_finite(special, dtype, path):
    """Every column-block quantizer path flags an inf / NaN of either sign in a live row (the
    reference raises InvalidInput, fp8.py:54-80); the same matrix with the value made finite
    passes.  A negative NaN is the case the packed-bf16 |x| maximum reaches through its unsigned
    half, a positive one through its signed half."""
    torch.manual_seed(9)
    sizes = (130, 0, 77)
    m, c = sum(sizes), 256
    x = torch.randn((m, c), device=DEV).to(dtype)
    gs = torch.tensor(sizes, dtype=torch.int32, device=DEV)
    idx = torch.arange(m, device=DEV, dtype=torch.int32).flip(0)

    def run(t):
        if path == "mxfp8":
            return tg.quantize_col_blocks_mx(t, gs, check=True)
        if path == "gather":
            return tg.quantize_col_blocks(t, gs, check=True, index=idx)
        return tg.quantize_col_blocks(t, gs, check=True, block_cols=128 if path == "block128" else 1)

    run(x)
    bits = _SPECIAL_BITS[special][0 if dtype == torch.bfloat16 else 1]
    for r, col in ((0, 0), (129, 255), (m - 1, 131)):
        y = x.clone()
        y.view(torch.int16 if dtype == torch.bfloat16 else torch.int32)[r, col] = bits
        with pytest.raises(tg.InvalidInput):
            run(y)


def _sf_blocks(scales):
    """The E8M0 factor blocks tagg_quantize_col_blocks_mx lays out: per (token block, 128
    columns) byte 16 l + 4 c + j = the exponent byte of column 32 c + l's scale (j = 0..3)."""
    tb, cols = scales.shape
    e = ((scales.view(np.uint32) >> 23) & 0xFF).astype(np.uint8).reshape(tb, cols // 128, 4, 32)  # [tb, blk, c, l]
    return np.repeat(e.transpose(0, 1, 3, 2)[..., None], 4, axis=-1).reshape(tb, cols // 128, 512)


@pytest.mark.parametrize("sizes", [(200,), (1, 0, 129, 255, 384)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("gather", [False, True])
def test_quantize_col_blocks_mx_is_bit_exact(sizes, dtype, gather):
    """The MXFP8 recipe: s = pow2_ceil(fl(amax / 448)), codes = e4m3(x / s) with an exact
    quotient -- bit-exact against oracle/fp8.quantize_col_blocks(..., scale_pow2=True) --, every
    scale a power of two, and the E8M0 factor blocks in the tcgen05.cp source layout.  The
    plain entry point with scale_pow2 gives the same codes and scales."""
    x, _ = _data(sizes, 256, 128, 11)
    m = sum(sizes)
    xt = torch.from_numpy(x).to(DEV).to(dtype)
    gs = torch.tensor(sizes, dtype=torch.int32, device=DEV)
    perm = torch.randperm(m, generator=torch.Generator().manual_seed(3)).to(DEV) if gather else None
    codes, scales, sf = tg.quantize_col_blocks_mx(xt, gs, check=True, index=perm)
    codes2, scales2 = tg.quantize_col_blocks(xt, gs, index=perm, scale_pow2=True)
    torch.cuda.synchronize()
    ref_x = xt.float()[perm].cpu().numpy() if gather else xt.float().cpu().numpy()
    want_c, want_s = ofp8.quantize_col_blocks(ref_x, sizes, scale_pow2=True)
    tb = want_s.shape[0]
    np.testing.assert_array_equal(codes.cpu().numpy(), want_c)
    got_s = scales[:tb].cpu().numpy()
    np.testing.assert_array_equal(got_s.view(np.uint32), want_s.view(np.uint32))
    assert np.all((got_s.view(np.uint32) & 0x7FFFFF) == 0), "every scale is a power of two"
    np.testing.assert_array_equal(sf[:tb].cpu().numpy(), _sf_blocks(want_s))
    np.testing.assert_array_equal(codes2.cpu().numpy(), want_c)
    np.testing.assert_array_equal(scales2[:tb].cpu().numpy().view(np.uint32), want_s.view(np.uint32))


@pytest.mark.parametrize("sizes,k,n", [
    ((128,), 128, 128),
    ((300, 0, 1, 77, 256), 256, 384),
    (tuple(range(1, 128, 9)), 128, 256),       # every residue class, ragged reduction
    ((1000, 513), 384, 256),
    ((0, 0, 700), 256, 256),                   # leading empty groups: their tiles store zeros
])
def test_wgrad_mx_matches_oracle(sizes, k, n):
    """wgrad_fp8_mx: power-of-two scales applied by the tensor core as E8M0 block scales
    (kind::mxf8f6f4.block_scale) with each tile's whole token range accumulated in TMEM, against
    the C oracle (per-block promotion in fp32) on the same operands: the same real sum, rounded
    differently in fp32, so within the bf16 tolerance."""
    x, dy = _data(sizes, k, n, sum(sizes) + 9)
    gs = torch.tensor(sizes, dtype=torch.int32, device=DEV)
    xc, xs, xf = tg.quantize_col_blocks_mx(torch.from_numpy(x).to(DEV), gs)
    dc, ds, df = tg.quantize_col_blocks_mx(torch.from_numpy(dy).to(DEV), gs)
    dw = tg.wgrad_fp8_mx(xc, xf, dc, df, gs)
    torch.cuda.synchronize()
    tb = sum(-(-s // 128) for s in sizes)
    want = orc.wgrad(xc.cpu().numpy(), xs[:tb].cpu().numpy(), dc.cpu().numpy(), ds[:tb].cpu().numpy(), sizes,
                     threads=8)
    got = dw.view(torch.int16).cpu().numpy().view(np.uint16)
    for g, m in enumerate(sizes):
        if m == 0:
            assert np.all(got[g] == 0), "an empty group's gradient is zero"
        else:
            assert_parity(got[g], want[g], label=f"mx group {g} (M_g={m})")


def test_wgrad_mx_never_reads_the_next_group():
    """MXFP8 path: poisoning the rows after a short group leaves its gradient unchanged."""
    sizes = (70, 300)
    k, n = 128, 256
    x, dy = _data(sizes, k, n, 6)
    gs = torch.tensor(sizes, dtype=torch.int32, device=DEV)
    xc, _, xf = tg.quantize_col_blocks_mx(torch.from_numpy(x).to(DEV), gs)
    dc, _, df = tg.quantize_col_blocks_mx(torch.from_numpy(dy).to(DEV), gs)
    base = tg.wgrad_fp8_mx(xc, xf, dc, df, gs)[0].clone()
    xc2, dc2 = xc.clone(), dc.clone()
    xc2[70:198] = 0x7E
    dc2[70:198] = 0x7E
    again = tg.wgrad_fp8_mx(xc2, xf, dc2, df, gs)[0]
    torch.cuda.synchronize()
    assert torch.equal(base.view(torch.int16), again.view(torch.int16))
