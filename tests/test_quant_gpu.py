"""Fused 1x128 quantize + dispatch permutation (csrc/tagg_quant.cu) against the oracle.

The codes and scales must equal the reference quantizer bit for bit
(quantize_row_tiles fp8.py:132-151, encode fp8.py:54-80, restated in
oracle/fp8.py), the route plan must equal a stable sort by expert, and the
dispatched rows must feed the grouped GEMM to the oracle's result.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2508_16584_b200 as tg
from helpers import assert_parity, oracle_c, per_expert_operands
from oracle import fp8 as ofp8

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def _reference_rows(rows, k, seed):
    """The reference's activation recipe: N(0,1) * 2^U{-4..4} per row (cli.py:112-121)."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence((seed, 0xA11CE))))
    x = rng.standard_normal((rows, k)).astype(np.float32)
    x *= np.exp2(rng.integers(-4, 5, size=(rows, 1))).astype(np.float32)
    return x


def _edge_rows(k):
    """Zero rows (scale 1.0), -0.0, subnormal-range quotients, a saturating tie, a lone spike."""
    x = np.zeros((6, k), np.float32)
    x[1, :] = -0.0
    x[2, :] = np.float32(1e-30) * np.arange(1, k + 1, dtype=np.float32)
    x[3, :] = 448.0
    x[3, ::7] = -464.0
    x[4, 0] = 3.0e38
    x[4, 1:] = 1.0
    x[5, :] = np.float32(2.0 ** -20)
    x[5, ::3] = np.float32(-2.0 ** -12)
    return x


@pytest.mark.parametrize("k", [1, 100, 128, 200, 512, 7168])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_quantize_row_tiles_is_bit_exact(k, dtype):
    x = np.concatenate([_reference_rows(37, k, k), _edge_rows(k)])
    xt = torch.from_numpy(x).to(DEV).to(dtype)
    codes, scales = tg.quantize_row_tiles(xt)
    torch.cuda.synchronize()
    want_c, want_s = ofp8.quantize_row_tiles(xt.float().cpu().numpy())
    np.testing.assert_array_equal(codes.cpu().numpy(), want_c)
    np.testing.assert_array_equal(scales.cpu().numpy().view(np.uint32), want_s.view(np.uint32))


def test_quantize_rejects_non_finite_when_checked():
    x = torch.ones((4, 256), device=DEV)
    x[2, 17] = float("nan")
    with pytest.raises(tg.InvalidInput):
        tg.quantize_row_tiles(x, check=True)
    x[2, 17] = float("inf")
    with pytest.raises(tg.InvalidInput):
        tg.quantize_row_tiles(x, check=True)


@pytest.mark.parametrize("rows,experts", [(0, 8), (1, 1), (1000, 7), (5000, 256), (70000, 64)])
def test_route_plan_is_a_stable_sort_by_expert(rows, experts):
    g = torch.Generator(device="cpu").manual_seed(rows + experts)
    ids = torch.randint(0, experts, (rows,), generator=g, dtype=torch.int32)
    gs, dest = tg.route_plan(ids.to(DEV), experts, check=True)
    torch.cuda.synchronize()
    ids_np = ids.numpy()
    np.testing.assert_array_equal(gs.cpu().numpy(), np.bincount(ids_np, minlength=experts))
    order = np.argsort(ids_np, kind="stable")  # grouped row j holds source row order[j]
    want = np.empty(rows, np.int64)
    want[order] = np.arange(rows)
    np.testing.assert_array_equal(dest.cpu().numpy(), want)


def test_route_plan_flags_bad_expert_ids():
    ids = torch.tensor([0, 3, 9, 1], dtype=torch.int32, device=DEV)
    with pytest.raises(tg.InvalidInput):
        tg.route_plan(ids, 4, check=True)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_quantize_dispatch_feeds_the_grouped_gemm(dtype):
    """Tokens -> (quantize + dispatch) -> padding-free grouped GEMM == oracle on the same rows."""
    tokens, topk, experts, k, n = 300, 4, 9, 384, 192
    x = torch.from_numpy(_reference_rows(tokens, k, 5)).to(DEV).to(dtype)
    g = torch.Generator(device="cpu").manual_seed(11)
    eids = torch.stack([torch.randperm(experts, generator=g)[:topk] for _ in range(tokens)]).to(torch.int32)
    d = tg.quantize_dispatch(x, eids.to(DEV), experts, check=True)
    torch.cuda.synchronize()
    # grouped layout: the rows of expert e are tokens routed to it, ascending (t, k)
    flat = eids.reshape(-1).numpy()
    order = np.argsort(flat, kind="stable")
    sizes = tuple(int(s) for s in np.bincount(flat, minlength=experts))
    assert tuple(d.group_sizes.cpu().tolist()) == sizes
    xc, xs = ofp8.quantize_row_tiles(x.float().cpu().numpy())
    want_codes = xc[order // topk]
    want_scales = xs[order // topk]
    np.testing.assert_array_equal(d.a_codes.cpu().numpy(), want_codes)
    np.testing.assert_array_equal(d.a_scales.cpu().numpy(), want_scales)
    # the GEMM over the dispatched rows
    _, _, bc, bsc = per_expert_operands(sizes, n, k, 3)
    c = tg.grouped_gemm_fp8(d.a_codes, d.a_scales, torch.from_numpy(bc).to(DEV), torch.from_numpy(bsc).to(DEV),
                            d.group_sizes)
    got = c.view(torch.int16).cpu().numpy().view(np.uint16)
    assert_parity(got, oracle_c(want_codes, want_scales, bc, bsc, sizes), label="dispatch->gemm")
    # and back to (token, slot) order
    back = tg.gather_rows(c, d.dest_rows, topk)
    assert back.shape == (tokens, topk, n)
    np.testing.assert_array_equal(back[5, 2].view(torch.int16).cpu().numpy(),
                                  c[int(d.dest_rows[5 * topk + 2])].view(torch.int16).cpu().numpy())


@pytest.mark.parametrize("shape", [(1, 1), (128, 128), (200, 300), (3, 256, 384), (2, 7168, 4096)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_quantize_blocks_is_bit_exact(shape, dtype):
    """fp8.py:154-176 per matrix of the batch (per-expert weights [G, K, N])."""
    rng = np.random.Generator(np.random.PCG64(sum(shape)))
    w = rng.standard_normal(shape).astype(np.float32) * np.exp2(rng.integers(-6, 6, size=shape[:-1] + (1,)))
    w = w.astype(np.float32)
    if w.ndim == 3 and w.shape[0] > 1:
        w[1, :128, :128] = 0.0  # an all-zero block: scale 1.0
    wt = torch.from_numpy(w).to(DEV).to(dtype)
    codes, scales = tg.quantize_blocks(wt, check=True)
    torch.cuda.synchronize()
    ref = wt.float().cpu().numpy().reshape((-1,) + shape[-2:])
    got_c = codes.cpu().numpy().reshape((-1,) + shape[-2:])
    got_s = scales.cpu().numpy().reshape((ref.shape[0],) + scales.shape[-2:])
    for b in range(ref.shape[0]):
        want_c, want_s = ofp8.quantize_blocks(ref[b])
        np.testing.assert_array_equal(got_c[b], want_c)
        np.testing.assert_array_equal(got_s[b].view(np.uint32), want_s.view(np.uint32))
