"""MoE FFN steps around the padding-free GEMM (csrc/tagg_moe.cu) against the CPU oracle.

* swiglu_quantize: scales equal fl(amax/448) of the oracle's v within a few ulp (numpy's and
  CUDA's float32 exp may differ by an ulp), codes within one e4m3 step, >= 99% identical;
  rows past sum(M_g) untouched.
* combine: bit-exact (same fp32 operation order, no FMA).
* moe_ffn: the whole padding-free chain against the oracle chain.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2508_16584_b200 as tg
from helpers import oracle_c
from oracle import fp8 as ofp8
from oracle import moe as omoe
from paper_2508_16584_b200 import moe
from paper_2508_16584_b200._lib import lib

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def _bf16_bits(x: np.ndarray) -> np.ndarray:
    return omoe.bf16_rne(x.astype(np.float32))


@pytest.mark.parametrize("i", [128, 200, 1536])
def test_swiglu_quantize_matches_oracle(i):
    rng = np.random.default_rng(i)
    sizes = (200, 0, 311, 17)
    m, m_alloc = sum(sizes), 700
    h = rng.standard_normal((m_alloc, 2 * i)).astype(np.float32) * np.exp2(rng.integers(-3, 4, (m_alloc, 1)))
    hb = _bf16_bits(h)
    ht = torch.from_numpy(hb.view(np.int16)).to(DEV)
    lda = -(-i // 16) * 16
    kb = -(-i // 128)
    a = torch.full((m_alloc, lda), 0x5A, dtype=torch.uint8, device=DEV)
    sa = torch.full((m_alloc, kb), -7.0, dtype=torch.float32, device=DEV)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    gs = torch.tensor(sizes, dtype=torch.int32, device=DEV)
    rc = lib().tagg_swiglu_quantize(ht.data_ptr(), 2 * i, gs.data_ptr(), len(sizes), m_alloc, i, a.data_ptr(), lda,
                                    sa.data_ptr(), err.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    got_a, got_s = a.cpu().numpy(), sa.cpu().numpy()
    assert np.all(got_a[m:] == 0x5A) and np.all(got_s[m:] == -7.0), "rows past sum(M_g) written"
    assert int(err.item()) == 0
    want_c, want_s = ofp8.quantize_row_tiles(omoe.swiglu(hb[:m]))
    np.testing.assert_allclose(got_s[:m], want_s, rtol=2.0 ** -20, atol=0)
    gc = got_a[:m, :i].astype(np.int16)
    wc = want_c.astype(np.int16)
    same_sign = (gc >> 7) == (wc >> 7)
    step = np.abs((gc & 0x7F) - (wc & 0x7F))
    assert np.all((same_sign & (step <= 1)) | ((gc & 0x7F) + (wc & 0x7F) <= 1)), "codes differ by more than one step"
    assert (gc == wc).mean() >= 0.99


@pytest.mark.parametrize("topk,n", [(1, 64), (4, 7168), (8, 1024)])
def test_combine_is_bit_exact(topk, n):
    rng = np.random.default_rng(topk * n)
    t = 333
    rows = t * topk
    c = _bf16_bits(rng.standard_normal((rows + 5, n)).astype(np.float32))
    dest = rng.permutation(rows).astype(np.int32)
    w = rng.random((t, topk)).astype(np.float32)
    w /= w.sum(1, keepdims=True)
    got = moe.combine(torch.from_numpy(c.view(np.int16)).to(DEV).view(torch.bfloat16), torch.from_numpy(dest).to(DEV),
                      torch.from_numpy(w).to(DEV))
    np.testing.assert_array_equal(got.view(torch.int16).cpu().numpy().view(np.uint16), omoe.combine(c, dest, w))


def test_moe_ffn_matches_the_oracle_chain():
    rng = np.random.default_rng(5)
    t, topk, e, hid, inter = 300, 4, 8, 256, 128
    x = (rng.standard_normal((t, hid)) * np.exp2(rng.integers(-2, 3, (t, 1)))).astype(np.float32)
    eids = np.stack([rng.permutation(e)[:topk] for _ in range(t)]).astype(np.int32)
    wts = rng.random((t, topk)).astype(np.float32)
    w1 = rng.standard_normal((e, hid, 2 * inter)).astype(np.float32) * 0.1
    w2 = rng.standard_normal((e, inter, hid)).astype(np.float32) * 0.1
    c1, s1 = tg.quantize_blocks(torch.from_numpy(w1).to(DEV))
    c2, s2 = tg.quantize_blocks(torch.from_numpy(w2).to(DEV))
    weights = moe.ExpertWeights(c1, s1, c2, s2)
    y = moe.moe_ffn(torch.from_numpy(x).to(DEV), torch.from_numpy(eids).to(DEV), torch.from_numpy(wts).to(DEV),
                    weights)
    got = ofp8.bf16_bits_to_f32(y.view(torch.int16).cpu().numpy().view(np.uint16))
    # oracle chain: quantize -> stable dispatch -> GEMM -> swiglu + quantize -> GEMM -> combine
    xc, xs = ofp8.quantize_row_tiles(x)
    flat = eids.reshape(-1)
    order = np.argsort(flat, kind="stable")
    sizes = tuple(int(v) for v in np.bincount(flat, minlength=e))
    dest = np.empty_like(order)
    dest[order] = np.arange(order.size)
    h = oracle_c(xc[order // topk], xs[order // topk], c1.cpu().numpy(), s1.cpu().numpy(), sizes)
    ac, asc = ofp8.quantize_row_tiles(omoe.swiglu(h))
    c = oracle_c(ac, asc, c2.cpu().numpy(), s2.cpu().numpy(), sizes)
    want = ofp8.bf16_bits_to_f32(omoe.combine(c, dest.astype(np.int32), wts))
    scale = np.abs(want).max(axis=1, keepdims=True)
    err = np.abs(got - want) / np.maximum(scale, 1e-30)
    assert err.max() <= 2.0 ** -4, err.max()
    assert err.mean() <= 2.0 ** -9, err.mean()
