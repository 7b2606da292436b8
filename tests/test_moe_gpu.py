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
                                    sa.data_ptr(), err.data_ptr(), None, 0, torch.cuda.current_stream().cuda_stream)
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


def _dequant_blocks(codes, scales):
    v = ofp8.DECODE_TABLE[codes].astype(np.float64)
    e, r, c = v.shape
    s = np.repeat(np.repeat(scales.astype(np.float64), 128, axis=1), 128, axis=2)[:, :r, :c]
    return v * s


@pytest.mark.parametrize("k", [7168, 200, 128])
@pytest.mark.parametrize("weighted", [True, False])
def test_quantize_gather_rows_equals_gather_then_quantize(k, weighted):
    """tagg_quantize_gather_rows (row r = bf16(w[r] * x[index[r]]), quantized in one pass) is
    bit-identical to K10's gathered rows quantized by quantize_row_tiles."""
    torch.manual_seed(k)
    t, r = 300, 1000
    x = (torch.randn((t, k), device=DEV) * 4).to(torch.bfloat16)
    idx = torch.randint(0, t, (r,), device=DEV, dtype=torch.int32)
    w = torch.rand(r, device=DEV) * 2 if weighted else None
    got_c, got_s = tg.quantize_gather_rows(x, idx, w, check=True)
    dc = moe.gather_scale_rows(x, idx, w)
    want_c, want_s = tg.quantize_row_tiles(dc)
    torch.cuda.synchronize()
    assert torch.equal(got_c, want_c)
    assert torch.equal(got_s.view(torch.int32), want_s.view(torch.int32))


@pytest.mark.parametrize("recipe", ["per_column", "dy_block128", "mxfp8"])
def test_moe_ffn_backward_matches_float64(recipe):
    """moe_ffn(save=True) + moe_ffn_backward against float64 math on the same (dequantized) FP8
    weights.  Activations and gradients pass through 1x128 / column-block FP8 on the GPU, so
    each gradient is compared by relative Frobenius error."""
    rng = np.random.default_rng(8)
    t, topk, e, hid, inter = 200, 2, 4, 256, 128
    x = rng.standard_normal((t, hid)).astype(np.float32)
    eids = np.stack([rng.permutation(e)[:topk] for _ in range(t)]).astype(np.int32)
    wts = rng.random((t, topk)).astype(np.float32)
    dy = rng.standard_normal((t, hid)).astype(np.float32)
    w1 = rng.standard_normal((e, hid, 2 * inter)).astype(np.float32) * 0.08
    w2 = rng.standard_normal((e, inter, hid)).astype(np.float32) * 0.08
    c1, s1 = tg.quantize_blocks(torch.from_numpy(w1).to(DEV))
    c2, s2 = tg.quantize_blocks(torch.from_numpy(w2).to(DEV))
    weights = moe.ExpertWeights(c1, s1, c2, s2)
    xb = torch.from_numpy(x).to(DEV).to(torch.bfloat16)
    y, ctx = moe.moe_ffn(xb, torch.from_numpy(eids).to(DEV), torch.from_numpy(wts).to(DEV), weights, save=True)
    g = moe.moe_ffn_backward(torch.from_numpy(dy).to(DEV).to(torch.bfloat16), ctx, weights, wgrad_recipe=recipe)
    torch.cuda.synchronize()
    W1 = _dequant_blocks(c1.cpu().numpy(), s1.cpu().numpy())
    W2 = _dequant_blocks(c2.cpu().numpy(), s2.cpu().numpy())
    xr = xb.float().cpu().numpy().astype(np.float64)
    dyr = torch.from_numpy(dy).to(torch.bfloat16).float().numpy().astype(np.float64)
    yr = np.zeros((t, hid))
    dx = np.zeros((t, hid))
    dW1 = np.zeros_like(W1)
    dW2 = np.zeros_like(W2)
    dw = np.zeros((t, topk))
    for ti in range(t):
        for k in range(topk):
            ex = eids[ti, k]
            z = xr[ti] @ W1[ex]
            gg, uu = z[:inter], z[inter:]
            sig = 1 / (1 + np.exp(-gg))
            v = gg * sig * uu
            o = v @ W2[ex]
            yr[ti] += wts[ti, k] * o
            do = wts[ti, k] * dyr[ti]
            dv = W2[ex] @ do
            dz = np.concatenate([dv * uu * sig * (1 + gg * (1 - sig)), dv * gg * sig])
            dx[ti] += W1[ex] @ dz
            dW2[ex] += np.outer(v, do)
            dW1[ex] += np.outer(xr[ti], dz)
            dw[ti, k] = dyr[ti] @ o

    def rel(got, want):
        return float(np.linalg.norm(got - want) / np.linalg.norm(want))

    assert rel(y.float().cpu().numpy(), yr) < 0.05
    assert rel(g.dx.float().cpu().numpy(), dx) < 0.08
    assert rel(g.dw_gate_up.float().cpu().numpy(), dW1) < 0.08
    assert rel(g.dw_down.float().cpu().numpy(), dW2) < 0.08
    assert rel(g.dweights.cpu().numpy(), dw) < 0.08


@pytest.mark.parametrize("i", [128, 384])
def test_swiglu_backward_quantize_matches_oracle(i):
    rng = np.random.default_rng(i + 1)
    sizes = (150, 0, 77)
    m, m_alloc = sum(sizes), 300
    hb = _bf16_bits(rng.standard_normal((m_alloc, 2 * i)).astype(np.float32) * 2)
    db = _bf16_bits(rng.standard_normal((m_alloc, i)).astype(np.float32))
    h = torch.from_numpy(hb.view(np.int16)).to(DEV).view(torch.bfloat16)
    dh = torch.from_numpy(db.view(np.int16)).to(DEV).view(torch.bfloat16)
    gs = torch.tensor(sizes, dtype=torch.int32, device=DEV)
    dgu, a, sa = moe.swiglu_backward_quantize(h, dh, gs, check=True)
    torch.cuda.synchronize()
    want = omoe.swiglu_backward(hb[:m], db[:m])
    got = dgu[:m].float().cpu().numpy()
    np.testing.assert_allclose(got, want, rtol=2.0 ** -7, atol=1e-6 * np.abs(want).max())
    wc, ws = ofp8.quantize_row_tiles(want)
    np.testing.assert_allclose(sa[:m].cpu().numpy(), ws, rtol=2.0 ** -6)
    gc = a[:m].cpu().numpy().astype(np.int16)
    wc = wc.astype(np.int16)
    step = np.abs((gc & 0x7F) - (wc & 0x7F))
    assert np.all((((gc >> 7) == (wc >> 7)) & (step <= 1)) | ((gc & 0x7F) + (wc & 0x7F) <= 1))


def test_gather_scale_rows_is_bit_exact_and_router_grad():
    rng = np.random.default_rng(3)
    t, topk, h = 97, 4, 384
    xb = _bf16_bits(rng.standard_normal((t, h)).astype(np.float32))
    idx = rng.integers(0, t, 500).astype(np.int32)
    w = rng.random(500).astype(np.float32)
    x = torch.from_numpy(xb.view(np.int16)).to(DEV).view(torch.bfloat16)
    got = moe.gather_scale_rows(x, torch.from_numpy(idx).to(DEV), torch.from_numpy(w).to(DEV))
    want = omoe.bf16_rne(w[:, None] * ofp8.bf16_bits_to_f32(xb)[idx])
    np.testing.assert_array_equal(got.view(torch.int16).cpu().numpy().view(np.uint16), want)
    plain = moe.gather_scale_rows(x, torch.from_numpy(idx).to(DEV))
    np.testing.assert_array_equal(plain.view(torch.int16).cpu().numpy().view(np.uint16), xb[idx])
    # router grad: <dy[t], c[dest[t*topk+k]]>
    cb = _bf16_bits(rng.standard_normal((t * topk, h)).astype(np.float32))
    dest = rng.permutation(t * topk).astype(np.int32)
    c = torch.from_numpy(cb.view(np.int16)).to(DEV).view(torch.bfloat16)
    g = moe.router_grad(x, c, torch.from_numpy(dest).to(DEV), topk).cpu().numpy()
    xf = ofp8.bf16_bits_to_f32(xb).astype(np.float64)
    cf = ofp8.bf16_bits_to_f32(cb).astype(np.float64)
    want_g = np.einsum("th,tkh->tk", xf, cf[dest].reshape(t, topk, h))
    np.testing.assert_allclose(g, want_g, rtol=1e-5, atol=1e-4)


def test_moe_ffn_forward_is_graph_capturable():
    """The whole padding-free MoE FFN forward has no host sync: it captures into one CUDA graph,
    and replays with new activations and new routing match eager calls bit for bit."""
    rng = np.random.default_rng(12)
    t, topk, e, hid, inter = 256, 4, 8, 256, 128
    w1 = torch.from_numpy(rng.standard_normal((e, hid, 2 * inter)).astype(np.float32) * 0.1).to(DEV)
    w2 = torch.from_numpy(rng.standard_normal((e, inter, hid)).astype(np.float32) * 0.1).to(DEV)
    c1, s1 = tg.quantize_blocks(w1)
    c2, s2 = tg.quantize_blocks(w2)
    weights = moe.ExpertWeights(c1, s1, c2, s2)

    def inputs(seed):
        r = np.random.default_rng(seed)
        x = torch.from_numpy(r.standard_normal((t, hid)).astype(np.float32)).to(DEV).to(torch.bfloat16)
        ids = torch.from_numpy(np.stack([r.permutation(e)[:topk] for _ in range(t)]).astype(np.int32)).to(DEV)
        wt = torch.from_numpy(r.random((t, topk)).astype(np.float32)).to(DEV)
        return x, ids, wt

    x, ids, wt = inputs(0)
    moe.moe_ffn(x, ids, wt, weights)  # warm-up outside capture (allocator, tensor maps)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        with torch.cuda.graph(graph, stream=side):
            y = moe.moe_ffn(x, ids, wt, weights)
    torch.cuda.current_stream().wait_stream(side)
    for seed in (1, 2):
        nx, nids, nwt = inputs(seed)
        x.copy_(nx)
        ids.copy_(nids)
        wt.copy_(nwt)
        graph.replay()
        want = moe.moe_ffn(nx, nids, nwt, weights)
        torch.cuda.synchronize()
        assert torch.equal(y.view(torch.int16), want.view(torch.int16)), seed
