"""GPU safety contracts: device-side validation of the group sizes, programmatic dependent
launch ordering, and dropped routes (expert id -1) in the dispatch / combine chain.

The reference raises on bad input (ConfigError for a negative M_g, engine.py:77-92;
ShapeMismatch when the operands do not hold sum(M_g) rows, engine.py:132-142; InvalidInput for
a bad expert id).  Group sizes here live on the device, so the kernel checks them and a bad
launch writes nothing.
"""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from helpers import assert_parity, oracle_c, per_expert_operands  # noqa: E402
from oracle import fp8 as ofp8  # noqa: E402
from oracle import moe as omoe  # noqa: E402

import paper_2508_16584_b200 as tg  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda"
SENTINEL = 0x5A5A


def _ops(sizes, n, k, seed, m_alloc=None):
    m = m_alloc if m_alloc is not None else sum(max(0, s) for s in sizes)
    g = torch.Generator(device=DEV).manual_seed(seed)
    kb, nb = -(-k // 128), -(-n // 128)
    a = torch.randint(0, 0x7E, (m, k), dtype=torch.uint8, device=DEV, generator=g)
    sa = torch.rand((m, kb), device=DEV, generator=g) + 0.5
    b = torch.randint(0, 0x7E, (len(sizes), k, n), dtype=torch.uint8, device=DEV, generator=g)
    sb = torch.rand((len(sizes), kb, nb), device=DEV, generator=g) + 0.5
    return a, sa, b, sb


@pytest.mark.parametrize("sizes,m_alloc,err,exc", [
    ((100, -1, 30), 130, tg.engine.ERR_NEGATIVE_SIZE, tg.ConfigError),
    ((100, 50, 30), 150, tg.engine.ERR_ROWS_OUT_OF_RANGE, tg.ShapeMismatch),
    ((2 ** 30, 2 ** 30, 5), 64, tg.engine.ERR_ROWS_OUT_OF_RANGE, tg.ShapeMismatch),  # int32 overflow
])
@pytest.mark.parametrize("tile", [None, "1cta", "pair_n256"])
def test_bad_device_group_sizes_flag_and_write_nothing(sizes, m_alloc, err, exc, tile):
    n, k = 256, 256
    a, sa, b, sb = _ops(sizes, n, k, 1, m_alloc=m_alloc)
    gs = torch.tensor(sizes, dtype=torch.int32, device=DEV)
    out = torch.full((m_alloc, n), SENTINEL, dtype=torch.int16, device=DEV)
    tmap = torch.full((tg.max_tiles(m_alloc, len(sizes), n), 9), -1, dtype=torch.int32, device=DEV)
    flag = torch.zeros(1, dtype=torch.int32, device=DEV)
    tg.grouped_gemm_fp8(a, sa, b, sb, gs, out=out, tile_map=tmap, err_flag=flag, tile=tile)
    torch.cuda.synchronize()
    assert int(flag.item()) == err
    assert bool((out == SENTINEL).all()), "a flagged launch stored rows"
    assert bool((tmap == -1).all()), "a flagged launch wrote the tile map"
    with pytest.raises(exc):
        tg.grouped_gemm_fp8(a, sa, b, sb, gs, out=out, check=True, tile=tile)


def test_c_row_offsets_outside_c_are_flagged():
    sizes = (40, 0, 70)
    n, k = 128, 128
    a, sa, b, sb = _ops(sizes, n, k, 2)
    gs = torch.tensor(sizes, dtype=torch.int32, device=DEV)
    out = torch.full((200, n), SENTINEL, dtype=torch.int16, device=DEV)
    for offs, ok in (((0, 5000, 100), True),     # an empty group may point anywhere
                     ((0, 50, 131), False),      # 131 + 70 > 200 rows of C
                     ((-1, 50, 100), False)):
        co = torch.tensor(offs, dtype=torch.int64, device=DEV)
        if ok:
            tg.grouped_gemm_fp8(a, sa, b, sb, gs, out=out, c_row_offsets=co, check=True)
        else:
            with pytest.raises(tg.ShapeMismatch):
                tg.grouped_gemm_fp8(a, sa, b, sb, gs, out=out, c_row_offsets=co, check=True)


def test_valid_launch_leaves_the_flag_clear():
    sizes = (3, 0, 129)
    a, sa, b, sb = _ops(sizes, 128, 256, 3)
    flag = torch.zeros(1, dtype=torch.int32, device=DEV)
    out = tg.grouped_gemm_fp8(a, sa, b, sb, torch.tensor(sizes, dtype=torch.int32, device=DEV), err_flag=flag,
                              check=True)
    assert int(flag.item()) == 0
    want = oracle_c(a.cpu().numpy(), sa.cpu().numpy(), b.cpu().numpy(), sb.cpu().numpy(), sizes)
    assert_parity(out.view(torch.int16).cpu().numpy().view(np.uint16), want)


def test_out_validation_on_the_host():
    sizes = (10, 20)
    a, sa, b, sb = _ops(sizes, 128, 128, 4)
    gs = torch.tensor(sizes, dtype=torch.int32, device=DEV)
    with pytest.raises(tg.ShapeMismatch):  # fewer columns than N
        tg.grouped_gemm_fp8(a, sa, b, sb, gs, out=torch.empty((30, 256), dtype=torch.bfloat16, device=DEV)[:, :64])
    # fewer rows than sum(M_g): the device check flags it (out may hold fewer rows than A)
    with pytest.raises(tg.ShapeMismatch):
        tg.grouped_gemm_fp8(a, sa, b, sb, gs, out=torch.empty((29, 128), dtype=torch.bfloat16, device=DEV),
                            check=True)
    tg.grouped_gemm_fp8(a[:40], sa[:40], b, sb, gs, out=torch.empty((30, 128), dtype=torch.bfloat16, device=DEV),
                        check=True)


@pytest.mark.parametrize("topk", [1, 4])
def test_quantize_dispatch_then_gemm_50_times_without_sync(topk):
    """Programmatic dependent launch must not let a GEMM read its inputs before the kernels
    that write them are done: quantize + dispatch (new activations every iteration, buffers
    recycled by the caching allocator) -> padding-free GEMM, 50 times with no sync, then
    every iteration's output against the oracle on that iteration's own inputs."""
    tokens, experts, k, n = 96, 5, 256, 128
    gen = torch.Generator(device=DEV).manual_seed(9)
    _, _, bc, bsc = per_expert_operands((1,) * experts, n, k, 21)
    b, sb = torch.from_numpy(bc).to(DEV), torch.from_numpy(bsc).to(DEV)
    xs, ids, outs = [], [], []
    for i in range(50):
        x = torch.randn((tokens, k), device=DEV, generator=gen) * (1 + i)
        e = torch.stack([torch.randperm(experts, device=DEV, generator=gen)[:topk] for _ in range(tokens)])
        e = e.to(torch.int32)
        d = tg.quantize_dispatch(x, e, experts)
        outs.append(tg.grouped_gemm_fp8(d.a_codes, d.a_scales, b, sb, d.group_sizes))
        xs.append(x)
        ids.append(e)
        del d
    torch.cuda.synchronize()
    for x, e, c in zip(xs, ids, outs):
        flat = e.reshape(-1).cpu().numpy()
        order = np.argsort(flat, kind="stable")
        sizes = tuple(int(s) for s in np.bincount(flat, minlength=experts))
        xc, xsc = ofp8.quantize_row_tiles(x.cpu().numpy())
        want = oracle_c(xc[order // topk], xsc[order // topk], bc, bsc, sizes)
        assert_parity(c.view(torch.int16).cpu().numpy().view(np.uint16), want)


@pytest.mark.parametrize("mode", ["default", "overlap", "serial"])
def test_gemm_chain_into_one_output_keeps_order(mode):
    """GEMM -> GEMM on one output buffer (write after write) and GEMM -> pad -> GEMM (the padded
    baseline reads what the previous kernel wrote), 30 rounds without a sync."""
    n, k = 256, 512
    big, small = (3000, 2000, 1000), (200, 0, 33)
    ab, sab, bb, sbb = _ops(big, n, k, 5)
    as_, sas, bs, sbs = _ops(small, n, k, 6)
    gb = torch.tensor(big, dtype=torch.int32, device=DEV)
    gsm = torch.tensor(small, dtype=torch.int32, device=DEV)
    kw = {"pdl": mode != "serial", "pdl_overlap": mode == "overlap"}
    want_b = tg.grouped_gemm_fp8(ab, sab, bb, sbb, gb).view(torch.int16).clone()
    want_s = tg.grouped_gemm_fp8(as_, sas, bs, sbs, gsm).view(torch.int16).clone()
    ws = tg.PaddedWorkspace(sum(small), 3, k, n, DEV)
    out = torch.empty((sum(big), n), dtype=torch.bfloat16, device=DEV)
    outp = torch.empty((sum(small), n), dtype=torch.bfloat16, device=DEV)
    torch.cuda.synchronize()
    for _ in range(30):
        tg.grouped_gemm_fp8(ab, sab, bb, sbb, gb, out=out, **kw)
        tg.grouped_gemm_fp8(as_, sas, bs, sbs, gsm, out=out, **kw)
        tg.padded_grouped_gemm_fp8(as_, sas, bs, sbs, gsm, ws, out=outp, **kw)
    torch.cuda.synchronize()
    ms = sum(small)
    assert torch.equal(out[:ms].view(torch.int16), want_s[:ms])
    assert torch.equal(out[ms:].view(torch.int16), want_b[ms:])
    assert torch.equal(outp.view(torch.int16), want_s[:ms])


def test_dropped_routes_are_skipped_end_to_end():
    """Expert ids outside [0, E) (a router's -1 for a dropped token, or E): no grouped row, no
    out-of-bounds write; the combine and router gradient treat the route as absent."""
    tokens, topk, experts, k, n = 64, 2, 4, 256, 128
    gen = torch.Generator(device=DEV).manual_seed(12)
    x = torch.randn((tokens, k), device=DEV, generator=gen)
    e = torch.stack([torch.randperm(experts, device=DEV, generator=gen)[:topk] for _ in range(tokens)])
    e = e.to(torch.int32)
    e[3, 0] = -1
    e[10, 1] = experts
    e[11, :] = -1
    with pytest.raises(tg.InvalidInput):
        tg.quantize_dispatch(x, e, experts, check=True)
    d = tg.quantize_dispatch(x, e, experts)
    torch.cuda.synchronize()
    flat = e.reshape(-1).cpu().numpy()
    ok = (flat >= 0) & (flat < experts)
    dest = d.dest_rows.cpu().numpy()
    assert np.all(dest[~ok] == -1)
    sizes = np.bincount(flat[ok], minlength=experts)
    assert tuple(d.group_sizes.cpu().tolist()) == tuple(int(s) for s in sizes)
    valid_src = np.flatnonzero(ok)
    order = valid_src[np.argsort(flat[ok], kind="stable")]
    xc, xsc = ofp8.quantize_row_tiles(x.cpu().numpy())
    m = int(sizes.sum())
    np.testing.assert_array_equal(d.a_codes[:m].cpu().numpy(), xc[order // topk])
    np.testing.assert_array_equal(dest[order], np.arange(m))
    # combine: a dropped route contributes nothing
    c = torch.randn((d.a_codes.shape[0], n), device=DEV, generator=gen).to(torch.bfloat16)
    w = torch.rand((tokens, topk), device=DEV, generator=gen)
    y = tg.moe.combine(c, d.dest_rows, w)
    torch.cuda.synchronize()
    cb = c.view(torch.int16).cpu().numpy().view(np.uint16)
    want = omoe.combine(cb, np.where(dest < 0, 0, dest), np.where(ok.reshape(tokens, topk), w.cpu().numpy(), 0))
    np.testing.assert_array_equal(y.view(torch.int16).cpu().numpy().view(np.uint16), want)


@pytest.mark.parametrize("layout", ["kn", "nk"])
@pytest.mark.parametrize("tile", [None, "1cta", "pair_n256"])
def test_b_index_groups_share_experts(layout, tile):
    """tagg_grouped_gemm_fp8_ex's b_index: 7 groups over 3 experts (the (source, expert)
    segments of an all-to-all).  Equals the oracle with each group's expert B spelled out."""
    sizes = (100, 0, 257, 3, 128, 64, 300)
    bidx = (2, 0, 1, 2, 0, 1, 1)
    n, k = 256, 384
    m = sum(sizes)
    g = torch.Generator(device=DEV).manual_seed(17)
    a = torch.randint(0, 0x7E, (m, k), dtype=torch.uint8, device=DEV, generator=g)
    sa = torch.rand((m, k // 128), device=DEV, generator=g) + 0.5
    shape = (3, k, n) if layout == "kn" else (3, n, k)
    sshape = (3, k // 128, n // 128) if layout == "kn" else (3, n // 128, k // 128)
    b = torch.randint(0, 0x7E, shape, dtype=torch.uint8, device=DEV, generator=g)
    sb = torch.rand(sshape, device=DEV, generator=g) + 0.5
    gs = torch.tensor(sizes, dtype=torch.int32, device=DEV)
    bi = torch.tensor(bidx, dtype=torch.int32, device=DEV)
    out = tg.grouped_gemm_fp8(a, sa, b, sb, gs, b_layout=layout, b_index=bi, tile=tile, check=True)
    bn, sbn = b.cpu().numpy()[list(bidx)], sb.cpu().numpy()[list(bidx)]
    want = oracle_c(a.cpu().numpy(), sa.cpu().numpy(), bn, sbn, sizes, b_layout=layout)
    assert_parity(out.view(torch.int16).cpu().numpy().view(np.uint16), want)
    bad = torch.tensor((2, 0, 1, 3, 0, 1, 1), dtype=torch.int32, device=DEV)  # expert 3 of 3
    with pytest.raises(tg.ShapeMismatch):
        tg.grouped_gemm_fp8(a, sa, b, sb, gs, b_layout=layout, b_index=bad, tile=tile, check=True)
    ok_empty = torch.tensor((2, 99, 1, 2, 0, 1, 1), dtype=torch.int32, device=DEV)  # empty group: ignored
    tg.grouped_gemm_fp8(a, sa, b, sb, gs, b_layout=layout, b_index=ok_empty, tile=tile, check=True)
