"""EP dispatch on the GPU with NCCL (world size 1 in-process; the multi-rank logic is
covered by tests/test_ep_gloo.py): the fused quantize-and-dispatch path equals
quantizing first and dispatching the FP8 rows, and combine() returns every row home."""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist

import paper_2508_16584_b200 as tg
from paper_2508_16584_b200 import ep

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl1():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29613")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_dispatch_tokens_equals_quantize_then_dispatch(nccl1):
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(9)
    tokens, topk, experts, k = 500, 4, 16, 384
    x = torch.randn((tokens, k), device=dev, generator=g).to(torch.bfloat16)
    eids = torch.topk(torch.rand((tokens, experts), device=dev, generator=g), topk, dim=1).indices.to(torch.int32)
    a1, sa1, m1 = ep.dispatch_tokens(x, eids, experts)
    codes, scales = tg.quantize_row_tiles(x)
    rows_codes = codes.repeat_interleave(topk, dim=0)                # local (t, k) rows
    rows_scales = scales.repeat_interleave(topk, dim=0)
    a2, sa2, m2 = ep.dispatch(rows_codes, rows_scales, eids.reshape(-1), experts)
    torch.cuda.synchronize()
    assert torch.equal(a1, a2) and torch.equal(sa1, sa2)
    assert torch.equal(m1.group_sizes, m2.group_sizes)
    # combine returns each grouped row to its (token, k) slot
    c = a1.to(torch.float32)[:, :8]
    back = ep.combine(c, m1)
    want = rows_codes.to(torch.float32)[:, :8]
    assert np.array_equal(back.cpu().numpy(), want.cpu().numpy())


@pytest.mark.parametrize("in_place", [True, False])
@pytest.mark.parametrize("chunks", [1, 3])
def test_pipelined_expert_gemm_matches_oracle(nccl1, chunks, in_place):
    """Chunked dispatch -> padding-free GEMM (SM-capped grid) -> combine, overlapped on two
    streams, equals the oracle row by row (values within helpers.REL_TOL)."""
    from helpers import assert_parity, oracle_c, per_expert_operands
    from oracle import fp8 as ofp8

    dev = torch.device("cuda", 0)
    rows, experts, k, n = 900, 8, 384, 256
    g = torch.Generator().manual_seed(chunks)
    eids = torch.multinomial(torch.arange(1, experts + 1, dtype=torch.float).pow(-1.0), rows, True, generator=g)
    a, sa, _, _ = ofp8.random_operands(rows, 128, k, 17)
    order = np.argsort(eids.numpy(), kind="stable")
    sizes = tuple(int(x) for x in np.bincount(eids.numpy(), minlength=experts))
    _, _, bc, bsc = per_expert_operands(sizes, n, k, 23)
    b, sb = torch.from_numpy(bc).to(dev), torch.from_numpy(bsc).to(dev)

    def gemm(codes, scales, gs, b_index=None, out=None):
        return tg.grouped_gemm_fp8(codes, scales, b, sb, gs, max_sms=120, b_index=b_index, out=out)

    out = ep.pipelined_expert_gemm(torch.from_numpy(a).to(dev), torch.from_numpy(sa).to(dev), eids.to(dev),
                                   experts, gemm, n, chunks=chunks, in_place=in_place)
    torch.cuda.synchronize()
    want_sorted = oracle_c(a[order], sa[order], bc, bsc, sizes)
    want = np.empty_like(want_sorted)
    want[order] = want_sorted
    assert_parity(out.view(torch.int16).cpu().numpy().view(np.uint16), want, label=f"chunks={chunks} in_place={in_place}")


def test_in_place_dispatch_gemm_combine_matches_regrouped(nccl1):
    """dispatch(in_place=True): the received (source, expert) segments feed the GEMM as groups with
    b_index; combine() returns rows home.  Bitwise equal to the regrouped path (same GEMM values:
    a group's rows are independent of how groups are cut)."""
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(3)
    rows, experts, k, n = 1500, 16, 256, 128
    a = torch.randint(0, 0x7E, (rows, k), dtype=torch.uint8, device=dev, generator=g)
    sa = torch.rand((rows, k // 128), device=dev, generator=g) + 0.5
    eid = torch.randint(0, experts, (rows,), device=dev, generator=g)
    b = torch.randint(0, 0x7E, (experts, k, n), dtype=torch.uint8, device=dev, generator=g)
    sb = torch.rand((experts, k // 128, n // 128), device=dev, generator=g) + 0.5
    a1, sa1, m1 = ep.dispatch(a, sa, eid, experts)
    c1 = tg.grouped_gemm_fp8(a1, sa1, b, sb, m1.group_sizes)
    a2, sa2, m2 = ep.dispatch(a, sa, eid, experts, in_place=True)
    assert m2.b_index is not None and m2.group_sizes.numel() == experts
    c2 = tg.grouped_gemm_fp8(a2, sa2, b, sb, m2.group_sizes, b_index=m2.b_index, check=True)
    back1, back2 = ep.combine(c1, m1), ep.combine(c2, m2)
    torch.cuda.synchronize()
    assert torch.equal(back1.view(torch.int16), back2.view(torch.int16))
