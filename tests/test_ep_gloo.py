"""Expert-parallel dispatch/combine over torch.distributed (gloo, world_size 2, CPU).

Checks the host-side multi-rank path of SURVEY.md §8e without a GPU.
* Every rank receives exactly the rows routed to its experts, in
  expert-contiguous (padding-free grouped) order, with matching scales and
  group sizes.
* combine() inverts dispatch() bit for bit.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_16584_b200 import ep


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(rank, rows, k, experts, seed):
    g = torch.Generator().manual_seed(seed * 100 + rank)
    a = torch.randint(0, 256, (rows, k), dtype=torch.uint8, generator=g)
    sa = torch.rand((rows, -(-k // 128)), generator=g)
    # skewed routing, some experts get nothing
    if rows == 0:
        return a, sa, torch.zeros(0, dtype=torch.int64)
    e = torch.multinomial(torch.arange(1, experts + 1, dtype=torch.float).pow(-0.8), rows, True, generator=g)
    e[e == experts - 1] = 0
    return a, sa, e


def _worker(rank, world, port, rows_per_rank, k, experts, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, sa, e = _inputs(rank, rows_per_rank[rank], k, experts, seed)
        a_loc, sa_loc, meta = ep.dispatch(a, sa, e, experts)
        # expected: all ranks' rows for my experts, expert-major then source rank, stable
        sl = ep.local_expert_slice(experts)
        want_a, want_sa, want_gs = [], [], []
        for ex in range(sl.start, sl.stop):
            cnt = 0
            for src in range(world):
                a2, sa2, e2 = _inputs(src, rows_per_rank[src], k, experts, seed)
                m = e2 == ex
                want_a.append(a2[m])
                want_sa.append(sa2[m])
                cnt += int(m.sum())
            want_gs.append(cnt)
        ok = torch.equal(a_loc, torch.cat(want_a)) and torch.equal(sa_loc, torch.cat(want_sa))
        ok = ok and meta.group_sizes.tolist() == want_gs
        # the "GEMM" stand-in: any row-wise map; combine must return it to the source rows
        c_loc = (a_loc[:, :64].to(torch.int16) * 3 + 1).to(torch.bfloat16)
        back = ep.combine(c_loc, meta)
        ok = ok and torch.equal(back, (a[:, :64].to(torch.int16) * 3 + 1).to(torch.bfloat16))
        # in place: rows stay in arrival order, one group per (source rank, expert) segment
        a_in, sa_in, m_in = ep.dispatch(a, sa, e, experts, in_place=True)
        want_a, want_sa, want_seg = [], [], []
        for src in range(world):
            a2, sa2, e2 = _inputs(src, rows_per_rank[src], k, experts, seed)
            for ex in range(sl.start, sl.stop):
                m = e2 == ex
                want_a.append(a2[m])
                want_sa.append(sa2[m])
                want_seg.append(int(m.sum()))
        ok = ok and torch.equal(a_in, torch.cat(want_a)) and torch.equal(sa_in, torch.cat(want_sa))
        ok = ok and m_in.group_sizes.tolist() == want_seg
        ok = ok and m_in.b_index.tolist() == [i % (sl.stop - sl.start) for i in range(world * (sl.stop - sl.start))]
        back_in = ep.combine((a_in[:, :64].to(torch.int16) * 3 + 1).to(torch.bfloat16), m_in)
        ok = ok and torch.equal(back_in, (a[:, :64].to(torch.int16) * 3 + 1).to(torch.bfloat16))
        q.put((rank, bool(ok), sum(want_gs)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rows_per_rank,experts", [((300, 170), 8), ((1, 0), 4), ((257, 513), 16)])
def test_dispatch_combine_world2(rows_per_rank, experts):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, rows_per_rank, 256, experts, 3, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert sum(n for _, _, n in res) == sum(rows_per_rank)


def _pipeline_worker(rank, world, port, rows_per_rank, k, experts, chunks, seed, q, in_place=True):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, sa, e = _inputs(rank, rows_per_rank[rank], k, experts, seed)
        epr = experts // world
        seen = []

        def fake_gemm(codes, scales, gs, b_index=None, out=None):
            """Stand-in for the grouped GEMM: echoes each row's first codes, its local expert
            (read off the group sizes and the groups' expert index, so it only matches if every
            group's rows belong to its expert) and scale."""
            bi = torch.arange(epr) if b_index is None else b_index.to(torch.int64)
            seen.append(torch.bincount(bi, weights=gs.to(torch.float64), minlength=epr).to(torch.int64))
            local_e = torch.repeat_interleave(bi, gs.to(torch.int64))
            return torch.cat([codes[:, :4].to(torch.float32), local_e[:, None].to(torch.float32),
                              scales[:, :1]], 1)

        out = ep.pipelined_expert_gemm(a, sa, e, experts, fake_gemm, 6, chunks=chunks, out_dtype=torch.float32,
                                       in_place=in_place)
        want = torch.cat([a[:, :4].to(torch.float32), (e % epr)[:, None].to(torch.float32), sa[:, :1]], 1)
        ok = out.shape == want.shape and torch.equal(out, want)
        # every chunk's GEMM got exactly that chunk's rows for my experts
        sl = ep.local_expert_slice(experts)
        total = torch.zeros(epr, dtype=torch.int64)
        for gs in seen:
            total += gs.to(torch.int64)
        want_total = torch.zeros(epr, dtype=torch.int64)
        for src in range(world):
            _, _, e2 = _inputs(src, rows_per_rank[src], k, experts, seed)
            want_total += torch.bincount(e2[(e2 >= sl.start) & (e2 < sl.stop)] - sl.start, minlength=epr)
        ok = ok and torch.equal(total, want_total)
        q.put((rank, bool(ok), len(seen)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("in_place", [True, False])
@pytest.mark.parametrize("rows_per_rank,experts,chunks", [((300, 170), 8, 3), ((1, 0), 4, 2), ((3, 2), 4, 5), ((257, 90), 8, 1)])
def test_pipelined_expert_gemm_world2(rows_per_rank, experts, chunks, in_place):
    """Chunked dispatch -> expert GEMM -> combine returns every row's result home, in order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pipeline_worker, args=(r, 2, port, rows_per_rank, 384, experts, chunks, 5, q, in_place))
             for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
