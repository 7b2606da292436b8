"""Expert-parallel token dispatch and combine for the grouped GEMM.

Experts shard across ranks.  Rank p owns experts
[p*E/P, (p+1)*E/P), their B weights and scales, and every routed row sent to
them.  Groups never interact (engine.py:269-279), so the GEMM itself needs no
collective.  The only exchange is token dispatch before it (and the combine
after it).  That exchange is the DeepSeek-V3 down-projection config of
BASELINE.json.

dispatch():
  1. stable sort of the local (token, expert) rows by expert -> per-expert counts [E]
  2. all_to_all_single of the int32 counts (every rank learns what it receives)
  3. one host read of the split sizes (the only sync)
  4. all_to_all_single of the FP8 rows [rows, K] and their 1x128 scales [rows, kb]
  5. in_place=False: a device permutation from (source rank, expert) order to
     expert-contiguous order (one group per local expert).  in_place=True (what the
     pipelined path uses): no permutation -- every (source rank, expert) segment is a
     group of its own and meta.b_index names its expert, so the grouped GEMM reads the
     received rows where they landed and writes C in the order combine() sends back
     (tagg_grouped_gemm_fp8_ex's b_index).
combine() reverses steps 5 and 4 on the bf16 outputs and restores the original
(token, k) order.  At world size 1 the all-to-alls are identities and are skipped.

The transport is torch.distributed, NCCL on GPUs (NVLink 5 / NVSwitch) and
gloo on CPU (tests).  No reference counterpart exists: the reference is
single-process.
"""

from __future__ import annotations

import contextlib
from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass
class DispatchMeta:
    """What combine() needs to send rows back and restore the local order."""

    order: torch.Tensor        # local sort permutation (rows sorted by expert)
    send_splits: list          # rows sent to each rank
    recv_splits: list          # rows received from each rank
    to_grouped: torch.Tensor   # received-row index of each grouped row
    group_sizes: torch.Tensor  # int32 [E_local] rows per local expert (device)
    experts_per_rank: int
    from_grouped: torch.Tensor | None = None  # inverse of to_grouped
    inv_order: torch.Tensor | None = None     # inverse of order: sorted position of each local row
    b_index: torch.Tensor | None = None       # in_place: int32 [P * E_local] expert of each segment group


def _inverse(perm: torch.Tensor) -> torch.Tensor:
    """Inverse permutation.  Both passes of combine are gathers (index_select) over it:
    a row gather streams at ~5 TB/s on B200, a row scatter (index_copy_) at ~1.5."""
    inv = torch.empty_like(perm)
    inv[perm] = torch.arange(perm.numel(), device=perm.device, dtype=perm.dtype)
    return inv


def _counts(expert_ids: torch.Tensor, num_experts: int) -> torch.Tensor:
    return torch.bincount(expert_ids.to(torch.int64), minlength=num_experts).to(torch.int32)


def dispatch(a_codes: torch.Tensor, a_scales: torch.Tensor, expert_ids: torch.Tensor, num_experts: int,
             group=None, in_place: bool = False):
    """Send each routed row to the rank that owns its expert.

    a_codes [R, K] uint8 / float8_e4m3fn, a_scales [R, kb] f32, expert_ids [R]
    (one expert per row; a top-k router flattens (token, k) into rows).
    Returns (a_local, sa_local, meta).  a_local is in expert-contiguous order
    for this rank's experts and meta.group_sizes holds the device group sizes.  With
    ``in_place`` the rows stay in arrival order, (source rank, expert) segments: then
    meta.group_sizes has one entry per segment and meta.b_index its expert.
    """
    world = dist.get_world_size(group)
    if num_experts % world:
        raise ValueError(f"{num_experts} experts do not split over {world} ranks")
    epr = num_experts // world
    if a_codes.dtype == torch.float8_e4m3fn:
        a_codes = a_codes.view(torch.uint8)
    order = torch.argsort(expert_ids.to(torch.int64), stable=True)
    a_sorted = a_codes.index_select(0, order)
    sa_sorted = a_scales.index_select(0, order)
    counts = _counts(expert_ids, num_experts)                       # [E] rows per expert, local
    return _exchange(a_sorted, sa_sorted, counts, order, epr, group, in_place=in_place)


def dispatch_tokens(x: torch.Tensor, expert_ids: torch.Tensor, num_experts: int, group=None,
                    in_place: bool = False):
    """Quantize-and-dispatch from bf16/f32 activations (SURVEY.md §8f ranks 1+3).

    x [T, K] activations, expert_ids [T, topk].  The fused kernel (quant.quantize_dispatch)
    quantizes every token once (1x128, fp8.py:132-151) and writes its topk rows already in
    expert order, so the local sort of dispatch() disappears; the rows then go through the
    same all-to-all.  Returns (a_local, sa_local, meta) like dispatch(); combine() inverts it
    back to (token, k) rows.
    """
    from . import quant

    world = dist.get_world_size(group)
    if num_experts % world:
        raise ValueError(f"{num_experts} experts do not split over {world} ranks")
    d = quant.quantize_dispatch(x, expert_ids, num_experts)
    order = torch.empty_like(d.dest_rows, dtype=torch.int64)       # sorted row -> local (t, k) row
    order[d.dest_rows.to(torch.int64)] = torch.arange(d.dest_rows.numel(), device=x.device)
    return _exchange(d.a_codes.contiguous(), d.a_scales, d.group_sizes, order, num_experts // world, group,
                     inv_order=d.dest_rows.to(torch.int64), in_place=in_place)


def _a2a(out, inp, out_splits, in_splits, group):
    """all_to_all_single, skipped at world size 1 where it is the identity (a full-size copy)."""
    if dist.get_world_size(group) == 1:
        return inp
    dist.all_to_all_single(out, inp, out_splits, in_splits, group=group)
    return out


def segment_b_index(world: int, epr: int, device) -> torch.Tensor:
    """Expert (local index) of each (source rank, expert) segment group, source-major."""
    return (torch.arange(world * epr, device=device, dtype=torch.int32) % epr).contiguous()


def _exchange(a_sorted, sa_sorted, counts, order, epr, group, inv_order=None, in_place=False):
    """All-to-all of expert-sorted local rows; regroup received rows to expert-contiguous
    (or, in_place, leave them as (source, expert) segment groups)."""
    world = dist.get_world_size(group)
    dev = a_sorted.device
    a_codes, a_scales = a_sorted, sa_sorted
    recv_counts = torch.empty_like(counts)                          # [P * epr] from each source
    dist.all_to_all_single(recv_counts, counts, group=group)
    send_splits = counts.view(world, epr).sum(1)
    recv_mat = recv_counts.view(world, epr)                          # [src, local expert]
    recv_splits_t = recv_mat.sum(1)
    both = torch.cat([send_splits, recv_splits_t]).cpu().tolist()   # the one host sync
    send_splits, recv_splits = both[:world], both[world:]
    n_recv = sum(recv_splits)
    a_recv = torch.empty((n_recv, a_codes.shape[1]), dtype=torch.uint8, device=dev) if world > 1 else None
    sa_recv = torch.empty((n_recv, a_scales.shape[1]), dtype=a_scales.dtype, device=dev) if world > 1 else None
    a_recv = _a2a(a_recv, a_sorted.contiguous(), recv_splits, send_splits, group)
    sa_recv = _a2a(sa_recv, sa_sorted.contiguous(), recv_splits, send_splits, group)
    if in_place:
        meta = DispatchMeta(order, send_splits, recv_splits, None, recv_mat.reshape(-1).to(torch.int32).contiguous(),
                            epr, inv_order=_inverse(order) if inv_order is None else inv_order,
                            b_index=segment_b_index(world, epr, dev))
        return a_recv, sa_recv, meta
    # received rows are ordered (src, expert); regroup them to (expert, src)
    src_off = torch.cumsum(recv_mat.reshape(-1).to(torch.int64), 0) - recv_mat.reshape(-1).to(torch.int64)
    src_off = src_off.view(world, epr)
    group_sizes = recv_mat.sum(0).to(torch.int32)                    # [epr]
    seg_len = recv_mat.t().reshape(-1).to(torch.int64)               # segments in (expert, src) order
    seg_start = src_off.t().reshape(-1)
    seg_dst = torch.cumsum(seg_len, 0) - seg_len
    idx = torch.arange(n_recv, device=dev, dtype=torch.int64)
    seg_of = torch.repeat_interleave(torch.arange(seg_len.numel(), device=dev), seg_len, output_size=n_recv)
    to_grouped = seg_start[seg_of] + (idx - seg_dst[seg_of])
    a_local = a_recv.index_select(0, to_grouped)
    sa_local = sa_recv.index_select(0, to_grouped)
    meta = DispatchMeta(order, send_splits, recv_splits, to_grouped, group_sizes.to(dev), epr,
                        from_grouped=_inverse(to_grouped), inv_order=_inverse(order) if inv_order is None else inv_order)
    return a_local, sa_local, meta


def combine(c_local: torch.Tensor, meta: DispatchMeta, group=None) -> torch.Tensor:
    """Return grouped outputs [rows_local, N] to the ranks and rows they came from."""
    c_recv_order = c_local if meta.from_grouped is None else c_local.index_select(0, meta.from_grouped)
    world = dist.get_world_size(group)
    out_sorted = None
    if world > 1:
        out_sorted = torch.empty((sum(meta.send_splits), c_local.shape[1]), dtype=c_local.dtype,
                                 device=c_local.device)
    out_sorted = _a2a(out_sorted, c_recv_order, meta.send_splits, meta.recv_splits, group)
    return out_sorted.index_select(0, meta.inv_order)


# ---------------------------------------------------------------------------------------------
# Overlapped dispatch -> GEMM -> combine


@dataclass
class ChunkPlan:
    """Exchange plan for C row chunks, built with ONE count all-to-all and ONE host read.

    Local rows are split into C contiguous chunks and stably sorted by (chunk, expert);
    chunk c's rows then sit at sorted positions [send_off[c], send_off[c+1]), grouped by
    destination rank because experts are rank-contiguous.
    """

    chunks: int
    order: torch.Tensor            # sorted position -> local row (int64 [R])
    send_splits: list              # [C][P] rows of chunk c sent to rank p
    recv_splits: list              # [C][P] rows of chunk c received from rank p
    send_off: list                 # [C+1] chunk offsets in the sorted send buffer
    to_grouped: list               # [C] received-row index of each grouped row (int64 device)
    from_grouped: list             # [C] inverse of to_grouped[c]
    inv_order: torch.Tensor        # inverse of order
    group_sizes: list              # [C] int32 [E_local] device group sizes of chunk c
    experts_per_rank: int
    seg_sizes: list | None = None  # [C] int32 [P * E_local]: chunk c's (source rank, expert) segments
    b_index: torch.Tensor | None = None  # int32 [P * E_local]: the expert of each segment

    @property
    def recv_rows(self) -> list:
        return [sum(r) for r in self.recv_splits]


def _regroup_index(recv_mat: torch.Tensor, n_recv: int) -> torch.Tensor:
    """Received rows arrive (src rank, expert)-ordered; index them in (expert, src) order."""
    world, epr = recv_mat.shape
    dev = recv_mat.device
    flat = recv_mat.reshape(-1).to(torch.int64)
    src_off = (torch.cumsum(flat, 0) - flat).view(world, epr)
    seg_len = recv_mat.t().reshape(-1).to(torch.int64)
    seg_start = src_off.t().reshape(-1)
    seg_dst = torch.cumsum(seg_len, 0) - seg_len
    idx = torch.arange(n_recv, device=dev, dtype=torch.int64)
    seg_of = torch.repeat_interleave(torch.arange(seg_len.numel(), device=dev), seg_len, output_size=n_recv)
    return seg_start[seg_of] + (idx - seg_dst[seg_of])


def plan_chunks(expert_ids: torch.Tensor, num_experts: int, chunks: int, group=None) -> ChunkPlan:
    """Sort R routed rows by (chunk, expert) and exchange every chunk's counts at once."""
    world = dist.get_world_size(group)
    if num_experts % world:
        raise ValueError(f"{num_experts} experts do not split over {world} ranks")
    if chunks < 1:
        raise ValueError("chunks must be >= 1")
    epr = num_experts // world
    ids = expert_ids.reshape(-1).to(torch.int64)
    rows = ids.numel()
    dev = ids.device
    chunk_of = torch.arange(rows, device=dev, dtype=torch.int64) * chunks // max(rows, 1)
    key = chunk_of * num_experts + ids
    order = torch.argsort(key, stable=True)
    counts = torch.bincount(key, minlength=chunks * num_experts).to(torch.int32).view(chunks, world, epr)
    send = counts.permute(1, 0, 2).contiguous()                    # [dst rank, chunk, local expert]
    recv = torch.empty_like(send)                                   # [src rank, chunk, local expert]
    dist.all_to_all_single(recv, send, group=group)
    both = torch.cat([counts.sum(2).reshape(-1), recv.sum(2).t().reshape(-1)]).cpu().tolist()  # one sync
    n = chunks * world
    send_splits = [both[c * world:(c + 1) * world] for c in range(chunks)]
    recv_splits = [both[n + c * world:n + (c + 1) * world] for c in range(chunks)]
    send_off = [0]
    for c in range(chunks):
        send_off.append(send_off[-1] + sum(send_splits[c]))
    to_grouped = [_regroup_index(recv[:, c, :], sum(recv_splits[c])) for c in range(chunks)]
    group_sizes = [recv[:, c, :].sum(0).to(torch.int32) for c in range(chunks)]
    seg_sizes = [recv[:, c, :].reshape(-1).to(torch.int32).contiguous() for c in range(chunks)]
    return ChunkPlan(chunks, order, send_splits, recv_splits, send_off, to_grouped,
                     [_inverse(t) for t in to_grouped], _inverse(order), group_sizes, epr, seg_sizes,
                     segment_b_index(world, epr, dev))


_COMM_STREAMS: dict = {}


def _comm_stream(dev: torch.device):
    """One side stream per device for the exchange (created once, reused by every call)."""
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    if key not in _COMM_STREAMS:
        _COMM_STREAMS[key] = torch.cuda.Stream(dev)
    return _COMM_STREAMS[key]


def pipelined_expert_gemm(a_codes: torch.Tensor, a_scales: torch.Tensor, expert_ids: torch.Tensor,
                          num_experts: int, expert_gemm, n_out: int, *, chunks: int = 4, group=None,
                          comm_stream=None, out_dtype=torch.bfloat16, plan: ChunkPlan | None = None,
                          in_place: bool = True):
    """Dispatch -> per-expert GEMM -> combine, pipelined over row chunks.

    a_codes [R, K] e4m3 codes, a_scales [R, kb] f32 and expert_ids [R] are this rank's routed
    rows (dispatch() semantics).  ``expert_gemm(codes, scales, group_sizes) -> [rows, n_out]``
    runs this rank's experts on one chunk's rows in the padding-free grouped layout (codes may
    be a row-strided view).  Returns [R, n_out]: every row's output back in local row order.

    With ``in_place`` (default) the GEMM reads each chunk's received rows where they landed:
    ``expert_gemm(codes, scales, group_sizes, b_index=..., out=...)`` gets one group per
    (source rank, expert) segment, b_index naming the expert, and writes its result straight
    into the buffer the return all-to-all sends (tagg_grouped_gemm_fp8_ex's b_index), so no
    row is permuted between the exchanges.  in_place=False regroups each chunk to one group
    per expert first and back after (3-argument expert_gemm).

    Codes and scales travel packed in one all-to-all per chunk (K + 4*kb bytes a row, padded
    to 16).  On CUDA the all-to-alls run on ``comm_stream``: chunk c's GEMM overlaps chunk
    c+1's dispatch and chunk c-1's combine.  Give the GEMM fewer SMs than the device has
    (grouped_gemm_fp8 ``max_sms``) so the NCCL kernels find room beside its persistent grid.
    """
    if a_codes.dtype == torch.float8_e4m3fn:
        a_codes = a_codes.view(torch.uint8)
    rows, k = a_codes.shape
    kb = a_scales.shape[1]
    dev = a_codes.device
    if plan is None and chunks == 1 and in_place:
        # one chunk has nothing to overlap: the sequential in-place exchange, without the
        # chunk plan's bookkeeping and the packed-row copy
        a_loc, sa_loc, meta = dispatch(a_codes, a_scales, expert_ids.reshape(-1), num_experts, group, in_place=True)
        out = torch.empty((a_loc.shape[0], n_out), dtype=out_dtype, device=dev)
        if a_loc.shape[0]:
            y = expert_gemm(a_loc, sa_loc, meta.group_sizes, b_index=meta.b_index, out=out)
            if y.data_ptr() != out.data_ptr():
                out.copy_(y[:a_loc.shape[0]])
        return combine(out, meta, group)
    if plan is None:
        plan = plan_chunks(expert_ids, num_experts, chunks, group)
    width = -(-(k + 4 * kb) // 16) * 16     # 16-byte rows: the GEMM's TMA reads codes in place
    cuda = dev.type == "cuda"
    compute = torch.cuda.current_stream(dev) if cuda else None
    comm = (comm_stream or _comm_stream(dev)) if cuda else None
    # one slab per buffer kind for all chunks, allocated up front on the compute stream
    # (4 allocations instead of 4 per chunk: the caching allocator then reuses them call to call)
    recv_off = [0]
    for n in plan.recv_rows:
        recv_off.append(recv_off[-1] + n)
    packed = torch.empty((rows, width), dtype=torch.uint8, device=dev)
    packed[:, :k] = a_codes.index_select(0, plan.order)
    packed[:, k:k + 4 * kb] = a_scales.contiguous().index_select(0, plan.order).view(torch.uint8)
    world = dist.get_world_size(group)
    recv_all = torch.empty((recv_off[-1], width), dtype=torch.uint8, device=dev) if world > 1 else packed
    grouped_all = None if in_place else torch.empty_like(recv_all)
    back_all = torch.empty((recv_off[-1], n_out), dtype=out_dtype, device=dev)
    out_sorted = back_all if world == 1 else torch.empty((rows, n_out), dtype=out_dtype, device=dev)

    def on(stream):
        return torch.cuda.stream(stream) if cuda else contextlib.nullcontext()

    arrived = [torch.cuda.Event() if cuda else None for _ in range(plan.chunks)]
    done = [torch.cuda.Event() if cuda else None for _ in range(plan.chunks)]
    if cuda:
        comm.wait_stream(compute)                                    # packed rows and the slabs exist

    def send_chunk(c):
        with on(comm):
            if world > 1:  # at world size 1 the received rows are the packed rows themselves
                dist.all_to_all_single(recv_all[recv_off[c]:recv_off[c + 1]],
                                       packed[plan.send_off[c]:plan.send_off[c + 1]], plan.recv_splits[c],
                                       plan.send_splits[c], group=group)
            if cuda:
                arrived[c].record(comm)

    def return_chunk(c):
        if world == 1:
            return  # back_all is out_sorted (below)
        with on(comm):
            if cuda:
                comm.wait_event(done[c])
            dist.all_to_all_single(out_sorted[plan.send_off[c]:plan.send_off[c + 1]],
                                   back_all[recv_off[c]:recv_off[c + 1]], plan.send_splits[c], plan.recv_splits[c],
                                   group=group)

    send_chunk(0)
    for c in range(plan.chunks):
        if cuda:
            compute.wait_event(arrived[c])
        lo, hi = recv_off[c], recv_off[c + 1]
        if hi > lo and in_place:
            rows_c = recv_all[lo:hi]
            y = expert_gemm(rows_c[:, :k], rows_c[:, k:k + 4 * kb].contiguous().view(torch.float32),
                            plan.seg_sizes[c], b_index=plan.b_index, out=back_all[lo:hi])
            if y.data_ptr() != back_all[lo:hi].data_ptr():
                back_all[lo:hi].copy_(y[:hi - lo])
        elif hi > lo:
            grouped = grouped_all[lo:hi]
            torch.index_select(recv_all[lo:hi], 0, plan.to_grouped[c], out=grouped)  # padding-free grouped layout
            y = expert_gemm(grouped[:, :k], grouped[:, k:k + 4 * kb].contiguous().view(torch.float32),
                            plan.group_sizes[c])
            torch.index_select(y[:hi - lo], 0, plan.from_grouped[c], out=back_all[lo:hi])
        if cuda:
            done[c].record(compute)
        if c + 1 < plan.chunks:
            send_chunk(c + 1)                                         # ahead of combine(c): GEMM c+1 needs it
        return_chunk(c)
    if cuda:
        compute.wait_stream(comm)
        for t in {id(x): x for x in (packed, recv_all, back_all, out_sorted)}.values():
            t.record_stream(comm)
    return out_sorted.index_select(0, plan.inv_order)


def local_expert_slice(num_experts: int, group=None) -> slice:
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    epr = num_experts // world
    return slice(rank * epr, (rank + 1) * epr)
