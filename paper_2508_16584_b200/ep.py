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
  5. a device permutation from (source rank, expert) order to expert-contiguous
     order, which is the padding-free grouped layout the kernel consumes, with
     no rows added
combine() reverses steps 5 and 4 on the bf16 outputs and restores the original
(token, k) order.

The transport is torch.distributed, NCCL on GPUs (NVLink 5 / NVSwitch) and
gloo on CPU (tests).  No reference counterpart exists: the reference is
single-process.
"""

from __future__ import annotations

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


def _counts(expert_ids: torch.Tensor, num_experts: int) -> torch.Tensor:
    return torch.bincount(expert_ids.to(torch.int64), minlength=num_experts).to(torch.int32)


def dispatch(a_codes: torch.Tensor, a_scales: torch.Tensor, expert_ids: torch.Tensor, num_experts: int,
             group=None):
    """Send each routed row to the rank that owns its expert.

    a_codes [R, K] uint8 / float8_e4m3fn, a_scales [R, kb] f32, expert_ids [R]
    (one expert per row; a top-k router flattens (token, k) into rows).
    Returns (a_local, sa_local, meta).  a_local is in expert-contiguous order
    for this rank's experts and meta.group_sizes holds the device group sizes.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if num_experts % world:
        raise ValueError(f"{num_experts} experts do not split over {world} ranks")
    epr = num_experts // world
    if a_codes.dtype == torch.float8_e4m3fn:
        a_codes = a_codes.view(torch.uint8)
    dev = a_codes.device
    order = torch.argsort(expert_ids.to(torch.int64), stable=True)
    a_sorted = a_codes.index_select(0, order)
    sa_sorted = a_scales.index_select(0, order)
    counts = _counts(expert_ids, num_experts)                       # [E] rows per expert, local
    return _exchange(a_sorted, sa_sorted, counts, order, epr, group)


def dispatch_tokens(x: torch.Tensor, expert_ids: torch.Tensor, num_experts: int, group=None):
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
    return _exchange(d.a_codes.contiguous(), d.a_scales, d.group_sizes, order, num_experts // world, group)


def _exchange(a_sorted, sa_sorted, counts, order, epr, group):
    """All-to-all of expert-sorted local rows; regroup received rows to expert-contiguous."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
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
    a_recv = torch.empty((n_recv, a_codes.shape[1]), dtype=torch.uint8, device=dev)
    sa_recv = torch.empty((n_recv, a_scales.shape[1]), dtype=a_scales.dtype, device=dev)
    dist.all_to_all_single(a_recv, a_sorted.contiguous(), recv_splits, send_splits, group=group)
    dist.all_to_all_single(sa_recv, sa_sorted.contiguous(), recv_splits, send_splits, group=group)
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
    meta = DispatchMeta(order, send_splits, recv_splits, to_grouped, group_sizes.to(dev), epr)
    del rank
    return a_local, sa_local, meta


def combine(c_local: torch.Tensor, meta: DispatchMeta, group=None) -> torch.Tensor:
    """Return grouped outputs [rows_local, N] to the ranks and rows they came from."""
    c_recv_order = torch.empty_like(c_local)
    c_recv_order.index_copy_(0, meta.to_grouped, c_local)
    out_sorted = torch.empty((sum(meta.send_splits), c_local.shape[1]), dtype=c_local.dtype, device=c_local.device)
    dist.all_to_all_single(out_sorted, c_recv_order, meta.send_splits, meta.recv_splits, group=group)
    out = torch.empty_like(out_sorted)
    out.index_copy_(0, meta.order, out_sorted)
    return out


def local_expert_slice(num_experts: int, group=None) -> slice:
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    epr = num_experts // world
    return slice(rank * epr, (rank + 1) * epr)
