"""Host-buffer batches through the grouped GEMM with the copies overlapped.

A caller holding its operands and results in host memory (the reference's
``run_adaptive`` takes and returns numpy arrays, engine.py:184-343) pays PCIe for
every byte.  ``run_host_batches`` streams a sequence of independent grouped GEMMs
so that batch i's device->host read of C overlaps batch i+1's GEMM and batch i+2's
host->device inputs:

    h2d stream      : inputs of batch i  (waits until batch i-depth's GEMM read its slot)
    current stream  : GEMM of batch i    (waits for its inputs and for batch i-depth's
                                          D2H to have read the C slot it reuses)
    d2h stream      : C rows of batch i  -> host

Device buffers rotate over ``depth`` slots.  Inputs already on the device are used
in place.  Everything is stream-ordered: the call returns with the work enqueued,
and the caller synchronizes, or reads ``done`` (an event on the current stream).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .engine import grouped_gemm_fp8
from .errors import ShapeMismatch


@dataclass
class HostBatch:
    """One grouped GEMM: A / S_A / group sizes (host, pinned for async copies, or device)
    and the host tensor receiving C's valid rows (bf16 [>= sum(M_g), N])."""

    a: torch.Tensor
    a_scales: torch.Tensor
    group_sizes: torch.Tensor
    out: torch.Tensor


def _stage(src: torch.Tensor, buf, dev):
    """src on the device: used as is.  On the host: copied into a (reused) device buffer."""
    if src.is_cuda:
        return src, buf
    if buf is None or buf.numel() < src.numel() or buf.dtype != src.dtype:
        buf = torch.empty(src.numel(), dtype=src.dtype, device=dev)
    view = buf[:src.numel()].view(src.shape)
    view.copy_(src, non_blocking=True)
    return view, buf


def run_host_batches(batches, b: torch.Tensor, b_scales: torch.Tensor, *, b_layout: str = "kn",
                     exact_promotion: bool = False, depth: int = 2):
    """Run every batch's padding-free grouped GEMM (same expert weights B resident on the
    device); C's first sum(M_g) rows land in ``batch.out``.  Returns an event recorded on
    the current stream once every copy has finished."""
    if depth < 1:
        raise ValueError("depth must be >= 1")
    dev = b.device
    compute = torch.cuda.current_stream(dev)
    h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    n = b.shape[-1] if b_layout == "kn" else b.shape[-2]
    slots = [{"a": None, "sa": None, "gs": None, "c": None, "read": None, "drained": None} for _ in range(depth)]
    h2d.wait_stream(compute)  # B and any device inputs are ready
    for i, bt in enumerate(batches):
        if bt.out.is_cuda or bt.out.dtype not in (torch.bfloat16, torch.int16, torch.uint16):
            raise ShapeMismatch("batch.out must be a host bf16 tensor")
        sl = slots[i % depth]
        with torch.cuda.stream(h2d):
            if sl["read"] is not None:
                h2d.wait_event(sl["read"])  # the GEMM of batch i - depth has read this slot
            a, sl["a"] = _stage(bt.a, sl["a"], dev)
            sa, sl["sa"] = _stage(bt.a_scales, sl["sa"], dev)
            gs, sl["gs"] = _stage(bt.group_sizes, sl["gs"], dev)
            staged = torch.cuda.Event()
            staged.record(h2d)
        compute.wait_event(staged)
        if sl["drained"] is not None:
            compute.wait_event(sl["drained"])  # batch i - depth's C has left the slot
        m_alloc = a.shape[0]
        if sl["c"] is None or sl["c"].shape[0] < m_alloc or sl["c"].shape[1] != n:
            sl["c"] = torch.empty((max(m_alloc, 1), n), dtype=torch.bfloat16, device=dev)
        # The only same-stream predecessor is the previous batch's GEMM, which writes another
        # C slot (or, at depth 1, this one: the stores keep WAW order); the inputs arrive by
        # event from the copy stream.  So the main loop may overlap that GEMM's tail.
        c = grouped_gemm_fp8(a, sa, b, b_scales, gs, b_layout=b_layout, out=sl["c"],
                             exact_promotion=exact_promotion, pdl_overlap=True)
        sl["read"] = torch.cuda.Event()
        sl["read"].record(compute)
        rows = int(bt.group_sizes.sum()) if not bt.group_sizes.is_cuda else m_alloc
        with torch.cuda.stream(d2h):
            d2h.wait_event(sl["read"])
            bt.out[:rows].copy_(c[:rows].view(bt.out.dtype), non_blocking=True)
            sl["drained"] = torch.cuda.Event()
            sl["drained"].record(d2h)
        for t in (a, sa, gs):
            if t.is_cuda:
                t.record_stream(compute)
        c.record_stream(d2h)
    compute.wait_stream(d2h)
    compute.wait_stream(h2d)
    done = torch.cuda.Event()
    done.record(compute)
    return done
