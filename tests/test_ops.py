"""torch.ops.tagg.* (SURVEY.md §8b item 2): CUDA-only registration, fake kernels, parity."""

from __future__ import annotations

import numpy as np
import pytest
import torch
from torch._subclasses.fake_tensor import FakeTensorMode

import paper_2508_16584_b200 as tg  # noqa: F401  (registers the ops)


def test_ops_are_registered():
    for name in ("grouped_gemm_fp8", "quantize_row_tiles", "quantize_dispatch", "wgrad_fp8", "swiglu_quantize",
                 "combine"):
        assert hasattr(torch.ops.tagg, name)


def test_no_cpu_kernel():
    a = torch.zeros((4, 128), dtype=torch.uint8)
    with pytest.raises(NotImplementedError):
        torch.ops.tagg.grouped_gemm_fp8(a, torch.ones((4, 1)), torch.zeros((1, 128, 64), dtype=torch.uint8),
                                        torch.ones((1, 1, 1)), torch.tensor([4], dtype=torch.int32))


def test_fake_kernels_infer_shapes():
    with FakeTensorMode():
        a = torch.empty((300, 512), dtype=torch.uint8, device="cuda")
        sa = torch.empty((300, 4), dtype=torch.float32, device="cuda")
        b = torch.empty((3, 512, 256), dtype=torch.uint8, device="cuda")
        sb = torch.empty((3, 4, 2), dtype=torch.float32, device="cuda")
        gs = torch.empty((3,), dtype=torch.int32, device="cuda")
        c = torch.ops.tagg.grouped_gemm_fp8(a, sa, b, sb, gs)
        assert c.shape == (300, 256) and c.dtype == torch.bfloat16
        x = torch.empty((10, 300), dtype=torch.bfloat16, device="cuda")
        codes, scales = torch.ops.tagg.quantize_row_tiles(x)
        assert codes.shape == (10, 300) and scales.shape == (10, 3)
        e = torch.empty((10, 4), dtype=torch.int32, device="cuda")
        ac, asc, gsz, dest = torch.ops.tagg.quantize_dispatch(x, e, 16)
        assert ac.shape == (40, 300) and asc.shape == (40, 3) and gsz.shape == (16,) and dest.shape == (40,)
        dw = torch.ops.tagg.wgrad_fp8(a[:, :256], sa, a[:, :128], sa, gs)
        assert dw.shape == (3, 256, 128) and dw.dtype == torch.bfloat16
        hq, hs = torch.ops.tagg.swiglu_quantize(torch.empty((300, 512), dtype=torch.bfloat16, device="cuda"), gs)
        assert hq.shape == (300, 256) and hs.shape == (300, 2)
        y = torch.ops.tagg.combine(c, torch.empty((300,), dtype=torch.int32, device="cuda"),
                                   torch.empty((75, 4), dtype=torch.float32, device="cuda"))
        assert y.shape == (75, 256) and y.dtype == torch.bfloat16


@pytest.mark.gpu
def test_op_matches_the_wrapper():
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    sizes = [67, 0, 200]
    m, k, n = sum(sizes), 384, 256
    a = torch.randint(0, 126, (m, k), dtype=torch.uint8, device=dev, generator=g)
    sa = torch.rand((m, 3), device=dev, generator=g) + 0.5
    b = torch.randint(0, 126, (3, k, n), dtype=torch.uint8, device=dev, generator=g)
    sb = torch.rand((3, 3, 2), device=dev, generator=g) + 0.5
    gs = torch.tensor(sizes, dtype=torch.int32, device=dev)
    want = tg.grouped_gemm_fp8(a, sa, b, sb, gs)
    got = torch.ops.tagg.grouped_gemm_fp8(a, sa, b, sb, gs)
    torch.cuda.synchronize()
    assert np.array_equal(got[:m].view(torch.int16).cpu().numpy(), want[:m].view(torch.int16).cpu().numpy())
    x = torch.randn((50, 300), device=dev, generator=g)
    c1, s1 = torch.ops.tagg.quantize_row_tiles(x)
    c2, s2 = tg.quantize_row_tiles(x)
    assert torch.equal(c1, c2) and torch.equal(s1, s2)


def test_product_paths_refuse_cpu_tensors():
    """No CPU fallback anywhere on the product path: CPU tensors raise before any work."""
    from paper_2508_16584_b200 import InvalidInput, ShapeMismatch, moe, quant
    from paper_2508_16584_b200.hostpipe import HostBatch, run_host_batches

    x = torch.zeros((4, 256), dtype=torch.bfloat16)
    gs = torch.tensor([4], dtype=torch.int32)
    with pytest.raises(InvalidInput):
        moe.swiglu_quantize(x, gs)
    with pytest.raises(InvalidInput):
        moe.swiglu_backward_quantize(torch.zeros((4, 256), dtype=torch.bfloat16), torch.zeros((4, 128),
                                                                                            dtype=torch.bfloat16), gs)
    with pytest.raises(InvalidInput):
        moe.combine(x, torch.zeros(4, dtype=torch.int32), torch.ones((4, 1)))
    with pytest.raises(ShapeMismatch):
        moe.gather_scale_rows(x, torch.zeros(2, dtype=torch.int32))
    with pytest.raises(InvalidInput):
        quant.quantize_row_tiles(x)
    with pytest.raises(InvalidInput):
        quant.route_plan(torch.zeros(4, dtype=torch.int32), 2)
    with pytest.raises(ValueError):
        tg.grouped_gemm_fp8(torch.zeros((4, 128), dtype=torch.uint8), torch.ones((4, 1)),
                            torch.zeros((1, 128, 64), dtype=torch.uint8), torch.ones((1, 1, 1)), gs)
    with pytest.raises((ValueError, RuntimeError, AssertionError, AttributeError, ShapeMismatch)):
        run_host_batches([HostBatch(x, x, gs, x)], torch.zeros((1, 128, 64), dtype=torch.uint8),
                         torch.ones((1, 1, 1)), depth=0)
