"""Vendor comparison (optional): flashinfer's CUTLASS grouped FP8 GEMM with the
same groupwise fp32 scales (1x128 A, 128x128 B) against this kernel, same device, same data.

flashinfer requires every group offset to be a multiple of 4, so its groups are padded to 4
rows (a few pad rows per group); TFLOP/s count valid rows only for both.  B is K-major [G, N, K]
(flashinfer's "nt"), which this kernel takes as b_layout="nk".  First call JIT-compiles
flashinfer's kernels (minutes).

python tools/vendor_cmp.py  -> one JSON line per shape
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2508_16584_b200 as tg  # noqa: E402
from bench import deepseek_gateup_sizes  # noqa: E402

dev = torch.device("cuda", 0)


def timed(fn, iters=20, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def case(name, sizes, n, k):
    from flashinfer.gemm import group_gemm_fp8_nt_groupwise

    G = len(sizes)
    g = torch.Generator(device=dev).manual_seed(7)
    m = sum(sizes)
    kb, nb = k // 128, n // 128
    a = (torch.randn((m, k), device=dev, generator=g) * 0.5).to(torch.float8_e4m3fn)
    sa = torch.rand((m, kb), device=dev, generator=g) * 1e-2 + 1e-3
    b = (torch.randn((G, n, k), device=dev, generator=g) * 0.5).to(torch.float8_e4m3fn)
    sb = torch.rand((G, nb, kb), device=dev, generator=g) * 1e-2 + 1e-3
    gs = torch.tensor(sizes, dtype=torch.int32, device=dev)
    ours = lambda: tg.grouped_gemm_fp8(a, sa, b, sb, gs, b_layout="nk")  # noqa: E731
    c_ours = ours()
    # flashinfer: groups padded to multiples of 4 rows
    psz = [-(-s // 4) * 4 for s in sizes]
    mp = sum(psz)
    idx, src = [], 0
    for s, p in zip(sizes, psz):
        idx += list(range(src, src + s)) + [m] * (p - s)
        src += s
    gather = torch.tensor(idx, dtype=torch.int64, device=dev)
    a_p = torch.cat([a.view(torch.uint8), torch.zeros((1, k), dtype=torch.uint8, device=dev)]).index_select(0, gather)
    sa_p = torch.cat([sa, torch.ones((1, kb), device=dev)]).index_select(0, gather)
    indptr = torch.tensor([0] + list(torch.tensor(psz).cumsum(0).tolist()), dtype=torch.int32, device=dev)
    out: dict = {"shape": name, "groups": G, "rows": m, "N": n, "K": k, "flashinfer_pad_rows": mp - m}
    flops = 2.0 * m * n * k
    out["ours_tflops"] = flops / (timed(ours) * 1e-3) / 1e12
    for mma_sm in (1, 2):
        try:
            fi = lambda: group_gemm_fp8_nt_groupwise(a_p.view(torch.float8_e4m3fn), b, sa_p, sb, indptr,  # noqa: E731
                                                     scale_major_mode="K", mma_sm=mma_sm, out_dtype=torch.bfloat16)
            c_fi = fi()
            ms = timed(fi)
            keep = torch.tensor([i for i, v in enumerate(idx) if v < m], dtype=torch.int64, device=dev)
            d = (c_fi.index_select(0, keep).float() - c_ours.float()).abs()
            ref = c_ours.float().abs().amax(dim=1, keepdim=True).clamp_min(1e-30)
            out[f"flashinfer_mma_sm{mma_sm}_tflops"] = flops / (ms * 1e-3) / 1e12
            out[f"flashinfer_mma_sm{mma_sm}_max_rel_diff_vs_ours"] = float((d / ref).max())
        except Exception as exc:  # noqa: BLE001
            out[f"flashinfer_mma_sm{mma_sm}_error"] = f"{type(exc).__name__}: {str(exc)[:200]}"
    print(json.dumps(out), flush=True)


_, local = deepseek_gateup_sizes(seed=0)
case("deepseek_v3_gateup_ep8_rank0", [int(x) for x in local], 4096, 7168)
q, _ = deepseek_gateup_sizes(seed=2, experts=128, local=128)
case("qwen3_dgrad_gateup", [int(x) for x in q], 4096, 3072)
counts, _ = deepseek_gateup_sizes(seed=1)
case("deepseek_v3_down_256e_1gpu", [int(x) for x in counts], 7168, 2048)
