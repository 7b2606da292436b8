"""Ablation timing of the GEMM kernel on one residual-sweep problem (r=64)."""
import sys, json
sys.path.insert(0, ".")
import torch
import paper_2508_16584_b200 as tg
import ctypes
from paper_2508_16584_b200 import _lib

# the ablation flags are honoured only by the diagnostics build (make -C paper_2508_16584_b200/csrc trace)
_L = ctypes.CDLL(str(_lib.PKG / "libtagg_trace.so"))
for _n, (_r, _a) in _lib.SIGNATURES.items():
    getattr(_L, _n).restype, getattr(_L, _n).argtypes = _r, _a
lib = lambda: _L  # noqa: E731
from bench import Problem

dev = torch.device("cuda", 0)
res = {}
for name, sizes, n, k, G in [("sweep_r64", [tuple(128 * g + 64 for g in range(8))], 4096, 7168, 8),
                             ("sq8192", [(8192,)], 8192, 8192, 1)]:
    P = Problem(torch, name, sizes, n, k, G, dev, seed=1)
    variants = [("n256", 16), ("n256_nomath", 16 | 1024), ("n256_noprom", 16 | 512), ("n256_neither", 16 | 256 | 512),
                ("n128", 8), ("n128_nomath", 8 | 1024), ("n128_noprom", 8 | 512), ("n128_neither", 8 | 256 | 512),
                ("c1_128", 4), ("c1_128_noprom", 4 | 512), ("c1_128_neither", 4 | 256 | 512)]
    for label, flags in variants:
        def run():
            rc = lib().tagg_grouped_gemm_fp8(P.a.data_ptr(), P.a.stride(0), P.sa.data_ptr(), P.m_alloc,
                                             P.b.data_ptr(), 0, G, P.sb.data_ptr(), P.sb.stride(0), P.sb.stride(1),
                                             P.sb.stride(2), P.gs[0].data_ptr(), G, n, k, P.out.data_ptr(), n,
                                             P.m_alloc, None, None, flags, torch.cuda.current_stream().cuda_stream)
            assert rc == 0, rc
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20):
            run()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 20
        res[f"{name}/{label}"] = (ms, P.flops[0] / ms / 1e9)
        print(f"{name:10s} {label:11s} {ms*1e3:8.1f} us  {P.flops[0]/ms/1e9:8.1f} TFLOP/s", flush=True)
    del P
# reference point: torch._scaled_mm fp8 8192^3 (cuBLAS)
a = torch.randn(8192, 8192, device=dev).to(torch.float8_e4m3fn)
b = torch.randn(8192, 8192, device=dev).to(torch.float8_e4m3fn).t()
one = torch.ones((), device=dev)
for _ in range(3):
    torch._scaled_mm(a, b, one, one, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    torch._scaled_mm(a, b, one, one, out_dtype=torch.bfloat16)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 20
print(f"cublas fp8 8192^3 scaled_mm: {2*8192**3/ms/1e9:.1f} TFLOP/s")
