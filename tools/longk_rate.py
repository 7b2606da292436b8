"""K1 k-block rate without tile transitions, in wall time: one 256x256 pair tile per cluster
(M = 256 x 74, N = 256, K = 16384: 128 k-blocks per tile), TFLOP/s over 10 launches, for the
production library and the diagnostics build's ablations (noload / nomath / noprom / neither).
Compare with tools/micro/nbuf.cu (same pipeline without TMA, scales or epilogue)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from bench import Problem  # noqa: E402
from paper_2508_16584_b200 import _lib  # noqa: E402


def load(path):
    L = ctypes.CDLL(path)
    for nm, (r, a) in _lib.SIGNATURES.items():
        if hasattr(L, nm):
            getattr(L, nm).restype, getattr(L, nm).argtypes = r, a
    return L


dev = torch.device("cuda", 0)
k = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
P = Problem(torch, "longk", [(256 * 74,)], 256, k, 1, dev, seed=1)
libs = [("prod", load(str(_lib.LIB_PATH)), 0)]
tr = _lib.PKG / "libtagg_trace.so"
if tr.exists():
    T = load(str(tr))
    libs += [("trace-build full", T, 0), ("noload", T, 256), ("nomath", T, 1024), ("noprom", T, 512),
             ("neither", T, 768)]
for rnd in range(2):
    for name, L, flags in libs:
        def run():
            rc = L.tagg_grouped_gemm_fp8(P.a.data_ptr(), P.a.stride(0), P.sa.data_ptr(), P.m_alloc, P.b.data_ptr(),
                                         0, 1, P.sb.data_ptr(), P.sb.stride(0), P.sb.stride(1), P.sb.stride(2),
                                         P.gs[0].data_ptr(), 1, P.n, P.k, P.out.data_ptr(), P.n, P.m_alloc, None, None,
                                         flags, torch.cuda.current_stream().cuda_stream)
            assert rc == 0, rc
        for _ in range(3):
            run()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(10):
            run()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 10
        print(f"{name:18s} K={k}: {ms * 1e3:8.1f} us  {P.flops[0] / ms / 1e9:7.1f} TFLOP/s  "
              f"({ms * 1e6 / (k // 128):.0f} ns per k-block)", flush=True)
