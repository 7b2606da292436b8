import sys, ctypes, torch
sys.path.insert(0, ".")
from bench import Problem
from paper_2508_16584_b200 import _lib
path = sys.argv[1]
L = ctypes.CDLL(path)
for nm, (r, a) in _lib.SIGNATURES.items():
    getattr(L, nm).restype, getattr(L, nm).argtypes = r, a
n, k, G = 4096, 3072, 128
P = Problem(torch, "q", [tuple([2048] * 128)], n, k, G, torch.device("cuda", 0), seed=1, b_layout="nk")
for _ in range(3):
    rc = L.tagg_grouped_gemm_fp8(P.a.data_ptr(), P.a.stride(0), P.sa.data_ptr(), P.m_alloc, P.b.data_ptr(), 1, G,
                                 P.sb.data_ptr(), P.sb.stride(0), P.sb.stride(1), P.sb.stride(2), P.gs[0].data_ptr(),
                                 G, n, k, P.out.data_ptr(), n, P.m_alloc, None, None, 0,
                                 torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
