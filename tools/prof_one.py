"""One configurable launch set for ncu captures: python tools/prof_one.py <name> <flags> [iters]."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2508_16584_b200._lib import lib
from bench import Problem

name, flags = sys.argv[1], int(sys.argv[2])
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
shapes = {"sq8192": ([(8192,)], 8192, 8192, 1), "sweep_r64": ([tuple(128 * g + 64 for g in range(8))], 4096, 7168, 8),
          "ds_gateup": (None, 4096, 7168, 32), "ds_down": ("down", 7168, 2048, 256)}
sizes, n, k, G = shapes[name]
if sizes is None:
    from bench import deepseek_gateup_sizes
    sizes = [deepseek_gateup_sizes(0)[1]]
elif sizes == "down":
    from bench import deepseek_gateup_sizes
    sizes = [deepseek_gateup_sizes(seed=1)[0]]
P = Problem(torch, name, sizes, n, k, G, torch.device("cuda", 0), seed=1)
for _ in range(iters):
    rc = lib().tagg_grouped_gemm_fp8(P.a.data_ptr(), P.a.stride(0), P.sa.data_ptr(), P.m_alloc, P.b.data_ptr(), 0, G,
                                     P.sb.data_ptr(), P.sb.stride(0), P.sb.stride(1), P.sb.stride(2), P.gs[0].data_ptr(),
                                     G, n, k, P.out.data_ptr(), n, P.m_alloc, None, None, flags,
                                     torch.cuda.current_stream().cuda_stream)
    assert rc == 0
torch.cuda.synchronize()
print("done", name, flags)
