"""ncu subject for the HBM-bound launches (north star: "achieved HBM GB/s for skinny or
residual-dominated groups"): the skinny sweep's padding-free GEMM at r = 1 / 8 / 64 rows per
group, and the pad + padded baseline's K2 pad / GEMM / K3 unpad at r = 1 and 64; "padbig" runs
the baseline at DeepSeek-V3 down size, where K2 / K3 move 0.6 / 7.5 GB.  8 groups,
N=4096, K=7168, per-expert B (235 MB).  Usage: prof_skinny.py {free,padded} r.  Runs 2 warm-up
calls, a sync, then the profiled call (ncu -s skips the warm-up launches)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2508_16584_b200 as tg  # noqa: E402

mode, r = sys.argv[1], int(sys.argv[2])
dev = torch.device("cuda", 0)
if mode == "padbig":  # the pad / unpad kernels at DeepSeek-V3 down size (262,144 rows, K=2048, N=7168)
    counts, _ = bench.deepseek_gateup_sizes(seed=1)
    P = bench.Problem(torch, "dsdown", [counts], 7168, 2048, 256, dev, seed=1)
    mode = "padded"
else:
    P = bench.Problem(torch, f"skinny_r{r}", [tuple([r] * 8)], 4096, 7168, 8, dev, seed=r)
gs = P.gs[0]
ws = tg.PaddedWorkspace(P.m_alloc, P.G, P.k, P.n, dev)


def call():
    if mode == "free":
        tg.grouped_gemm_fp8(P.a, P.sa, P.b, P.sb, gs, out=P.out)
    else:
        tg.padded_grouped_gemm_fp8(P.a, P.sa, P.b, P.sb, gs, ws, out=P.out)


for _ in range(2):
    call()
torch.cuda.synchronize()
call()
torch.cuda.synchronize()
