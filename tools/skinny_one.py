"""One skinny launch (8 groups of r rows, N=4096, K=7168) for ncu: python tools/skinny_one.py r tile"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2508_16584_b200 as tg  # noqa: E402

r, tile = int(sys.argv[1]), sys.argv[2]
P = bench.Problem(torch, "s", [tuple([r] * 8)], 4096, 7168, 8, torch.device("cuda", 0), seed=r)
for _ in range(3):
    tg.grouped_gemm_fp8(P.a, P.sa, P.b, P.sb, P.gs[0], out=P.out, tile=tile)
torch.cuda.synchronize()
