"""One launch of a configurable grouped GEMM for ncu stage-count probes:
python tools/stage_probe.py <G> <rows_total> <N> <K> <flags> [zipf|uniform] [iters]"""
import sys

import torch

sys.path.insert(0, ".")
from bench import Problem, deepseek_gateup_sizes  # noqa: E402
from paper_2508_16584_b200._lib import lib  # noqa: E402

G, rows, n, k, flags = (int(x) for x in sys.argv[1:6])
mode = sys.argv[6] if len(sys.argv) > 6 else "uniform"
iters = int(sys.argv[7]) if len(sys.argv) > 7 else 2
if mode == "zipf":
    sizes = [int(x) for x in deepseek_gateup_sizes(seed=1, tokens=rows // 8, experts=G, local=G)[0]]
else:
    sizes = [rows // G] * G
P = Problem(torch, "probe", [tuple(sizes)], n, k, G, torch.device("cuda", 0), seed=1)
for _ in range(iters):
    rc = lib().tagg_grouped_gemm_fp8(P.a.data_ptr(), P.a.stride(0), P.sa.data_ptr(), P.m_alloc, P.b.data_ptr(), 0, G,
                                     P.sb.data_ptr(), P.sb.stride(0), P.sb.stride(1), P.sb.stride(2),
                                     P.gs[0].data_ptr(), G, n, k, P.out.data_ptr(), n, P.m_alloc, None, None, flags,
                                     torch.cuda.current_stream().cuda_stream)
    assert rc == 0, rc
torch.cuda.synchronize()
