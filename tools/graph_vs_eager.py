"""ABBA timing of the headline step (127 grouped GEMMs) as plain launches vs CUDA-graph replay."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2508_16584_b200 as tg  # noqa: E402

dev = torch.device("cuda", 0)
P = bench.Problem(torch, "residual_sweep", bench.sweep_problems(), 4096, 7168, 8, dev, seed=1000)
flops = sum(P.flops)


def step():
    for gs in P.gs:
        tg.grouped_gemm_fp8(P.a, P.sa, P.b, P.sb, gs, out=P.out)


for _ in range(3):
    step()
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    with torch.cuda.graph(graph, stream=side):
        step()
torch.cuda.current_stream().wait_stream(side)
torch.cuda.synchronize()


def timed(fn, n=5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return flops / (s.elapsed_time(e) / n * 1e-3) / 1e12


res = {"graph": [], "eager": []}
for i in range(4):
    order = ("graph", "eager") if i % 2 == 0 else ("eager", "graph")
    for k in order:
        res[k].append(timed(graph.replay if k == "graph" else step))
for k, v in res.items():
    print(k, " ".join(f"{x:.0f}" for x in v))
