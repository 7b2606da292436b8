"""ABBA timing of the headline step (127 grouped GEMMs): PDL modes x (eager, graph)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2508_16584_b200 as tg  # noqa: E402

dev = torch.device("cuda", 0)
P = bench.Problem(torch, "residual_sweep", bench.sweep_problems(), 4096, 7168, 8, dev, seed=1000)
flops = sum(P.flops)
MODES = {"serial": dict(pdl=False), "default": dict(), "overlap": dict(pdl_overlap=True)}


def make_step(kw):
    def step():
        for gs in P.gs:
            tg.grouped_gemm_fp8(P.a, P.sa, P.b, P.sb, gs, out=P.out, **kw)
    return step


def make_graph(fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            fn()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    return g.replay


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


fns = {}
for m, kw in MODES.items():
    st = make_step(kw)
    fns[m + "/eager"] = st
    fns[m + "/graph"] = make_graph(st)
res = {k: [] for k in fns}
keys = list(fns)
for i in range(4):
    for k in (keys if i % 2 == 0 else keys[::-1]):
        res[k].append(timed(fns[k]))
for k, v in res.items():
    print(f"{k:16s}", " ".join(f"{x:.0f}" for x in v), flush=True)
