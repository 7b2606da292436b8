"""Graph replay vs eager launches of the headline step, alternated over many short blocks
(5 steps, 1 warm-up: the bench's comparison blocks), with and without programmatic dependent
launch, to tell the launch method from the power state."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2508_16584_b200 as tg  # noqa: E402

dev = torch.device("cuda", 0)
probs = bench.sweep_problems()
ops = bench.headline_operands(bench.HEADLINE_SEED, max(sum(s) for s in probs))
P = bench.Problem(torch, "residual_sweep", probs, 4096, 7168, 8, dev, seed=bench.HEADLINE_SEED, host=ops)
flops = sum(P.flops)


def make(pdl):
    def step():
        for gs in P.gs:
            tg.grouped_gemm_fp8(P.a, P.sa, P.b, P.sb, gs, out=P.out, pdl_overlap=pdl)
    return step


def graph_of(fn):
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
    return g


def timed(fn, n=5, w=1):
    for _ in range(w):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return flops / (s.elapsed_time(e) / n * 1e-3) / 1e12


arms = {"eager_pdl": make(True), "eager_nopdl": make(False)}
arms["graph_pdl"] = graph_of(arms["eager_pdl"]).replay
arms["graph_nopdl"] = graph_of(arms["eager_nopdl"]).replay
res = {k: [] for k in arms}
names = list(arms)
for rnd in range(8):
    order = names if rnd % 2 == 0 else names[::-1]
    for k in order:
        res[k].append(timed(arms[k]))
for k, v in res.items():
    v = sorted(v)
    print(f"{k:12s} median {v[len(v) // 2]:7.1f}  min {v[0]:7.1f}  max {v[-1]:7.1f} TFLOP/s")
