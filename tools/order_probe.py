"""The headline step timed as CUDA-graph replays and as eager launches, alternately (ABAB...),
to separate the launch method from the order of measurement (power / clock state)."""
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


def step():
    for gs in P.gs:
        tg.grouped_gemm_fp8(P.a, P.sa, P.b, P.sb, gs, out=P.out, pdl_overlap=True)


for _ in range(2):
    step()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    with torch.cuda.graph(g, stream=side):
        step()
torch.cuda.current_stream().wait_stream(side)
torch.cuda.synchronize()


def timed(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return flops / (s.elapsed_time(e) / n * 1e-3) / 1e12


for rnd in range(4):
    for name, fn in (("graph", g.replay), ("eager", step)) if rnd % 2 == 0 else (("eager", step), ("graph", g.replay)):
        print(f"round {rnd} {name}: {timed(fn):.1f} TFLOP/s", flush=True)
