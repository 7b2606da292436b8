"""Is the first timed block of the headline slower?  Times 6 consecutive blocks of 10 steps
(eager launches, then graph replay), with nvidia-smi sampling on or off."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2508_16584_b200 as tg  # noqa: E402

dev = torch.device("cuda", 0)
probs = bench.sweep_problems()
ops = bench.headline_operands(bench.HEADLINE_SEED, max(sum(s) for s in probs))
P = bench.Problem(torch, "sweep", probs, 4096, 7168, 8, dev, seed=0, host=ops)
flops = sum(P.flops)


def step():
    for gs in P.gs:
        tg.grouped_gemm_fp8(P.a, P.sa, P.b, P.sb, gs, out=P.out, pdl_overlap=True)


def block(fn, n=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return flops * n / (s.elapsed_time(e) * 1e-3) / 1e12


for _ in range(3):
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
for sampler in (False, True, False):
    ctx = bench.ClockSampler(0) if sampler else None
    if ctx:
        ctx.__enter__()
    e = [block(step) for _ in range(4)]
    gr = [block(g.replay) for _ in range(4)]
    e2 = [block(step) for _ in range(2)]
    if ctx:
        ctx.__exit__(None, None, None)
        print("clocks", ctx.summary())
    print(f"sampler={sampler} eager", " ".join(f"{x:.0f}" for x in e), "| graph", " ".join(f"{x:.0f}" for x in gr),
          "| eager", " ".join(f"{x:.0f}" for x in e2), flush=True)
