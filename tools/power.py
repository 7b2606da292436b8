"""Clock / power under sustained load: runs each workload back to back for ~2 s while
nvidia-smi samples SM clock, power and throttle reasons every 50 ms.

python tools/power.py
"""
import subprocess
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import Problem, deepseek_gateup_sizes  # noqa: E402
from paper_2508_16584_b200._lib import lib  # noqa: E402

dev = torch.device("cuda", 0)


def sample(fn, label, secs=2.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    q = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    n = 0
    s.record()
    while time.time() - t0 < secs:
        for _ in range(10):
            fn()
        n += 10
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    q.terminate()
    out = q.communicate()[0].strip().splitlines()
    ms = s.elapsed_time(e) / n
    vals = [line.split(", ") for line in out if line.count(",") == 2]
    clk = sorted(float(v[0]) for v in vals)
    pw = sorted(float(v[1]) for v in vals)
    reasons = sorted({v[2] for v in vals})
    mid = len(clk) // 2
    return ms, clk[mid] if clk else 0, pw[mid] if pw else 0, reasons


def gemm(name, sizes, n, k, G, bl="kn"):
    P = Problem(torch, name, [sizes], n, k, G, dev, seed=1, b_layout=bl)
    layout = 0 if bl == "kn" else 1

    def run():
        rc = lib().tagg_grouped_gemm_fp8(P.a.data_ptr(), P.a.stride(0), P.sa.data_ptr(), P.m_alloc, P.b.data_ptr(),
                                         layout, G, P.sb.data_ptr(), P.sb.stride(0), P.sb.stride(1), P.sb.stride(2),
                                         P.gs[0].data_ptr(), G, n, k, P.out.data_ptr(), n, P.m_alloc, None, None, 0,
                                         torch.cuda.current_stream().cuda_stream)
        assert rc == 0, rc
    return run, P.flops[0], P


for name, sizes, n, k, G in [("sq8192", (8192,), 8192, 8192, 1),
                             ("ds_gateup", tuple(int(x) for x in deepseek_gateup_sizes(0)[1]), 4096, 7168, 32)]:
    fn, flops, P = gemm(name, sizes, n, k, G)
    ms, clk, pw, rs = sample(fn, name)
    print(f"{name:12s} {flops / ms / 1e9:8.1f} TFLOP/s  sm {clk:6.0f} MHz  {pw:6.1f} W  reasons {rs}", flush=True)
    del P
a = torch.randn(8192, 8192, device=dev).to(torch.float8_e4m3fn)
b = torch.randn(8192, 8192, device=dev).to(torch.float8_e4m3fn).t()
one = torch.ones((), device=dev)
ms, clk, pw, rs = sample(lambda: torch._scaled_mm(a, b, one, one, out_dtype=torch.bfloat16), "cublas")
print(f"{'cublas fp8':12s} {2 * 8192 ** 3 / ms / 1e9:8.1f} TFLOP/s  sm {clk:6.0f} MHz  {pw:6.1f} W  reasons {rs}")
