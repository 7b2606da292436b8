"""Same grouped GEMM with B in both layouts (kn = MN-major smem tiles, nk = K-major), ABBA:
python tools/layout_ab.py [shape]  (ds_gateup | ds_down | sq8192)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2508_16584_b200 as tg  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "ds_gateup"
dev = torch.device("cuda", 0)
if name == "ds_gateup":
    sizes, n, k, G = [bench.deepseek_gateup_sizes(0)[1]], 4096, 7168, 32
elif name == "ds_down":
    sizes, n, k, G = [bench.deepseek_gateup_sizes(seed=1)[0]], 7168, 2048, 256
else:
    sizes, n, k, G = [(8192,)], 8192, 8192, 1
probs = {lay: bench.Problem(torch, name, sizes, n, k, G, dev, seed=3, b_layout=lay) for lay in ("kn", "nk")}
res = {lay: [] for lay in probs}
for rnd in range(6):
    for lay in (("kn", "nk") if rnd % 2 == 0 else ("nk", "kn")):
        P = probs[lay]
        f = lambda: tg.grouped_gemm_fp8(P.a, P.sa, P.b, P.sb, P.gs[0], b_layout=lay, out=P.out)  # noqa: E731
        for _ in range(2):
            f()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(10):
            f()
        e.record()
        torch.cuda.synchronize()
        res[lay].append(s.elapsed_time(e) / 10)
for lay, v in res.items():
    ms = sorted(v)[len(v) // 2]
    print(f"{name} B {lay}: {ms * 1e3:8.1f} us  {probs[lay].flops[0] / ms / 1e9:7.1f} TFLOP/s")
