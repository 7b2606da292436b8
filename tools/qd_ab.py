"""A/B timing of libtagg builds' quantize + dispatch (route plan + K5) at the bench shape
(32768 tokens x 7168 bf16, top-8 of 256 experts), ABBA rounds:  python tools/qd_ab.py A.so B.so ..."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2508_16584_b200 as tg  # noqa: E402
from paper_2508_16584_b200 import _lib  # noqa: E402

libs = sys.argv[1:]
L = []
for path in libs:
    lib = ctypes.CDLL(path)
    for nm, (r, a) in _lib.SIGNATURES.items():
        if hasattr(lib, nm):
            getattr(lib, nm).restype, getattr(lib, nm).argtypes = r, a
    L.append(lib)
dev = torch.device("cuda", 0)
tokens, k, topk, experts = 32768, 7168, 8, 256
gen = torch.Generator(device=dev).manual_seed(3)
x = torch.randn((tokens, k), device=dev, generator=gen).to(torch.bfloat16)
eids = torch.topk(torch.randn((tokens, experts), device=dev, generator=gen), topk, dim=1).indices.to(torch.int32)
kb = -(-k // 128)
rows = tokens * topk
nbytes = tokens * k * 2 + rows * 4 + rows * (k + 4 * kb) + rows * 4 + experts * 4
peak = bench._peaks()[0]["hbm_gbs"]
ref = None
times = {p: [] for p in libs}
for rnd in range(6):
    order = list(range(len(libs))) if rnd % 2 == 0 else list(range(len(libs)))[::-1]
    for i in order:
        _lib._lib = L[i]  # the package's entry points call through this library
        out = tg.quantize_dispatch(x, eids, experts)
        if rnd == 0:
            codes = out.a_codes.clone()
            if ref is None:
                ref = codes
            else:
                assert torch.equal(ref, codes), f"{libs[i]}: codes differ from {libs[0]}"
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            tg.quantize_dispatch(x, eids, experts)
        e.record()
        torch.cuda.synchronize()
        times[libs[i]].append(s.elapsed_time(e) / 10)
for p in libs:
    ms = sorted(times[p])[3]
    print(f"{p.rsplit('/', 1)[-1]:18s} {ms:7.3f} ms {nbytes / ms / 1e6:7.0f} GB/s {nbytes / ms / 1e6 / peak:6.1%} of HBM")
