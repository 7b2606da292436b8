"""A/B timing of libtagg builds' weight gradient (K6) on the DeepSeek-V3 gate+up shapes (ABBA rounds):
python tools/wg_ab.py A.so B.so ...   -> TFLOP/s per recipe (per-column dY, 128x128 dY, MXFP8)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2508_16584_b200 as tg  # noqa: E402
from bench import deepseek_gateup_sizes  # noqa: E402
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
_, sizes = deepseek_gateup_sizes(seed=0)
sizes = [int(s) for s in sizes]
m, k, n = sum(sizes), 7168, 4096
gen = torch.Generator(device=dev).manual_seed(5)
gs = torch.tensor(sizes, dtype=torch.int32, device=dev)
x = torch.randn((m, k), device=dev, generator=gen).to(torch.bfloat16)
dy = torch.randn((m, n), device=dev, generator=gen).to(torch.bfloat16)
xc, xs = tg.quantize_col_blocks(x, gs)
dc, ds = tg.quantize_col_blocks(dy, gs)
dcb, dsb = tg.quantize_col_blocks(dy, gs, block_cols=128)
xm, _, xf = tg.quantize_col_blocks_mx(x, gs)
dm, _, df = tg.quantize_col_blocks_mx(dy, gs)
dw = torch.empty((len(sizes), k, n), dtype=torch.bfloat16, device=dev)
flops = 2.0 * m * k * n
st = torch.cuda.current_stream().cuda_stream
G = len(sizes)
recipes = {
    "per_column": lambda lib: lib.tagg_wgrad_fp8_ex(xc.data_ptr(), xs.data_ptr(), dc.data_ptr(), ds.data_ptr(), m,
                                                    gs.data_ptr(), G, k, n, dw.data_ptr(), 0, st),
    "dy_block128": lambda lib: lib.tagg_wgrad_fp8_ex(xc.data_ptr(), xs.data_ptr(), dcb.data_ptr(), dsb.data_ptr(), m,
                                                     gs.data_ptr(), G, k, n, dw.data_ptr(), 1, st),
    "mxfp8": lambda lib: lib.tagg_wgrad_fp8_mx(xm.data_ptr(), xf.data_ptr(), dm.data_ptr(), df.data_ptr(), m,
                                               gs.data_ptr(), G, k, n, dw.data_ptr(), st),
}
for name, call in recipes.items():
    times = {p: [] for p in libs}
    for rnd in range(6):
        order = list(range(len(libs))) if rnd % 2 == 0 else list(range(len(libs)))[::-1]
        for i in order:
            assert call(L[i]) == 0
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(5):
                call(L[i])
            e.record()
            torch.cuda.synchronize()
            times[libs[i]].append(s.elapsed_time(e) / 5)
    for p in libs:
        ms = sorted(times[p])[3]
        print(f"{name:12s} {p.rsplit('/', 1)[-1]:18s} {ms:7.3f} ms {flops / ms / 1e9:7.0f} TFLOP/s")
