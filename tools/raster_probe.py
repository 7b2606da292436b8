"""DeepSeek-V3 down (or gate+up) with the diagnostics library libtagg_r.so (TAGG_RASTER_EXPERIMENT
build: TAGG_RASTER sets the super-row height of the tile raster).  One process per setting;
prints the launch time.  Under ncu it gives the DRAM bytes per raster."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2508_16584_b200 import _lib  # noqa: E402

L = ctypes.CDLL(str(_lib.PKG / "libtagg_r.so"))
for nm, (r, a) in _lib.SIGNATURES.items():
    if hasattr(L, nm):
        getattr(L, nm).restype, getattr(L, nm).argtypes = r, a
name = sys.argv[1] if len(sys.argv) > 1 else "ds_down"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
if name == "ds_down":
    sizes, n, k, G = [bench.deepseek_gateup_sizes(seed=1)[0]], 7168, 2048, 256
else:
    sizes, n, k, G = [bench.deepseek_gateup_sizes(0)[1]], 4096, 7168, 32
dev = torch.device("cuda", 0)
P = bench.Problem(torch, name, sizes, n, k, G, dev, seed=1)


def run():
    rc = L.tagg_grouped_gemm_fp8(P.a.data_ptr(), P.a.stride(0), P.sa.data_ptr(), P.m_alloc, P.b.data_ptr(), 0, G,
                                 P.sb.data_ptr(), P.sb.stride(0), P.sb.stride(1), P.sb.stride(2), P.gs[0].data_ptr(),
                                 G, n, k, P.out.data_ptr(), n, P.m_alloc, None, None, 0,
                                 torch.cuda.current_stream().cuda_stream)
    assert rc == 0, rc


for _ in range(2):
    run()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
s.record()
for _ in range(iters):
    run()
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / iters
print(f"{name} raster={os.environ.get('TAGG_RASTER', '8')}: {ms * 1e3:.1f} us {P.flops[0] / ms / 1e9:.1f} TFLOP/s")
