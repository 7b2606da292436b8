"""Pipeline trace of the MXFP8 weight gradient (TAGG_WGRAD_MX) at the DeepSeek-V3 gate+up shapes
(libtagg_trace.so).  Per k-block of CTA 0: MMA full / sfready / tempty waits and issue; per tile:
accumulator full seen by the epilogue warps, freed, epilogue start / end."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2508_16584_b200 as tg  # noqa: E402
from bench import deepseek_gateup_sizes  # noqa: E402
from paper_2508_16584_b200 import _lib  # noqa: E402

L = ctypes.CDLL(str(_lib.PKG / "libtagg_trace.so"))
for name, (res, args) in _lib.SIGNATURES.items():
    if hasattr(L, name):
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
EV = ["mma_tempty", "mma_full", "mma_issued", "prod_empty", "promo_full", "promo_freed", "promo_done", "promo_sfull",
      "epi_start", "epi_end"]
dev = torch.device("cuda", 0)
_, sizes = deepseek_gateup_sizes(seed=0)
sizes = [int(s) for s in sizes]
m, k, n = sum(sizes), 7168, 4096
gen = torch.Generator(device=dev).manual_seed(5)
gs = torch.tensor(sizes, dtype=torch.int32, device=dev)
xc, _, xs = tg.quantize_col_blocks_mx(torch.randn((m, k), device=dev, generator=gen).to(torch.bfloat16), gs)
dc, _, ds = tg.quantize_col_blocks_mx(torch.randn((m, n), device=dev, generator=gen).to(torch.bfloat16), gs)
dw = torch.empty((len(sizes), k, n), dtype=torch.bfloat16, device=dev)
buf = torch.zeros((2, 10, 1024), dtype=torch.int64, device=dev)


def run():
    rc = L.tagg_wgrad_fp8_mx(xc.data_ptr(), xs.data_ptr(), dc.data_ptr(), ds.data_ptr(), m, gs.data_ptr(), len(sizes),
                             k, n, dw.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert rc == 0, rc


run()
L.tagg_debug_trace(ctypes.c_void_p(buf.data_ptr()))
run()
torch.cuda.synchronize()
L.tagg_debug_trace(None)
t = buf[0].cpu().numpy().astype(np.float64)
E = {e: t[i] for i, e in enumerate(EV)}
t0 = E["mma_full"][0]
print("k-block: full / (unused) / tempty / issued (clk from the first full), then tile events")
for i in range(40):
    print(f"  kb {i:3d}: {E['mma_full'][i] - t0:9.0f} {E['promo_sfull'][i] - t0:9.0f} {E['mma_tempty'][i] - t0:9.0f} "
          f"{E['mma_issued'][i] - t0:9.0f}")
for i in range(8):
    print(f"  tile {i}: acc full seen {E['promo_full'][i] - t0:9.0f}  freed {E['promo_freed'][i] - t0:9.0f}  "
          f"epi {E['epi_start'][i] - t0:9.0f} -> {E['epi_end'][i] - t0:9.0f}")
lo, hi = 40, 600


def d(a, b, sh=0):
    return E[a][lo:hi] - E[b][lo - sh:hi - sh]


print(f"--- medians over k-blocks [{lo},{hi}) of CTA 0 (clk): median / p10 / p90")
for name, v in {"mma issue period": d("mma_issued", "mma_issued", 1),
                "mma full seen -> issued": d("mma_issued", "mma_full"),
                "prod empty period": d("prod_empty", "prod_empty", 1),
                "prod empty -> mma full (load latency)": d("mma_full", "prod_empty"),
                "mma issued -> next full seen": d("mma_full", "mma_issued", 1)}.items():
    print(f"  {name:40s} {np.median(v):8.0f} {np.percentile(v, 10):8.0f} {np.percentile(v, 90):8.0f}")
