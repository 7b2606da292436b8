"""Pipeline trace of the wgrad kernel (K6) at the DeepSeek-V3 gate+up shapes; needs
libtagg_trace.so (`make -C paper_2508_16584_b200/csrc trace`).  Same event layout as tools/trace.py."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2508_16584_b200 as tg  # noqa: E402
from bench import deepseek_gateup_sizes  # noqa: E402
from paper_2508_16584_b200 import _lib  # noqa: E402

import os
L = ctypes.CDLL(os.environ.get("TAGG_TRACE_LIB", str(_lib.PKG / "libtagg_trace.so")))
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
xc, xs = tg.quantize_col_blocks(torch.randn((m, k), device=dev, generator=gen).to(torch.bfloat16), gs)
dc, ds = tg.quantize_col_blocks(torch.randn((m, n), device=dev, generator=gen).to(torch.bfloat16), gs)
dw = torch.empty((len(sizes), k, n), dtype=torch.bfloat16, device=dev)
buf = torch.zeros((2, 10, 1024), dtype=torch.int64, device=dev)


def run():
    rc = L.tagg_wgrad_fp8(xc.data_ptr(), xs.data_ptr(), dc.data_ptr(), ds.data_ptr(), m, gs.data_ptr(), len(sizes), k,
                          n, dw.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert rc == 0, rc


run()
L.tagg_debug_trace(ctypes.c_void_p(buf.data_ptr()))
run()
torch.cuda.synchronize()
L.tagg_debug_trace(None)
t = buf[0].cpu().numpy().astype(np.float64)
lo, hi = 40, 600


def d(a, b, sh=0):
    return t[EV.index(a), lo:hi] - t[EV.index(b), lo - sh:hi - sh]


rows = {
    "mma issue period": d("mma_issued", "mma_issued", 1),
    "mma wait tempty (after prev issue)": d("mma_tempty", "mma_issued", 1),
    "mma wait full": d("mma_full", "mma_tempty"),
    "prod empty period": d("prod_empty", "prod_empty", 1),
    "promo sfull wait (after prev done)": d("promo_sfull", "promo_done", 1),
    "promo tfull wait (after sfull)": d("promo_full", "promo_sfull"),
    "promo full->freed (drain)": d("promo_freed", "promo_full"),
    "promo freed->done (math)": d("promo_done", "promo_freed"),
    "mma issue -> promo sees full": d("promo_full", "mma_issued"),
}
print(f"--- wgrad DSv3 gate+up, k-block iterations [{lo},{hi}) of CTA 0, clk (median / p10 / p90)")
for name, v in rows.items():
    print(f"  {name:38s} {np.median(v):8.0f} {np.percentile(v, 10):8.0f} {np.percentile(v, 90):8.0f}")
es, ee = t[EV.index("epi_start")], t[EV.index("epi_end")]
nt = int((ee > 0).sum())
if nt > 1:
    print(f"  epilogue per tile (clk): median {np.median(ee[:nt] - es[:nt]):.0f} over {nt} tiles")
    ts = es[1:nt] - es[:nt - 1]
    print(f"  tile period (clk): median {np.median(ts):.0f}")
