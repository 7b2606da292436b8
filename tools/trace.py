"""Pipeline trace of the GEMM kernel (diagnostics; needs libtagg_trace.so from `make -C
paper_2508_16584_b200/csrc trace`).  Stamps clock64 at 8 events per k-block in CTAs 0/1
and prints steady-state intervals: who waits on whom."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from bench import Problem  # noqa: E402
from paper_2508_16584_b200 import _lib  # noqa: E402

L = ctypes.CDLL(str(_lib.PKG / "libtagg_trace.so"))
for name, (res, args) in _lib.SIGNATURES.items():
    fn = getattr(L, name)
    fn.restype, fn.argtypes = res, args

EV = ["mma_tempty", "mma_full", "mma_issued", "prod_empty", "promo_full", "promo_freed", "promo_done", "promo2_full",
      "epi_start", "epi_end", "epi_bar1", "epi_stores"]
dev = torch.device("cuda", 0)
buf = torch.zeros((2, len(EV), 1024), dtype=torch.int64, device=dev)


def run(P, flags, G):
    rc = L.tagg_grouped_gemm_fp8(P.a.data_ptr(), P.a.stride(0), P.sa.data_ptr(), P.m_alloc, P.b.data_ptr(), 0, G,
                                 P.sb.data_ptr(), P.sb.stride(0), P.sb.stride(1), P.sb.stride(2), P.gs[0].data_ptr(),
                                 G, P.n, P.k, P.out.data_ptr(), P.n, P.m_alloc, None, None, flags,
                                 torch.cuda.current_stream().cuda_stream)
    assert rc == 0, rc


def report(tr, lo, hi, label):
    t = tr[0].astype(np.float64)  # CTA 0 (leader)
    d = lambda a, b, sh=0: (t[EV.index(a), lo:hi] - t[EV.index(b), lo - sh:hi - sh])  # noqa: E731
    rows = {
        "mma issue period": d("mma_issued", "mma_issued", 1),
        "mma wait full (after prev issue)": d("mma_full", "mma_issued", 1),
        "mma wait tempty (after full)": d("mma_tempty", "mma_full"),
        "mma tempty seen->issued": d("mma_issued", "mma_tempty"),
        "mma issue->promo sees full": d("promo_full", "mma_issued"),
        "promo wait full (after prev done)": d("promo_full", "promo_done", 1),
        "promo full->freed (drain)": d("promo_freed", "promo_full"),
        "promo freed->done (math tail)": d("promo_done", "promo_freed"),
        "promo freed(i-2)->mma tempty(i)": d("mma_tempty", "promo_freed", 2),
        "prod empty period": d("prod_empty", "prod_empty", 1),
    }
    print(f"--- {label}: k-block iterations [{lo},{hi}) of CTA 0, clk (median / p10 / p90)")
    for k, v in rows.items():
        print(f"  {k:38s} {np.median(v):8.0f} {np.percentile(v, 10):8.0f} {np.percentile(v, 90):8.0f}")
    es, ee = t[EV.index("epi_start")], t[EV.index("epi_end")]
    nt = int((ee > 0).sum())
    if nt > 1:
        dur = ee[:nt] - es[:nt]
        print(f"  epilogue per tile (clk): median {np.median(dur):.0f} over {nt} tiles")
        b1, st = t[EV.index("epi_bar1")][:nt], t[EV.index("epi_stores")][:nt]
        if (b1 > 0).all():
            print(f"    start->barrier {np.median(b1 - es[:nt]):.0f} | barrier->staged {np.median(st - b1):.0f} | "
                  f"store issue {np.median(ee[:nt] - st):.0f}")
    t1 = tr[1].astype(np.float64)
    v = t1[EV.index("promo_full"), lo:hi] - t1[EV.index("promo_full"), lo - 1:hi - 1]
    print(f"  {'CTA1 promo full period':38s} {np.median(v):8.0f}")


cases = [("sq8192", [(8192,)], 8192, 8192, 1), ("sweep_r64", [tuple(128 * g + 64 for g in range(8))], 4096, 7168, 8)]
if len(sys.argv) > 1 and sys.argv[1] == "ds":
    from bench import deepseek_gateup_sizes
    cases = [("ds", [tuple(int(x) for x in deepseek_gateup_sizes(0)[1])], 4096, 7168, 32)]
if len(sys.argv) > 1 and sys.argv[1] == "dsdown":
    from bench import deepseek_gateup_sizes
    cases = [("dsdown", [tuple(int(x) for x in deepseek_gateup_sizes(seed=1)[0])], 7168, 2048, 256)]
if len(sys.argv) > 1 and sys.argv[1] == "qdown":
    cases = [("qdown", [tuple([2048] * 128)], 4096, 1536, 128)]
if len(sys.argv) > 1 and sys.argv[1] == "longk":
    # one pair tile per cluster, 256 k-blocks per tile: no tile transitions in the window
    cases = [("longk", [(256 * 74,)], 256, 8192, 1)]
for name, sizes, n, k, G in cases:
    P = Problem(torch, name, sizes, n, k, G, dev, seed=1)
    modes = [("full", 0), ("noload", 256), ("nomath", 1024), ("noprom", 512), ("neither", 256 | 512)]
    for label, flags in modes:
        L.tagg_debug_trace(None)
        run(P, flags, G)
        L.tagg_debug_trace(ctypes.c_void_p(buf.data_ptr()))
        buf.zero_()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        run(P, flags, G)
        ev1.record()
        torch.cuda.synchronize()
        t0 = buf[0].cpu().numpy().astype(np.float64)
        iss = t0[EV.index("mma_issued")]
        nz = iss[iss > 0]
        if len(nz) > 10:
            # CTA 0's issue stamps span (n-1) periods: clk over the launch's wall time ~ the SM clock
            span = nz[-1] - nz[0]
            print(f"  [{label}] launch {ev0.elapsed_time(ev1) * 1e3:.0f} us; CTA0 issue span {span:.0f} clk over "
                  f"{len(nz)} k-blocks -> >= {span / (ev0.elapsed_time(ev1) * 1e3):.0f} MHz")
        L.tagg_debug_trace(None)
        import os
        win = os.environ.get("TRACE_WINDOW")
        lo, hi = (int(v) for v in win.split(",")) if win else (
            8 if name == "longk" else 64, {"sq8192": 880, "sweep_r64": 270, "longk": 60, "qdown": 600, "ds": 1000,
                                           "dsdown": 1000}[name])
        report(buf.cpu().numpy(), lo, hi, f"{name} {label} [{lo},{hi})")
    del P
