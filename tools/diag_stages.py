"""Stage-count sensitivity of the GEMM kernel (flags bits 12-15 cap the ring depth)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2508_16584_b200._lib import lib
from bench import Problem, deepseek_gateup_sizes

dev = torch.device("cuda", 0)
cases = [("sweep_r64", [tuple(128 * g + 64 for g in range(8))], 4096, 7168, 8),
         ("ds_gateup", [deepseek_gateup_sizes(0)[1]], 4096, 7168, 32),
         ("ds_down", [deepseek_gateup_sizes(1)[0]], 7168, 2048, 256)]
for name, sizes, n, k, G in cases:
    P = Problem(torch, name, sizes, n, k, G, dev, seed=1)
    for rep in range(2):
        for cap in (2, 3, 4, 0):
            flags = 16 | (cap << 12)
            def run():
                rc = lib().tagg_grouped_gemm_fp8(P.a.data_ptr(), P.a.stride(0), P.sa.data_ptr(), P.m_alloc,
                                                 P.b.data_ptr(), 0, G, P.sb.data_ptr(), P.sb.stride(0), P.sb.stride(1),
                                                 P.sb.stride(2), P.gs[0].data_ptr(), G, n, k, P.out.data_ptr(), n,
                                                 P.m_alloc, None, None, flags, torch.cuda.current_stream().cuda_stream)
                assert rc == 0, rc
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(10):
                run()
            e.record()
            torch.cuda.synchronize()
            ms = s.elapsed_time(e) / 10
            print(f"{name:10s} stages_cap={cap} {ms*1e3:8.1f} us {P.flops[0]/ms/1e9:8.1f} TFLOP/s", flush=True)
    del P
    torch.cuda.empty_cache()
