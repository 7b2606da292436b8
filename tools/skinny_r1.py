import sys, torch
sys.path.insert(0, ".")
import bench, paper_2508_16584_b200 as tg
dev = torch.device("cuda", 0)
for rep in range(3):
    for r in (1, 2, 3):
        P = bench.Problem(torch, "s", [tuple([r] * 8)], 4096, 7168, 8, dev, seed=r)
        gs = P.gs[0]
        for tile in (None, "pair_n256", "1cta"):
            fn = lambda: tg.grouped_gemm_fp8(P.a, P.sa, P.b, P.sb, gs, out=P.out, tile=tile)
            for _ in range(3): fn()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(10): fn()
            e.record(); torch.cuda.synchronize()
            print(rep, r, tile, round(s.elapsed_time(e) / 10 * 1e3, 1))
        del P
