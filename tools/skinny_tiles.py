import sys, torch
sys.path.insert(0, ".")
import bench, paper_2508_16584_b200 as tg
dev = torch.device("cuda", 0)
hbm = bench._peaks()[0]["hbm_gbs"]
for r in (1, 2, 3, 8):
    P = bench.Problem(torch, "s", [tuple([r] * 8)], 4096, 7168, 8, dev, seed=r)
    gs = P.gs[0]
    nb = P.algorithmic_bytes(P.sizes_list[0])
    for tile in ("pair_n256", "1cta"):
        fn = lambda: tg.grouped_gemm_fp8(P.a, P.sa, P.b, P.sb, gs, out=P.out, tile=tile)
        for _ in range(3): fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20): fn()
        e.record(); torch.cuda.synchronize()
        t = s.elapsed_time(e) / 20
        print(r, tile, round(t * 1e3, 1), "us", round(nb / t / 1e6 / hbm, 3))
