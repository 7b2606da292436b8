import sys, torch
sys.path.insert(0, ".")
import bench, paper_2508_16584_b200 as tg
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(1)
N, K, G = 4096, 7168, 8
b = bench._codes(torch, (G, K, N), g, dev); sb = bench._scales(torch, (G, K // 128, N // 128), g, dev)
for m_alloc in (8, 24, 64, 256):
    for r in (1, 3):
        a = bench._codes(torch, (m_alloc, K), g, dev); sa = bench._scales(torch, (m_alloc, K // 128), g, dev)
        gs = torch.tensor([r] * G, dtype=torch.int32, device=dev)
        out = torch.empty((m_alloc, N), dtype=torch.bfloat16, device=dev)
        if r * G > m_alloc: continue
        for tile in ("pair_n256", "1cta"):
            fn = lambda: tg.grouped_gemm_fp8(a, sa, b, sb, gs, out=out, tile=tile)
            for _ in range(3): fn()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(10): fn()
            e.record(); torch.cuda.synchronize()
            print(m_alloc, r, tile, round(s.elapsed_time(e) / 10 * 1e3, 1))
