"""Column-block quantizer timing on the MoE backward shapes (262144 grouped rows, 256 groups)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2508_16584_b200 as tg  # noqa: E402

dev = torch.device("cuda", 0)
gs = torch.full((256,), 1024, dtype=torch.int32, device=dev)
for cols in (2048, 4096, 7168):
    x = torch.randn((262144, cols), device=dev).to(torch.bfloat16)
    for label, fn in (("fp32 scales", lambda: tg.quantize_col_blocks(x, gs)),
                      ("MXFP8", lambda: tg.quantize_col_blocks_mx(x, gs))):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            fn()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 5
        nbytes = x.numel() * 3  # bf16 read once + codes written (the scales are small)
        print(cols, label, round(ms, 3), "ms", round(nbytes / ms / 1e9, 2), "TB/s (one read + codes)")
