"""Small invocations of every product kernel, for compute-sanitizer (memcheck / racecheck /
synccheck): python tools/sanitize.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2508_16584_b200 as tg  # noqa: E402
from oracle import fp8 as ofp8  # noqa: E402

dev = torch.device("cuda", 0)
sizes = (1, 67, 0, 128, 255, 300)
n, k = 384, 640
m = sum(sizes)
ac, asc, _, _ = ofp8.random_operands(m, 64, k, 3)
bs = [ofp8.random_operands(1, n, k, 10 + g) for g in range(len(sizes))]
bc = np.stack([b[2] for b in bs])
bsc = np.stack([b[3] for b in bs])
a, sa = torch.from_numpy(ac).to(dev), torch.from_numpy(asc).to(dev)
b, sb = torch.from_numpy(bc).to(dev), torch.from_numpy(bsc).to(dev)
gs = torch.tensor(sizes, dtype=torch.int32, device=dev)
PART = os.environ.get("SANITIZE_PART", "all")  # diagnostics: run one piece (base / bidx / flag / overlap)
if PART in ("all", "base"):
    for tile in ("pair_n256", "pair_n128", "1cta"):
        for exact in (False, True):
            tg.grouped_gemm_fp8(a, sa, b, sb, gs, tile=tile, exact_promotion=exact)
# exact-size output: any store past sum(M_g) would be out of bounds
out = torch.empty((m, n), dtype=torch.bfloat16, device=dev)
tg.grouped_gemm_fp8(a[:m].contiguous(), sa[:m].contiguous(), b, sb, gs, out=out)
ws = tg.PaddedWorkspace(m, len(sizes), k, n, dev)
tg.padded_grouped_gemm_fp8(a, sa, b, sb, gs, ws)
x = torch.randn((100, k), device=dev)
eids = torch.randint(0, 6, (100, 4), device=dev, dtype=torch.int32)
d = tg.quantize_dispatch(x, eids, 6)
tg.quantize_blocks(torch.randn((2, 256, 384), device=dev))
xc, xs = tg.quantize_col_blocks(torch.randn((m, 256), device=dev), gs)
dyc, dys = tg.quantize_col_blocks(torch.randn((m, 128), device=dev), gs)
tg.wgrad_fp8(xc, xs, dyc, dys, gs)
dbc, dbs = tg.quantize_col_blocks(torch.randn((m, 128), device=dev), gs, block_cols=128)
tg.wgrad_fp8(xc, xs, dbc, dbs, gs, dy_block128=True)
# MXFP8 weight gradient: power-of-two quantizer with factor blocks, block-scaled MMA
xm, _, xf = tg.quantize_col_blocks_mx(torch.randn((m, 256), device=dev), gs)
dm, _, df = tg.quantize_col_blocks_mx(torch.randn((m, 256), device=dev), gs)
tg.wgrad_fp8_mx(xm, xf, dm, df, gs)
# bf16 column quantizer (persistent kernel), plain and gathered
xb = torch.randn((m, 512), device=dev).to(torch.bfloat16)
tg.quantize_col_blocks(xb, gs)
idx = torch.randperm(m, device=dev).to(torch.int32)
tg.quantize_col_blocks(xb, gs, index=idx, row_weights=torch.rand(m, device=dev))
# groups sharing experts (b_index), the device error flag, a PDL-overlap chain into one output
bi = torch.tensor([1, 0, 2, 1, 5, 3], dtype=torch.int32, device=dev)
if PART in ("all", "bidx"):
    tg.grouped_gemm_fp8(a, sa, b, sb, gs, b_index=bi, check=True)
if PART in ("all", "flag"):
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    tg.grouped_gemm_fp8(a, sa, b, sb, torch.tensor([5000, 1, 0, 0, 0, 0], dtype=torch.int32, device=dev),
                        err_flag=flag)
if PART in ("all", "overlap"):
    for _ in range(3):
        tg.grouped_gemm_fp8(a, sa, b, sb, gs, pdl_overlap=True)
if PART == "overlap_sync":  # the same launches with a device sync between them: no grid overlap
    for _ in range(3):
        tg.grouped_gemm_fp8(a, sa, b, sb, gs, pdl_overlap=True)
        torch.cuda.synchronize()
from paper_2508_16584_b200 import moe  # noqa: E402

h = torch.randn((m + 40, 512), device=dev).to(torch.bfloat16)
hq, hs = moe.swiglu_quantize(h, gs)
cc = torch.randn((400, 256), device=dev).to(torch.bfloat16)
moe.combine(cc, d.dest_rows, torch.rand((100, 4), device=dev))
torch.cuda.synchronize()
print("sanitize workload done")
