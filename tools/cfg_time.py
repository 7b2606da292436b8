"""Time the grouped GEMM on the BASELINE config shapes (bench.run_extra's problems), one line
per config: ms per launch, TFLOP/s, % of the FP8 peak.  Env knobs (TAGG_L2_HINT, ...) are read
by libtagg.so, so each setting runs in its own process.  Usage: cfg_time.py [names...] [--iters N]."""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2508_16584_b200 as tg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("names", nargs="*")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--exact", action="store_true")
ap.add_argument("--tag", default="")
ap.add_argument("--tile", default=None)
args = ap.parse_args()
dev = torch.device("cuda", 0)
peak = 2.0 * bench._peaks()[0]["bf16_tflops"]
specs = {}
_, local = bench.deepseek_gateup_sizes(seed=0)
specs["ds_gateup"] = ([local], 4096, 7168, 32, "kn")
counts, _ = bench.deepseek_gateup_sizes(seed=1)
specs["ds_down"] = ([counts], 7168, 2048, 256, "kn")
q, _ = bench.deepseek_gateup_sizes(seed=2, experts=128, local=128)
specs["q_fgu"] = ([q], 3072, 4096, 128, "kn")
specs["q_fdn"] = ([q], 4096, 1536, 128, "kn")
specs["q_ddn"] = ([q], 1536, 4096, 128, "nk")
specs["q_dgu"] = ([q], 4096, 3072, 128, "nk")
specs["sweep_r64"] = ([tuple(128 * g + 64 for g in range(8))], 4096, 7168, 8, "kn")
specs["sq8192"] = ([(8192,)], 8192, 8192, 1, "kn")
names = args.names or list(specs)
for name in names:
    sizes, n, k, G, layout = specs[name]
    P = bench.Problem(torch, name, sizes, n, k, G, dev, seed=7, b_layout=layout)
    gs = P.gs[0]

    def fn():
        tg.grouped_gemm_fp8(P.a, P.sa, P.b, P.sb, gs, b_layout=layout, out=P.out, exact_promotion=args.exact,
                            pdl_overlap=True, tile=args.tile)

    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / args.iters
    tf = P.flops[0] / (ms * 1e-3) / 1e12
    print(json.dumps({"tag": args.tag, "name": name, "ms": round(ms, 4), "tflops": round(tf, 1),
                      "frac": round(tf / peak, 4)}), flush=True)
    del P
    torch.cuda.empty_cache()
