"""One MoE FFN step chain at DeepSeek-V3 scale (for ncu): python tools/moe_one.py"""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2508_16584_b200 as tg  # noqa: E402

print(json.dumps(bench.run_moe_ffn(torch, tg, torch.device("cuda", 0), 3296.0, iters=1, warmup=1)))
