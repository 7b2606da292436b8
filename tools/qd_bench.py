import sys, json, torch
sys.path.insert(0, ".")
import bench
import paper_2508_16584_b200 as tg
r = bench.run_quantize_dispatch(torch, tg, torch.device("cuda", 0))
print(json.dumps(r))
