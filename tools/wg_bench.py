import sys, json, torch
sys.path.insert(0, ".")
import bench
import paper_2508_16584_b200 as tg
print(json.dumps(bench.run_wgrad(torch, tg, torch.device("cuda", 0), 3296.0)))
