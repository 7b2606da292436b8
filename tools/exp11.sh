timeout 300 python -m pytest tests/test_wgrad_gpu.py tests/test_moe_gpu.py -q 2>&1 | tail -3
timeout 200 python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, json, paper_2508_16584_b200 as tg
dev=torch.device('cuda',0)
print(json.dumps(bench.run_wgrad(torch, tg, dev, 3296.0)))
"
