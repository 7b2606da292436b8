./tools/micro/div_check
timeout 600 python -m pytest tests/test_quant_gpu.py tests/test_wgrad_gpu.py tests/test_moe_gpu.py tests/test_safety_gpu.py -q 2>&1 | tail -3
timeout 120 python tools/colq_bench.py
timeout 200 python -c "
import sys; sys.path.insert(0,'.')
import torch, bench, paper_2508_16584_b200 as tg
dev=torch.device('cuda',0)
print(bench.run_quantize_dispatch(torch, tg, dev))
print(bench.run_wgrad(torch, tg, dev, 3296.0))
"
