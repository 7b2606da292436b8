"""Time ep.plan_chunks and ep.pipelined_expert_gemm pieces at the DeepSeek-V3 down EP size (world 1)."""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
import paper_2508_16584_b200 as tg  # noqa: E402
from paper_2508_16584_b200 import ep  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29656")
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
E, N, K, R = 256, 7168, 2048, 262144
eid = torch.randint(0, E, (R,), device=dev)
a = torch.randint(0, 120, (R, K), dtype=torch.uint8, device=dev)
sa = torch.rand((R, K // 128), device=dev) * 1e-2
b = torch.randint(0, 120, (E, K, N), dtype=torch.uint8, device=dev)
sb = torch.rand((E, K // 128, N // 128), device=dev) * 1e-2


def gemm(codes, scales, gs):
    return tg.grouped_gemm_fp8(codes, scales, b, sb, gs, max_sms=132)


def timed(name, fn, it=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it):
        fn()
    e.record()
    torch.cuda.synchronize()
    print(f"{name:36s} gpu {s.elapsed_time(e) / it:8.2f} ms   wall {(time.perf_counter() - t0) * 1e3 / it:8.2f} ms",
          flush=True)


for ch in (1, 2, 4):
    timed(f"plan_chunks c={ch}", lambda: ep.plan_chunks(eid, E, ch))
    plan = ep.plan_chunks(eid, E, ch)
    timed(f"pipelined (plan given) c={ch}", lambda: ep.pipelined_expert_gemm(a, sa, eid, E, gemm, N, plan=plan))
    timed(f"pipelined (with plan) c={ch}", lambda: ep.pipelined_expert_gemm(a, sa, eid, E, gemm, N, chunks=ch))
dist.destroy_process_group()
