"""Time the pieces of ep.combine / ep.dispatch at the DeepSeek-V3 down EP size (world 1)."""
import os
import torch
import torch.distributed as dist

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29655")
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
R, N = 262144, 7168
c = torch.randn((R, N), device=dev).to(torch.bfloat16)
perm = torch.randperm(R, device=dev)
out = torch.empty_like(c)


def t(name, fn, it=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / it
    gb = 2 * c.numel() * 2 / 1e9
    print(f"{name:28s} {ms:8.3f} ms  {gb / ms:7.1f} GB/s (2 x {c.numel() * 2 / 1e9:.2f} GB)")


t("index_select", lambda: torch.index_select(c, 0, perm, out=out))
t("index_copy_", lambda: out.index_copy_(0, perm, c))
t("copy_", lambda: out.copy_(c))
t("a2a world1", lambda: dist.all_to_all_single(out, c, [R], [R]))
t("a2a world1 (even)", lambda: dist.all_to_all_single(out, c))
dist.destroy_process_group()
