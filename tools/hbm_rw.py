"""HBM write-only / copy / read-only rates with torch's own kernels (4 GiB buffers): the context
for write-dominated kernels such as quantize + dispatch (80% of its bytes are writes)."""
import torch

x = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
y = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")


def rate(fn, nbytes, name):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"{name}: {nbytes / ms / 1e6:.0f} GB/s")


rate(lambda: x.fill_(1), x.numel(), "write (fill_)")
rate(lambda: y.copy_(x), 2 * x.numel(), "copy (read + write)")
rate(lambda: x.view(torch.int64).max(), x.numel(), "read (max)")
