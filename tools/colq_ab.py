"""A/B timing of libtagg builds' column-block quantizer (bf16, 262144 grouped rows, 256 groups):
python tools/colq_ab.py [--gather] A.so B.so ...  (ABBA rounds; GB/s counts one read of x + the codes;
--gather: the weighted gather form from a token-ordered tensor)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_16584_b200 import _lib  # noqa: E402

GATHER = "--gather" in sys.argv
libs = [a for a in sys.argv[1:] if a != "--gather"]
L = []
for path in libs:
    lib = ctypes.CDLL(path)
    for nm, (r, a) in _lib.SIGNATURES.items():
        if hasattr(lib, nm):
            getattr(lib, nm).restype, getattr(lib, nm).argtypes = r, a
    L.append(lib)
dev = torch.device("cuda", 0)
gs = torch.full((256,), 1024, dtype=torch.int32, device=dev)
err = torch.zeros(1, dtype=torch.int32, device=dev)
for cols in (2048, 7168):
    x = torch.randn((262144, cols), device=dev).to(torch.bfloat16)
    codes = torch.empty((262144, cols), dtype=torch.uint8, device=dev)
    sc = torch.empty((2048 + 256, cols), dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream().cuda_stream

    # gather mode (MoE backward's dC): row r = w[r] * x_tok[index[r]] from a token-ordered
    # [32768, cols] tensor, top-8 rows per token
    xt = x[:32768]
    idx = torch.randint(0, 32768, (262144,), device=dev, dtype=torch.int32)
    wts = torch.rand(262144, device=dev)

    def run(lib):
        if GATHER:
            rc = lib.tagg_quantize_col_blocks_gather(xt.data_ptr(), 0, cols, idx.data_ptr(), wts.data_ptr(), 262144,
                                                     cols, gs.data_ptr(), 256, codes.data_ptr(), cols, sc.data_ptr(),
                                                     err.data_ptr(), st)
        else:
            rc = lib.tagg_quantize_col_blocks(x.data_ptr(), 0, 262144, cols, cols, gs.data_ptr(), 256,
                                              codes.data_ptr(), cols, sc.data_ptr(), err.data_ptr(), st)
        assert rc == 0, rc
    times = {p: [] for p in libs}
    for rnd in range(6):
        order = list(range(len(libs))) if rnd % 2 == 0 else list(range(len(libs)))[::-1]
        for i in order:
            run(L[i])
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(5):
                run(L[i])
            e.record()
            torch.cuda.synchronize()
            times[libs[i]].append(s.elapsed_time(e) / 5)
    for p in libs:
        ms = sorted(times[p])[3]
        print(f"cols {cols:5d} {p.rsplit('/', 1)[-1]:16s} {ms:7.3f} ms {x.numel() * 3 / ms / 1e6:7.0f} GB/s")
