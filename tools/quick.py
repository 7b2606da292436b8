"""Quick A/B timing of the production kernel (libtagg.so) on a few shapes.

python tools/quick.py [flags]   -> TFLOP/s per shape (CUDA events, 20 launches after 3 warm-ups)
"""
import sys

import torch

sys.path.insert(0, ".")
from bench import Problem, deepseek_gateup_sizes  # noqa: E402
import ctypes  # noqa: E402

from paper_2508_16584_b200 import _lib  # noqa: E402

args = [a for a in sys.argv[1:] if not a.endswith(".so")]
libs = [a for a in sys.argv[1:] if a.endswith(".so")] or [str(_lib.LIB_PATH)]
flags = int(args[0], 0) if args else 0


def load(path):
    L = ctypes.CDLL(path)
    for nm, (r, a) in _lib.SIGNATURES.items():
        if hasattr(L, nm):
            getattr(L, nm).restype, getattr(L, nm).argtypes = r, a
    return L
dev = torch.device("cuda", 0)
shapes = [
    ("tiles4", [(256 * 74,)], 1024, 8192, 1, "kn"),
    ("sq8192", [(8192,)], 8192, 8192, 1, "kn"),
    ("sweep_r64", [tuple(128 * g + 64 for g in range(8))], 4096, 7168, 8, "kn"),
    ("ds_gateup", [tuple(int(x) for x in deepseek_gateup_sizes(0)[1])], 4096, 7168, 32, "kn"),
    ("qwen_dgrad_gu", None, 4096, 3072, 128, "nk"),
    ("ds_down", [tuple(int(x) for x in deepseek_gateup_sizes(seed=1)[0])], 7168, 2048, 256, "kn"),
    ("qwen_fwd_gu", [tuple(int(x) for x in deepseek_gateup_sizes(seed=2, experts=128, local=128)[0])], 3072, 4096, 128,
     "kn"),
    ("qwen_fwd_down", [tuple(int(x) for x in deepseek_gateup_sizes(seed=2, experts=128, local=128)[0])], 4096, 1536,
     128, "kn"),
    ("qwen_dgrad_down", [tuple(int(x) for x in deepseek_gateup_sizes(seed=2, experts=128, local=128)[0])], 1536, 4096,
     128, "nk"),
]
only = [a for a in args[1:]] if len(args) > 1 else None
shapes = [s for s in shapes if only is None or s[0] in only]
for name, sizes, n, k, G, bl in shapes:
    if sizes is None:
        sizes = [tuple([2048] * 128)]
    P = Problem(torch, name, sizes, n, k, G, dev, seed=1, b_layout=bl)
    layout = 0 if bl == "kn" else 1

    def run():
        rc = L.tagg_grouped_gemm_fp8(P.a.data_ptr(), P.a.stride(0), P.sa.data_ptr(), P.m_alloc, P.b.data_ptr(),
                                         layout, G, P.sb.data_ptr(), P.sb.stride(0), P.sb.stride(1), P.sb.stride(2),
                                         P.gs[0].data_ptr(), G, n, k, P.out.data_ptr(), n, P.m_alloc, None, None,
                                         flags, torch.cuda.current_stream().cuda_stream)
        assert rc == 0, rc

    # ABBA-interleaved rounds: power/boost state drifts over a run, so libraries are
    # timed alternately and each reports its median over rounds.
    loaded = [load(path) for path in libs]
    times = {path: [] for path in libs}
    order = list(range(len(libs)))
    for rnd in range(6):
        seq = order if rnd % 2 == 0 else order[::-1]
        for i in seq:
            L = loaded[i]
            for _ in range(2):
                run()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(10):
                run()
            e.record()
            torch.cuda.synchronize()
            times[libs[i]].append(s.elapsed_time(e) / 10)
    for path in libs:
        ms = sorted(times[path])[len(times[path]) // 2]
        tag = path.rsplit("/", 1)[-1]
        print(f"{name:14s} {tag:22s} {ms * 1e3:9.1f} us  {P.flops[0] / ms / 1e9:8.1f} TFLOP/s", flush=True)
    del P
