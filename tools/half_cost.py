"""Relative cost of a half tile (a group's last pair tile with <= 128 rows: one M=128 cta_group::2
MMA per K step) against a full 256-row pair tile: the same number of tiles, all half or all
full (74 groups, one pair m-tile each), N = 1024, K = 7168.  ABBA, median of 6 rounds."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2508_16584_b200 as tg  # noqa: E402

dev = torch.device("cuda", 0)
n, k, G = 1024, 7168, 74
probs = {rows: bench.Problem(torch, f"g{rows}", [(rows,) * G], n, k, G, dev, seed=5) for rows in (256, 128, 96, 64)}
res = {r: [] for r in probs}
for rnd in range(6):
    for rows in (list(probs) if rnd % 2 == 0 else list(probs)[::-1]):
        P = probs[rows]
        f = lambda: tg.grouped_gemm_fp8(P.a, P.sa, P.b, P.sb, P.gs[0], out=P.out, tile="pair_n256")  # noqa: E731
        for _ in range(2):
            f()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(10):
            f()
        e.record()
        torch.cuda.synchronize()
        res[rows].append(s.elapsed_time(e) / 10)
base = sorted(res[256])[3]
for rows, v in res.items():
    ms = sorted(v)[3]
    print(f"{G} groups x {rows:3d} rows (N={n}, K={k}): {ms * 1e3:7.1f} us  = {ms / base:.2f} x the full-tile launch")
