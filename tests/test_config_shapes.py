"""GPU parity at the BASELINE.json configuration shapes, at full size.

configs[2] (C3) DeepSeek-V3 gate+up, configs[3] (C4) DeepSeek-V3 down with 256 experts (one
GPU, and one EP=8 rank's shard), configs[4] (C5) the four Qwen3-235B-A22B forward / dgrad
GEMMs, the dgrad ones with K-major B ("nk", the layout dgrad reads the forward weights in) and
every shape in both B layouts.  The group sizes are the bench's own Zipf top-8 routing draws
(bench.deepseek_gateup_sizes), so these are the very problems bench.py times.

The full outputs are computed on the GPU.  The CPU oracle (oracle/, pinned to the reference's
goldens in test_oracle.py) recomputes one 128-column slice of EVERY row (the reference's
semantics are column-block independent: engine.py:161-169 scales by column block n // 128), at
a pseudo-random column block per test.  Values must lie within helpers.REL_TOL; the
untouched-memory check is bit-exact (a sentinel row band after sum(M_g)).
Anchor: engine.py:346-402 / test_acceptance.py:180-201 (the reference's own parity claim).
"""

from __future__ import annotations

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from bench import deepseek_gateup_sizes  # noqa: E402
from helpers import assert_parity, oracle_c  # noqa: E402

import paper_2508_16584_b200 as tg  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda"
SENTINEL = 0x7BCD
THREADS = max(1, min(16, len(os.sched_getaffinity(0))))


def _codes(shape, gen):
    c = torch.randint(0, 256, shape, dtype=torch.uint8, device=DEV, generator=gen)
    return torch.where((c & 0x7F) == 0x7F, c - 1, c)  # no NaN code


def _scales(shape, gen):
    e = torch.randint(-12, -4, shape, device=DEV, generator=gen).float()
    return (torch.rand(shape, device=DEV, generator=gen) * 0.5 + 0.5) * torch.exp2(e)


def _run_and_check(sizes, n, k, layout, seed, exact=False, tile=None):
    sizes = tuple(int(s) for s in sizes)
    G, m = len(sizes), sum(sizes)
    kb, nb = -(-k // 128), -(-n // 128)
    gen = torch.Generator(device=DEV).manual_seed(seed)
    a, sa = _codes((m, k), gen), _scales((m, kb), gen)
    if layout == "kn":
        b, sb = _codes((G, k, n), gen), _scales((G, kb, nb), gen)
    else:
        b, sb = _codes((G, n, k), gen), _scales((G, nb, kb), gen)
    gs = torch.tensor(sizes, dtype=torch.int32, device=DEV)
    out = torch.full((m + 64, n), SENTINEL, dtype=torch.int16, device=DEV)
    tg.grouped_gemm_fp8(a, sa, b, sb, gs, b_layout=layout, out=out, exact_promotion=exact, tile=tile)
    torch.cuda.synchronize()
    # rows past sum(M_g) are never written (the store pool + dual-phase store)
    assert bool((out[m:] == SENTINEL).all()), "rows past sum(M_g) were written"
    # one 128-column block of every row against the oracle
    cb = int(np.random.default_rng(seed).integers(0, nb))
    c0, c1 = 128 * cb, min(n, 128 * cb + 128)
    if layout == "kn":
        bs = b[:, :, c0:c1].contiguous().cpu().numpy()
        sbs = sb[:, :, cb:cb + 1].contiguous().cpu().numpy()
    else:
        bs = b[:, c0:c1, :].contiguous().cpu().numpy()
        sbs = sb[:, cb:cb + 1, :].contiguous().cpu().numpy()
    want = oracle_c(a.cpu().numpy(), sa.cpu().numpy(), bs, sbs, sizes, b_layout=layout, threads=THREADS)
    got = out[:m, c0:c1].contiguous().cpu().numpy().view(np.uint16)
    rep = assert_parity(got, want, label=f"G={G} M={m} N={n} K={k} {layout} cols [{c0},{c1})")
    print(f"G={G} M={m} N={n} K={k} {layout} cols [{c0},{c1}): {rep}")
    return rep


@pytest.mark.parametrize("exact", [False, True])
def test_c3_deepseek_v3_gate_up_bench_routing(exact):
    """configs[2]: 32 local experts (EP rank 0 of 8), 32k tokens top-8 with Zipf routing, N=4096,
    K=7168 -- the bench's deepseek_v3_gateup_ep8_rank0 problem, both promotion modes."""
    _, local = deepseek_gateup_sizes(seed=0)
    _run_and_check(local, 4096, 7168, "kn", seed=30, exact=exact)


def test_c4_deepseek_v3_down_256_experts_one_gpu():
    """configs[3] at P=1: all 256 experts, 262,144 routed rows, N=7168, K=2048."""
    counts, _ = deepseek_gateup_sizes(seed=1)
    assert int(counts.sum()) == 32768 * 8 and len(counts) == 256
    _run_and_check(counts, 7168, 2048, "kn", seed=40)


@pytest.mark.parametrize("rank", [0, 7])
def test_c4_deepseek_v3_down_ep8_shard(rank):
    """configs[3] at P=8: one rank's 32 experts (experts [32 rank, 32 rank + 32))."""
    counts, _ = deepseek_gateup_sizes(seed=1)
    _run_and_check(counts[32 * rank:32 * rank + 32], 7168, 2048, "kn", seed=41 + rank)


QWEN3 = {
    "fwd_gateup": (3072, 4096),
    "fwd_down": (4096, 1536),
    "dgrad_down": (1536, 4096),
    "dgrad_gateup": (4096, 3072),
}


@pytest.mark.parametrize("layout", ["kn", "nk"])
@pytest.mark.parametrize("name", list(QWEN3))
def test_c5_qwen3_235b_shapes(name, layout):
    """configs[4]: 128 experts, top-8 of 32768 tokens (262,144 rows): forward gate+up / down
    and the dgrad GEMMs (dH = dY W^T reads the forward weights K-major, "nk"), each shape in
    both B layouts."""
    n, k = QWEN3[name]
    q, _ = deepseek_gateup_sizes(seed=2, experts=128, local=128)
    _run_and_check(q, n, k, layout, seed=50 + len(name) + (layout == "nk"))


@pytest.mark.parametrize("tile", ["1cta", "pair_n128"])
def test_c3_other_tile_shapes(tile):
    """The explicit tile shapes on the C3 problem."""
    _, local = deepseek_gateup_sizes(seed=0)
    _run_and_check(local, 4096, 7168, "kn", seed=33, tile=tile)
