"""GPU parity: the sm_100a kernel (through the C ABI) against the CPU oracle.

Every comparison uses the oracle (oracle/, pinned to the reference's own
goldens in test_oracle.py), the committed golden fixtures, or a
size-independent property.  Values must lie within helpers.REL_TOL.  The
index map and the untouched-memory checks are bit-exact.
"""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from helpers import assert_parity, oracle_c, per_expert_operands, tolerance_report  # noqa: E402
from oracle import fp8 as ofp8  # noqa: E402
from oracle import plan as oplan  # noqa: E402
from tmas import CASES, load_case  # noqa: E402

import paper_2508_16584_b200 as tg  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _cfg_ops(case):
    layout = "nk" if case.get("b_layout") == "expert_nk" else "kn"
    cfg = tg.ProblemConfig(n=case["n"], k=case["k"], group_sizes=tuple(case["group_sizes"]))
    ops = tg.GroupedOperands(case["a_codes"], case["a_scales"], case["b_codes"], case["b_scales"], b_layout=layout)
    return cfg, ops, layout


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("mode", ["ffma2", "exact", "plain_staging", "1cta", "1cta_exact", "pair_n128",
                                  "pair_n128_exact", "pair_n256"])
def test_golden_fixtures(name, mode):
    case = load_case(name)
    cfg, ops, _ = _cfg_ops(case)
    tile = next((t for t in ("1cta", "pair_n128", "pair_n256") if mode.startswith(t)), None)
    run = tg.run_adaptive(cfg, ops, exact_promotion=("exact" in mode), plain_staging=(mode == "plain_staging"),
                          tile=tile)
    rep = assert_parity(run.c_bits, case["c_golden"], label=f"{name}/{mode}")
    print(f"{name}/{mode}: {rep}")


def _pairs(sizes, n):
    """CTA pairs of a 256x256 pair-tile launch over these groups (tagg_launch_clusters)."""
    from paper_2508_16584_b200._lib import lib
    return lib().tagg_launch_clusters(int(sum(sizes)), len(sizes), n, 16)



@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("tile", ["1cta", "pair_n128", "pair_n256"])
def test_tile_map_is_bit_exact(name, tile):
    """The store geometry the kernel used equals the reference tile loop (engine.py:269-335)."""
    case = load_case(name)
    cfg, ops, _ = _cfg_ops(case)
    run = tg.run_adaptive(cfg, ops, tile=tile)
    got = sorted(tuple(int(x) for x in r) for r in run.tile_map)
    want = sorted(oplan.kernel_tile_map(cfg.group_sizes, cfg.n, tile, num_pairs=_pairs(cfg.group_sizes, cfg.n)))
    assert got == want
    # the rows each group's pieces write are exactly the reference tile loop's rows
    covered = sorted({(r[0], r[2], row) for r in got for row in range(r[6], r[6] + r[4])})
    ref = sorted({(r[0], r[2], row) for r in oplan.tile_map(cfg.group_sizes, cfg.n)
                  for row in range(r[6], r[6] + r[4])})
    assert covered == ref


@pytest.mark.parametrize("name", ["c1", "k640", "perexpert"])
def test_padded_baseline_equals_adaptive_bitwise(name):
    """Paper claim: the padding-free path is bitwise identical to
    pad + padded GEMM on the valid rows."""
    case = load_case(name)
    cfg, ops, _ = _cfg_ops(case)
    a = tg.run_adaptive(cfg, ops).c_bits
    b = tg.run_padded_baseline(cfg, ops)
    assert tg.verify_bitwise(a, b).equal


def test_poison_never_reaches_output_and_all_rows_written():
    case = load_case("k640")
    cfg, ops, _ = _cfg_ops(case)
    outs = [tg.run_adaptive(cfg, ops, poison=p).c_bits for p in (0xA5, 0x5A, 0x7F)]
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def _dev(x, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(x)).to(DEV)
    return t if dtype is None else t.to(dtype)


@pytest.mark.parametrize("gap", [1, 3, 128])
@pytest.mark.parametrize("tile", ["1cta", "pair_n128", "pair_n256"])
def test_untouched_memory_between_groups(gap, tile):
    """No row beyond M_g is ever written: sentinel rows between groups survive."""
    sizes = (1, 67, 128, 255, 0, 129, 200, 64, 3)
    n, k = 192, 384
    ac, asc, bc, bsc = per_expert_operands(sizes, n, k, 21)
    offs, o = [], 0
    for s in sizes:
        offs.append(o)
        o += s + gap
    sentinel = 0x7BCD
    out = torch.full((o, n), sentinel, dtype=torch.int16, device=DEV)
    tg.grouped_gemm_fp8(_dev(ac), _dev(asc), _dev(bc), _dev(bsc), _dev(np.array(sizes, np.int32)),
                        out=out, c_row_offsets=_dev(np.array(offs, np.int64)), tile=tile)
    got = out.cpu().numpy().view(np.uint16)
    want = oracle_c(ac, asc, bc, bsc, sizes)
    a = 0
    for g, s in enumerate(sizes):
        assert_parity(got[offs[g]:offs[g] + s], want[a:a + s], label=f"group {g}")
        assert np.all(got[offs[g] + s:offs[g] + s + gap] == sentinel), f"gap after group {g} written"
        a += s


@pytest.mark.parametrize("tile", ["1cta", "pair_n128", "pair_n256"])
def test_residual_sweep_every_residue_small(tile):
    """Every M_g mod 128 in 1..127 (configs[1] pattern, M_g = 128*g + r) at N=256, K=256."""
    n, k = 256, 256
    for r0 in range(1, 128, 16):
        sizes = tuple(128 * g + ((r0 + g) % 127 + 1) for g in range(8))
        ac, asc, bc, bsc = per_expert_operands(sizes, n, k, r0)
        cfg = tg.ProblemConfig(n=n, k=k, group_sizes=sizes)
        run = tg.run_adaptive(cfg, tg.GroupedOperands(ac, asc, bc, bsc), tile=tile)
        assert_parity(run.c_bits, oracle_c(ac, asc, bc, bsc, sizes), label=f"r0={r0}")
        got = sorted(tuple(int(x) for x in rr) for rr in run.tile_map)
        assert got == sorted(oplan.kernel_tile_map(sizes, n, tile, num_pairs=_pairs(sizes, n)))


def _synthetic(sizes, n, k, seed, layout="kn"):
    """Fast synthetic operands (uniform finite e4m3 codes, positive fp32 scales)."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    m = int(sum(sizes))
    G = len(sizes)
    kb, nb = -(-k // 128), -(-n // 128)

    def codes(*shape):
        c = torch.randint(0, 256, shape, generator=g, dtype=torch.int32)
        c = torch.where((c & 0x7F) == 0x7F, c - 1, c)  # avoid the two NaN codes
        return c.to(torch.uint8).numpy()

    def scales(*shape):
        e = torch.randint(-12, -4, shape, generator=g).float()
        return (torch.rand(shape, generator=g) * 0.5 + 0.5).mul(torch.exp2(e)).numpy().astype(np.float32)

    ac, asc = codes(m, k), scales(m, kb)
    if layout == "kn":
        bc, bsc = codes(G, k, n), scales(G, kb, nb)
    else:
        bc, bsc = codes(G, n, k), scales(G, nb, kb)
    return ac, asc, bc, bsc


@pytest.mark.parametrize("layout", ["kn", "nk"])
@pytest.mark.parametrize("tile", ["1cta", "pair_n128", "pair_n256"])
def test_deepseek_shape_sampled_columns(layout, tile):
    """DeepSeek-V3 gate+up shape (N=4096, K=7168) with ragged groups.  Parity is
    checked on two 128-column slices and all rows against the oracle."""
    sizes = (300, 0, 1, 1024, 77, 513, 128, 255)
    n, k = 4096, 7168
    ac, asc, bc, bsc = _synthetic(sizes, n, k, 7, layout)
    out = tg.grouped_gemm_fp8(_dev(ac), _dev(asc), _dev(bc), _dev(bsc), _dev(np.array(sizes, np.int32)),
                              b_layout=layout, tile=tile)
    got = out.view(torch.int16).cpu().numpy().view(np.uint16)
    for n0 in (0, 2944):
        want = np.zeros((sum(sizes), n), dtype=np.uint16)
        oracle_c(ac, asc, bc, bsc, sizes, b_layout=layout, n_range=(n0, n0 + 128), out=want)
        rep = assert_parity(got[:, n0:n0 + 128], want[:, n0:n0 + 128], label=f"n0={n0}")
        print(f"deepseek {layout} n0={n0}: {rep}")


@pytest.mark.parametrize("tile", ["1cta", "pair_n128", "pair_n256"])
def test_k_tail_and_n_tail_shapes(tile):
    sizes = (5, 130, 37, 300)
    for n, k in ((64, 16), (192, 208), (320, 1664), (64, 4112), (448, 640)):
        ac, asc, bc, bsc = _synthetic(sizes, n, k, n + k)
        out = tg.grouped_gemm_fp8(_dev(ac), _dev(asc), _dev(bc), _dev(bsc), _dev(np.array(sizes, np.int32)),
                                  tile=tile)
        got = out.view(torch.int16).cpu().numpy().view(np.uint16)
        assert_parity(got, oracle_c(ac, asc, bc, bsc, sizes), label=f"n={n} k={k}")


def test_shared_b_reference_api_and_empty_groups():
    sizes = (0, 0, 131, 0)
    n, k = 256, 512
    ac, asc, bc, bsc = ofp8.random_operands(sum(sizes), n, k, 4)
    run = tg.run_adaptive(tg.ProblemConfig(n=n, k=k, group_sizes=sizes), tg.GroupedOperands(ac, asc, bc, bsc))
    assert_parity(run.c_bits, oracle_c(ac, asc, bc, bsc, sizes))
    empty = tg.run_adaptive(tg.ProblemConfig(n=64, k=64, group_sizes=(0,)),
                            tg.GroupedOperands(np.zeros((0, 64), np.uint8), np.zeros((0, 1), np.float32),
                                               np.zeros((64, 64), np.uint8), np.ones((1, 1), np.float32)))
    assert empty.c_bits.shape == (0, 64)


def test_device_group_sizes_without_host_sync_under_graph_capture():
    """The whole call is capturable in a CUDA graph.  Group sizes live on the
    device and can change between replays."""
    sizes = [100, 200, 50]
    n, k = 256, 256
    ac, asc, bc, bsc = _synthetic((512, 0, 0), n, k, 3)  # 512 rows, 3 experts
    a, sa, b, sb = _dev(ac), _dev(asc), _dev(bc), _dev(bsc)
    gs = _dev(np.array(sizes, np.int32))
    out = torch.zeros((512, n), dtype=torch.bfloat16, device=DEV)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        tg.grouped_gemm_fp8(a, sa, b, sb, gs, out=out)  # warm-up (sets smem attribute)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        tg.grouped_gemm_fp8(a, sa, b, sb, gs, out=out)
    for new in ([100, 200, 50], [1, 127, 384], [0, 512, 0]):
        gs.copy_(torch.tensor(new, dtype=torch.int32))
        out.zero_()
        graph.replay()
        torch.cuda.synchronize()
        got = out.view(torch.int16).cpu().numpy().view(np.uint16)
        m = sum(new)
        assert_parity(got[:m], oracle_c(ac[:m], asc[:m], bc, bsc, new), label=str(new))
        assert np.all(got[m:] == 0)


def test_error_mapping():
    a = torch.zeros((4, 128), dtype=torch.uint8, device=DEV)
    sa = torch.ones((4, 1), dtype=torch.float32, device=DEV)
    b = torch.zeros((128, 96), dtype=torch.uint8, device=DEV)
    sb = torch.ones((1, 1), dtype=torch.float32, device=DEV)
    gs = torch.tensor([4], dtype=torch.int32, device=DEV)
    with pytest.raises(tg.ConfigError):
        tg.grouped_gemm_fp8(a, sa, b, sb, gs)  # N = 96 is not a multiple of 64
    b = torch.zeros((130, 128), dtype=torch.uint8, device=DEV)
    with pytest.raises(tg.ShapeMismatch):
        tg.grouped_gemm_fp8(a, sa, b, sb, gs)


def test_identical_fraction_reported_for_reference_recipe():
    """The reference input recipe at configs[0]: report the bit-identical fraction."""
    case = load_case("c1")
    cfg, ops, _ = _cfg_ops(case)
    for exact in (False, True):
        run = tg.run_adaptive(cfg, ops, exact_promotion=exact)
        rep = tolerance_report(run.c_bits, case["c_golden"])
        print(f"c1 exact={exact}: {rep}")
        assert rep["out_of_tol"] == 0
        assert rep["bit_identical"] > 0.9


@pytest.mark.parametrize("max_sms", [2, 22, 132])
@pytest.mark.parametrize("tile", ["1cta", "pair_n256"])
def test_sm_limited_grid(max_sms, tile):
    """TAGG_SM_LIMIT(n) caps the persistent grid (room for NCCL beside the GEMM): values and
    the tile map (whose tail balancing depends on the cluster count) stay exact."""
    from paper_2508_16584_b200._lib import lib

    sizes = (700, 3, 129, 0, 1000, 255)
    n, k = 768, 384
    ac, asc, bc, bsc = _synthetic(sizes, n, k, max_sms)
    m = sum(sizes)
    flags = (4 if tile == "1cta" else 16) | (max_sms << 16)
    clusters = lib().tagg_launch_clusters(m, len(sizes), n, flags)
    assert 0 < clusters * (1 if tile == "1cta" else 2) <= max_sms
    tmap = torch.full((tg.max_tiles(m, len(sizes), n), 9), -1, dtype=torch.int32, device=DEV)
    out = tg.grouped_gemm_fp8(_dev(ac), _dev(asc), _dev(bc), _dev(bsc), _dev(np.array(sizes, np.int32)),
                              tile=tile, tile_map=tmap, max_sms=max_sms)
    got = out.view(torch.int16).cpu().numpy().view(np.uint16)
    assert_parity(got, oracle_c(ac, asc, bc, bsc, sizes), label=f"max_sms={max_sms}")
    tm = tmap.cpu().numpy()
    tm = sorted(tuple(int(x) for x in r) for r in tm[tm[:, 0] >= 0])
    assert tm == sorted(oplan.kernel_tile_map(sizes, n, tile, num_pairs=clusters))
    if tile == "pair_n256":
        with pytest.raises(tg.ConfigError):
            tg.grouped_gemm_fp8(_dev(ac), _dev(asc), _dev(bc), _dev(bsc), _dev(np.array(sizes, np.int32)),
                                tile=tile, max_sms=1)


@pytest.mark.parametrize("max_sms", [0, 60])
def test_tile_map_with_tall_groups_spanning_super_rows(max_sms):
    """Groups taller than one raster super-row (8 pair m-tiles), with a tail split: the tile
    map still equals the reference tile loop's store geometry."""
    sizes = (8 * 256 * 5 + 77, 3, 300, 8 * 256 + 256)
    n, k = 512, 256
    ac, asc, bc, bsc = _synthetic(sizes, n, k, 31)
    m = sum(sizes)
    from paper_2508_16584_b200._lib import lib
    clusters = lib().tagg_launch_clusters(m, len(sizes), n, max_sms << 16)
    tmap = torch.full((tg.max_tiles(m, len(sizes), n), 9), -1, dtype=torch.int32, device=DEV)
    out = tg.grouped_gemm_fp8(_dev(ac), _dev(asc), _dev(bc), _dev(bsc), _dev(np.array(sizes, np.int32)),
                              tile_map=tmap, max_sms=max_sms or None)
    tm = tmap.cpu().numpy()
    tm = sorted(tuple(int(x) for x in r) for r in tm[tm[:, 0] >= 0])
    assert tm == sorted(oplan.kernel_tile_map(sizes, n, "pair_n256", num_pairs=clusters))
    got = out.view(torch.int16).cpu().numpy().view(np.uint16)
    want = np.zeros((m, n), dtype=np.uint16)
    oracle_c(ac, asc, bc, bsc, sizes, n_range=(256, 384), out=want)
    assert_parity(got[:, 256:384], want[:, 256:384], label="tall groups")


def test_largest_k_and_the_unsupported_limit():
    """K is bounded by the S_B staging (128 k-blocks): every K <= 16384 runs -- the S_A window
    drops to one slot when two do not fit beside two pipeline stages -- and K = 16512 raises
    Unsupported before launch (tagg.h TAGG_ERR_UNSUPPORTED), never a wrong result."""
    sizes = (130, 1, 256)
    n = 128
    for k in (15872, 16384, 16512):
        ac, asc, bc, bsc = _synthetic(sizes, n, k, k)
        args = (_dev(ac), _dev(asc), _dev(bc), _dev(bsc), _dev(np.array(sizes, np.int32)))
        if k == 16512:
            with pytest.raises(tg.Unsupported):
                tg.grouped_gemm_fp8(*args)
            continue
        for tile in ("1cta", "pair_n256"):
            got = tg.grouped_gemm_fp8(*args, tile=tile).view(torch.int16).cpu().numpy().view(np.uint16)
            assert_parity(got, oracle_c(ac, asc, bc, bsc, sizes), label=f"k={k} {tile}")


def test_thousands_of_groups_mostly_empty():
    """G = 4096 experts (device group tables in smem), 95% of them empty, ragged rest."""
    rng = np.random.default_rng(4096)
    sizes = tuple(int(x) if rng.random() < 0.05 else 0 for x in rng.integers(1, 300, 4096))
    n, k = 128, 256
    ac, asc, bc, bsc = _synthetic(sizes, n, k, 5)
    m = sum(sizes)
    tmap = torch.full((tg.max_tiles(m, len(sizes), n), 9), -1, dtype=torch.int32, device=DEV)
    out = tg.grouped_gemm_fp8(_dev(ac), _dev(asc), _dev(bc), _dev(bsc), _dev(np.array(sizes, np.int32)),
                              tile_map=tmap, tile="pair_n256")
    got = out.view(torch.int16).cpu().numpy().view(np.uint16)
    assert_parity(got, oracle_c(ac, asc, bc, bsc, sizes), label="G=4096")
    tm = tmap.cpu().numpy()
    tm = sorted(tuple(int(x) for x in r) for r in tm[tm[:, 0] >= 0])
    assert tm == sorted(oplan.kernel_tile_map(sizes, n, "pair_n256", num_pairs=_pairs(sizes, n)))


def test_too_many_groups_is_unsupported_not_wrong():
    sizes = (5,) + (0,) * 19999
    ac, asc, bc, bsc = _synthetic(sizes[:1], 128, 128, 1)
    bc = np.broadcast_to(bc, (len(sizes),) + bc.shape[1:]).copy()
    bsc = np.broadcast_to(bsc, (len(sizes),) + bsc.shape[1:]).copy()
    with pytest.raises(tg.Unsupported):
        tg.grouped_gemm_fp8(_dev(ac), _dev(asc), _dev(bc), _dev(bsc), _dev(np.array(sizes, np.int32)))


def test_host_batches_overlapped_copies_match_direct_calls():
    """hostpipe.run_host_batches (H2D / GEMM / D2H on three streams, slots reused) writes each
    batch's C rows to its host tensor exactly as direct calls do."""
    from paper_2508_16584_b200.hostpipe import HostBatch, run_host_batches

    n, k, G = 256, 384, 3
    batches, wants = [], []
    _, _, bc, bsc = _synthetic((1, 1, 1), n, k, 77)
    b, sb = _dev(bc), _dev(bsc)
    for i in range(5):
        sizes = (37 * i + 1, 0 if i % 2 else 130, 64 + i)
        ac, asc, _, _ = _synthetic(sizes, n, k, i)
        gs = torch.tensor(sizes, dtype=torch.int32)
        on_host = i != 3  # one batch with device-resident inputs
        a = torch.from_numpy(ac).pin_memory() if on_host else _dev(ac)
        sa = torch.from_numpy(asc).pin_memory() if on_host else _dev(asc)
        out = torch.full((sum(sizes) + 5, n), 0x7BCD, dtype=torch.int16).pin_memory()
        batches.append(HostBatch(a, sa, gs.pin_memory(), out))
        want = tg.grouped_gemm_fp8(_dev(ac), _dev(asc), b, sb, gs.to(DEV))
        wants.append(want[:sum(sizes)].view(torch.int16).cpu())
    done = run_host_batches(batches, b, sb, depth=2)
    done.synchronize()
    for bt, want in zip(batches, wants):
        m = want.shape[0]
        assert torch.equal(bt.out[:m], want)
        assert bool((bt.out[m:] == 0x7BCD).all())  # rows past sum(M_g) untouched


def test_acceptance_random_configs_bitwise_vs_padded_and_oracle():
    """The reference's acceptance 06 (test_acceptance.py:180-201) on the GPU: 100 random
    configs (1/4/8 groups of 0..512 rows, N and K in {128, 192, 256, 384}, the reference's
    operand recipe).  The padding-free path equals the padded baseline bit for bit, and both
    match the oracle within helpers.REL_TOL."""
    rng = np.random.Generator(np.random.PCG64(2024))
    dims = (128, 192, 256, 384)
    for i in range(100):
        groups = int(rng.choice((1, 4, 8)))
        sizes = tuple(int(x) for x in rng.integers(0, 513, size=groups))
        n, k = int(rng.choice(dims)), int(rng.choice(dims))
        m = sum(sizes)
        ac, asc, bc, bsc = ofp8.random_operands(m, n, k, i)
        cfg = tg.ProblemConfig(n=n, k=k, group_sizes=sizes)
        ops = tg.GroupedOperands(ac, asc, bc, bsc)
        got = tg.run_adaptive(cfg, ops).c_bits
        want = tg.run_padded_baseline(cfg, ops)
        assert tg.verify_bitwise(got, want).equal, (i, sizes, n, k)
        if m:
            assert_parity(got, oracle_c(ac, asc, bc, bsc, sizes), label=f"config {i}")


@pytest.mark.parametrize("pdl", [True, False])
def test_back_to_back_launches_into_one_buffer_keep_stream_order(pdl):
    """Programmatic dependent launch: a grouped GEMM may start while the previous one drains,
    but stores only after it completed.  A long GEMM then a short one into the same output,
    with no sync between: the short one's rows hold its result, the rest the long one's."""
    n, k = 512, 1024
    big = (4000, 3000, 2500)
    small = (300, 0, 17)
    ab, asb, bcb, bsb = _synthetic(big, n, k, 1)
    as_, ass, bcs, bss = _synthetic(small, n, k, 2)
    want_big = tg.grouped_gemm_fp8(_dev(ab), _dev(asb), _dev(bcb), _dev(bsb), _dev(np.array(big, np.int32)))
    want_small = tg.grouped_gemm_fp8(_dev(as_), _dev(ass), _dev(bcs), _dev(bss), _dev(np.array(small, np.int32)))
    ms = sum(small)
    args_big = (_dev(ab), _dev(asb), _dev(bcb), _dev(bsb), _dev(np.array(big, np.int32)))
    args_small = (_dev(as_), _dev(ass), _dev(bcs), _dev(bss), _dev(np.array(small, np.int32)))
    out = torch.empty((sum(big), n), dtype=torch.bfloat16, device=DEV)
    torch.cuda.synchronize()
    for _ in range(20):
        tg.grouped_gemm_fp8(*args_big, out=out, pdl=pdl)
        tg.grouped_gemm_fp8(*args_small, out=out, pdl=pdl)
    torch.cuda.synchronize()
    assert torch.equal(out[:ms].view(torch.int16), want_small[:ms].view(torch.int16))
    assert torch.equal(out[ms:].view(torch.int16), want_big[ms:].view(torch.int16))


@pytest.mark.parametrize("depth", [1, 3])
def test_host_batches_depths_and_device_group_sizes(depth):
    """Slot depth 1 (fully serialized reuse) and 3; group sizes given on the device (the C
    rows copied back are then all m_alloc rows)."""
    from paper_2508_16584_b200.hostpipe import HostBatch, run_host_batches

    n, k = 128, 256
    _, _, bc, bsc = _synthetic((1, 1), n, k, 5)
    b, sb = _dev(bc), _dev(bsc)
    batches, wants = [], []
    for i in range(4):
        sizes = (50 + 30 * i, 7 * i)
        ac, asc, _, _ = _synthetic(sizes, n, k, 40 + i)
        gs_dev = _dev(np.array(sizes, np.int32))
        out = torch.zeros((sum(sizes), n), dtype=torch.int16).pin_memory()
        batches.append(HostBatch(torch.from_numpy(ac).pin_memory(), torch.from_numpy(asc).pin_memory(), gs_dev, out))
        wants.append(tg.grouped_gemm_fp8(_dev(ac), _dev(asc), b, sb, gs_dev).view(torch.int16).cpu())
    run_host_batches(batches, b, sb, depth=depth).synchronize()
    for bt, want in zip(batches, wants):
        assert torch.equal(bt.out, want[:bt.out.shape[0]])


def test_auto_tile_picks_1cta_for_skinny_groups():
    """tile=None: 1-CTA 128x128 tiles when m_alloc <= 128 G (the tile map shows the
    128x128 schedule), the CTA pair otherwise; values match the oracle either way."""
    from paper_2508_16584_b200._lib import lib

    n, k = 256, 384
    for sizes in ((5, 100, 0, 120), (300, 129, 2), (1, 2, 0, 1)):
        ac, asc, bc, bsc = _synthetic(sizes, n, k, sum(sizes))
        m = sum(sizes)
        tmap = torch.full((tg.max_tiles(m, len(sizes), n), 9), -1, dtype=torch.int32, device=DEV)
        out = tg.grouped_gemm_fp8(_dev(ac), _dev(asc), _dev(bc), _dev(bsc), _dev(np.array(sizes, np.int32)),
                                  tile_map=tmap)
        assert_parity(out.view(torch.int16).cpu().numpy().view(np.uint16), oracle_c(ac, asc, bc, bsc, sizes))
        tm = tmap.cpu().numpy()
        tm = sorted(tuple(int(x) for x in r) for r in tm[tm[:, 0] >= 0])
        skinny = m <= 128 * len(sizes)
        clusters = lib().tagg_launch_clusters(m, len(sizes), n, 0)
        tile = "1cta" if skinny else "pair_n256"
        assert tm == sorted(oplan.kernel_tile_map(sizes, n, tile, num_pairs=clusters))
