"""Pin the CPU oracle against the reference's own golden vectors (CPU only).

The oracle (oracle/) is trusted only because these tests hold: every
fixture under tests/golden/ was produced by the reference itself
(tests/golden/make_golden.py), including the reference's canonical
residual253 case whose sha256 values SURVEY.md Appendix A pins.
"""

from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

from oracle import fp8 as ofp8
from oracle import oracle as orc
from oracle import plan as oplan
from tmas import CASES, GOLDEN, load_case

SHA = {
    "a_codes.bin": "f1ee649821c385c950ea8a44ebf88acfeabfbbebd2d87ce9f80c842caec21d40",
    "a_scales.bin": "4ea4eb308de7c5919780939f7be88c5e04c833b9cc1523be5e113c2de151273f",
    "b_codes.bin": "2e0c0943f8e234cdf17f684a0bcf17a159766436d8273939988c458376e4933c",
    "b_scales.bin": "761ec4e0a7e023d0892eb83aed9cf8892cb2dc5166e7d80626c55033e5d10d88",
    "c_golden.bin": "65f249eaa68a96b04c6fc6c11171b956e157da7d3046ec9be881863024ffec75",
}


def test_residual253_fixture_matches_pinned_sha256():
    for name, want in SHA.items():
        got = hashlib.sha256((GOLDEN / "residual253" / name).read_bytes()).hexdigest()
        assert got == want, name


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("threads", [1, 3])
def test_oracle_reproduces_reference_goldens_bitwise(name, threads):
    c = load_case(name)
    layout = "nk" if c.get("b_layout") == "expert_nk" else "kn"
    got = orc.grouped_gemm(c["a_codes"], c["a_scales"], c["b_codes"], c["b_scales"],
                           c["group_sizes"], b_layout=layout, threads=threads)
    assert got.shape == c["c_golden"].shape
    assert np.array_equal(got, c["c_golden"]), name


def test_oracle_column_slices_compose():
    c = load_case("c1")
    full = c["c_golden"]
    out = np.zeros_like(full)
    for n0 in range(0, c["n"], 128):
        orc.grouped_gemm(c["a_codes"], c["a_scales"], c["b_codes"], c["b_scales"],
                         c["group_sizes"], n_range=(n0, n0 + 128), out=out)
    assert np.array_equal(out, full)


def test_oracle_row_offsets_leave_gaps_untouched():
    c = load_case("k640")
    sizes = c["group_sizes"]
    offs, o = [], 0
    for s in sizes:
        offs.append(o)
        o += s + 3  # 3-row gap after every group
    out = np.full((o, c["n"]), 0xBEEF, dtype=np.uint16)
    orc.grouped_gemm(c["a_codes"], c["a_scales"], c["b_codes"], c["b_scales"], sizes,
                     c_row_offsets=offs, out=out)
    a = 0
    for g, s in enumerate(sizes):
        assert np.array_equal(out[offs[g]:offs[g] + s], c["c_golden"][a:a + s])
        assert np.all(out[offs[g] + s:offs[g] + s + 3] == 0xBEEF)
        a += s


def test_scalar_triple_loop_matches_oracle():
    """test_engine.py:29-46 scalar oracle, restated with np.float32 scalars."""
    m_sizes, n, k = (5, 0, 14), 128, 192
    ac, asc, bc, bsc = ofp8.random_operands(sum(m_sizes), n, k, 3)
    f32 = np.float32
    a = ofp8.DECODE_TABLE[ac]
    b = ofp8.DECODE_TABLE[bc]
    want = np.zeros((sum(m_sizes), n), dtype=np.uint16)
    for m in range(sum(m_sizes)):
        for col in range(n):
            acc = f32(0)
            for kb in range(oplan.k_blocks(k)):
                inner = f32(0)
                for j in range(kb * 128, min(k, (kb + 1) * 128)):
                    inner = f32(inner + f32(a[m, j] * b[j, col]))
                scale = f32(asc[m, kb] * bsc[kb, col // 128])
                acc = f32(acc + f32(inner * scale))
            want[m, col] = orc.lib().tagg_oracle_bf16_from_f32(float(acc))
    got = orc.grouped_gemm(ac, asc, bc, bsc, m_sizes)
    assert np.array_equal(got, want)


def test_bf16_rounding_goldens():
    """test_engine.py:49-62"""
    L = orc.lib()
    cases = [(0x3F800000, 0x3F80), (0xC0000000, 0xC000), (0, 0),
             (0x3F808000, 0x3F80), (0x3F818000, 0x3F82), (0x3F808001, 0x3F81)]
    for u, want in cases:
        x = float(np.uint32(u).view(np.float32))
        assert L.tagg_oracle_bf16_from_f32(x) == want


def test_decode_table_matches_torch_e4m3fn():
    torch = pytest.importorskip("torch")
    codes = torch.arange(256, dtype=torch.uint8).view(torch.float8_e4m3fn).float().numpy()
    ours = ofp8.DECODE_TABLE
    nan = np.isnan(ours)
    assert np.array_equal(np.isnan(codes), nan)
    assert np.array_equal(codes[~nan], ours[~nan])
    L = orc.lib()
    for c in range(256):
        v = L.tagg_oracle_decode(c)
        assert (np.isnan(v) and nan[c]) or v == ours[c]


def test_planner_restatement_matches_reference_pins():
    pins = json.loads((GOLDEN / "plans.json").read_text())
    for key, text in pins["format_plan"].items():
        sizes = [int(x) for x in key.split(",")]
        assert oplan.format_plan(oplan.plan_group_stores(sizes, 128)) == text
    for rows, want in enumerate(pins["two_phase_128"]):
        got = oplan.plan_two_phase(rows, 128)
        assert (got is None and want is None) or list(got) == want
    for b, hs in pins["pool_heights"].items():
        assert oplan.pool_heights(int(b)) == hs
    for rb, row, start, rp, rn, tot in pins["prefetch"]:
        assert oplan.plan_prefetch(row * rb, rb, 128) == (start, rp, rn, tot)
    for sizes, n, k, m, pad, ba, bp, sav, elim, ops in pins["account"]:
        r = oplan.account(sizes, n, k)
        assert (r["m_total"], r["padded_rows"], r["bytes_actual"], r["bytes_padded"],
                r["eliminated_traffic_bytes"], r["residual_store_ops"]) == (m, pad, ba, bp, elim, ops)
        assert r["saving_pct"] == pytest.approx(sav, abs=1e-12)
    for m, g, s, want in pins["generate_group_sizes"]:
        assert list(oplan.generate_group_sizes(m, g, s)) == want


def test_c1_accounting_matches_survey_appendix():
    r = oplan.account((1, 67, 128, 255), 256, 512)
    assert r["m_total"] == 451 and r["padded_rows"] == 189
    assert r["bytes_actual"] == 469040 and r["bytes_padded"] == 665600
    assert r["saving_pct"] == pytest.approx(29.53125)
    assert r["eliminated_traffic_bytes"] == 199584 and r["residual_store_ops"] == 12


def test_tile_map_restatement_covers_rows_exactly():
    sizes = (1, 67, 128, 255, 0, 256, 129)
    recs = oplan.tile_map(sizes, 256)
    m = sum(sizes)
    hits = np.zeros((m, 2), dtype=int)
    for g, t, n0, r0, valid, d, ag, bs, bg in recs:
        for gm in (ag, bg) if valid < 128 else (ag,):
            hits[gm:gm + d, n0 // 128] += 1
        # never beyond the group's last row
        off = sum(sizes[:g])
        assert bg + d <= off + sizes[g]
    assert np.all(hits >= 1)


@pytest.mark.parametrize("sizes", [(1, 67, 128, 255, 0, 256, 129), (64, 65, 192, 320, 384, 3), (128 * 3 + 77,),
                                   tuple(128 * g + 64 for g in range(8))])
@pytest.mark.parametrize("pairs", [None, 3, 74])
@pytest.mark.parametrize("raster", [1, 8, 64])
def test_kernel_tile_map_stores_exactly_the_reference_rows(sizes, pairs, raster):
    """The kernel's half-tile pieces (64-row reference plans, group tails and the
    tail-balanced last wave) cover exactly the rows of the reference tile loop and
    never a row past M_g."""
    n = 512
    ker = oplan.kernel_tile_map(sizes, n, num_pairs=pairs, raster=raster)
    ref = oplan.tile_map(sizes, n)
    rows = lambda recs: sorted({(r[0], r[2], x) for r in recs for x in range(r[6], r[6] + r[4])})  # noqa: E731
    assert rows(ker) == rows(ref)
    for g, t, n0, r0, valid, d, ag, bs, bg in ker:
        off = sum(sizes[:g])
        assert 1 <= valid and d <= valid < 2 * d
        assert ag + d <= off + sizes[g] and bg + d <= off + sizes[g]
        assert bg - ag == valid - d == bs


def test_moe_oracle_combine_and_swiglu_against_float64():
    """The MoE step oracles (oracle/moe.py) against float64 arithmetic."""
    from oracle import moe as omoe

    rng = np.random.default_rng(0)
    c = omoe.bf16_rne(rng.standard_normal((40, 16)).astype(np.float32))
    dest = rng.permutation(40).astype(np.int32)
    w = rng.random((10, 4)).astype(np.float32)
    got = ofp8.bf16_bits_to_f32(omoe.combine(c, dest, w)).astype(np.float64)
    want = (w[:, :, None].astype(np.float64) * ofp8.bf16_bits_to_f32(c)[dest].reshape(10, 4, 16)).sum(1)
    assert np.all(np.abs(got - want) <= 2.0 ** -7 * np.abs(want) + 1e-30)
    h = omoe.bf16_rne(rng.standard_normal((5, 32)).astype(np.float32) * 4)
    hf = ofp8.bf16_bits_to_f32(h).astype(np.float64)
    ref = hf[:, :16] / (1 + np.exp(-hf[:, :16])) * hf[:, 16:]
    np.testing.assert_allclose(omoe.swiglu(h), ref, rtol=1e-6, atol=1e-30)
    # bf16 RNE ties (engine.py:49 goldens, test_engine.py:49-62)
    assert list(omoe.bf16_rne(np.array([0x3F808000, 0x3F818000, 0x3F808001], np.uint32).view(np.float32))) == \
        [0x3F80, 0x3F82, 0x3F81]


@pytest.mark.parametrize("name", CASES)
def test_input_recipe_reproduces_golden_operand_bytes(name):
    """oracle/fp8.random_operands (the restatement of cli.py:112-121 + fp8.py:54-176) draws
    exactly the operand bytes the reference wrote for every fixture.  The GPU quantizer
    tests compare against this restatement, so this pins it to the reference itself."""
    c = load_case(name)
    sizes, n, k, seed = c["group_sizes"], c["n"], c["k"], c["seed"]
    m = int(sum(sizes))
    ac, asc, bc, bsc = ofp8.random_operands(m, n, k, seed)
    assert np.array_equal(ac, c["a_codes"]), "A codes"
    assert np.array_equal(asc.view(np.uint32), c["a_scales"].view(np.uint32)), "A scales"
    if c["b_layout"] == "shared_kn":
        assert np.array_equal(bc, c["b_codes"]), "B codes"
        assert np.array_equal(bsc.view(np.uint32), c["b_scales"].view(np.uint32)), "B scales"
        return
    # per-expert fixtures: expert g's B is drawn from seed * 1000 + 17 + g (make_golden.py)
    for g in range(len(sizes)):
        _, _, b, sb = ofp8.random_operands(1, n, k, seed * 1000 + 17 + g)
        if c["b_layout"] == "expert_nk":
            b, sb = b.T, sb.T
        assert np.array_equal(b, c["b_codes"][g]), f"B codes expert {g}"
        assert np.array_equal(sb.view(np.uint32), np.ascontiguousarray(c["b_scales"][g]).view(np.uint32)), g
