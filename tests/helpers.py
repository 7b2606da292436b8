"""Shared test helpers: the parity tolerance and the oracle comparisons."""

from __future__ import annotations

import numpy as np

from oracle import fp8 as ofp8
from oracle import oracle as orc

# Parity tolerance for bf16 C (SURVEY.md §8a / BASELINE.md §4):
#   |c - c_ref| <= 2^-7 * max(|c_ref|, 2^-10 * rowabsmax(c_ref))
# The oracle's products are exact.  Only the fp32 add order inside a 128-wide
# k block differs (tensor cores vs the reference's sequential chain).  The
# FFMA2 promotion also rounds once instead of twice.  2^-7 is one bf16 ulp at
# the value's own magnitude.  The row-max floor covers cancellation (elements
# far below the row's scale).
REL_TOL = 2.0 ** -7
FLOOR = 2.0 ** -10


def tolerance_report(got_bits: np.ndarray, want_bits: np.ndarray) -> dict:
    assert got_bits.shape == want_bits.shape
    got = ofp8.bf16_bits_to_f32(got_bits).astype(np.float64)
    ref = ofp8.bf16_bits_to_f32(want_bits).astype(np.float64)
    if ref.size == 0:
        return dict(out_of_tol=0, bit_identical=1.0, max_rel=0.0, n=0)
    rowmax = np.abs(ref).max(axis=1, keepdims=True)
    tol = REL_TOL * np.maximum(np.abs(ref), FLOOR * rowmax)
    err = np.abs(got - ref)
    nan_mismatch = np.isnan(got) != np.isnan(ref)
    bad = (err > tol) | nan_mismatch
    denom = np.maximum(np.abs(ref), FLOOR * rowmax)
    rel = np.where(denom > 0, err / np.where(denom > 0, denom, 1), 0)
    return dict(out_of_tol=int(bad.sum()), bit_identical=float((got_bits == want_bits).mean()),
                max_rel=float(np.nanmax(rel)) if rel.size else 0.0, n=int(ref.size))


def assert_parity(got_bits, want_bits, min_identical=0.0, label=""):
    rep = tolerance_report(got_bits, want_bits)
    assert rep["out_of_tol"] == 0, f"{label}: {rep}"
    assert rep["bit_identical"] >= min_identical, f"{label}: {rep}"
    return rep


def oracle_c(ac, asc, bc, bsc, sizes, b_layout="kn", threads=8, **kw):
    return orc.grouped_gemm(ac, asc, bc, bsc, sizes, b_layout=b_layout, threads=threads, **kw)


def per_expert_operands(sizes, n, k, seed):
    """A/S_A with the reference recipe.  Each expert's B/S_B comes from its own seed."""
    m = int(sum(sizes))
    ac, asc, _, _ = ofp8.random_operands(m, 64, k, seed)
    bs, sbs = [], []
    for g in range(len(sizes)):
        _, _, b, sb = ofp8.random_operands(1, n, k, seed * 1000 + 17 + g)
        bs.append(b)
        sbs.append(sb)
    return ac, asc, np.stack(bs), np.stack(sbs)
